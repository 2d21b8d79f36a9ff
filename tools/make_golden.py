"""Generate tests/golden/ from the REFERENCE implementation (oracle/_ref,
compiled from /root/reference/proj/src by oracle/Makefile).

Run here (the container that has /root/reference); the outputs are small
committed fixtures, so the GPU box never needs the reference.

  python tools/make_golden.py plans      # plan JSON per config x P (seconds)
  python tools/make_golden.py outputs    # full-size reference runs (~20 min)
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from tests.configs import CONFIGS, c2_inputs, seeded  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def plans():
    os.makedirs(os.path.join(GOLD, "plans"), exist_ok=True)
    for name, c in CONFIGS.items():
        for P in c["procs"]:
            ext = c["extents"](P)
            for mode, e in enumerate(c["einsums"]):
                txt = oracle.ref_plan_json(e, ext, P, 1024.0, include_messages=True)
                tag = f"{name}_m{mode}" if len(c["einsums"]) > 1 else name
                with open(os.path.join(GOLD, "plans", f"{tag}_P{P}.json"), "w") as f:
                    f.write(txt)
    print("plans written")


SAMPLE = 4096


def summary(out):
    flat = out.ravel()
    idx = np.random.default_rng(1234).choice(flat.size, size=min(SAMPLE, flat.size), replace=False)
    idx.sort()
    return {"shape": list(out.shape), "sum": float(flat.sum()),
            "norm2": float(np.sqrt(np.sum(flat.astype(np.longdouble) ** 2))),
            "sample_index": idx.tolist(), "sample_value": flat[idx].tolist()}


def outputs(which):
    meta_path = os.path.join(GOLD, "reference_runs.json")
    meta = json.load(open(meta_path)) if os.path.exists(meta_path) else {}
    for name in which:
        c = CONFIGS[name]
        P = 1
        ext = c["extents"](P)
        for mode, e in enumerate(c["einsums"]):
            tag = f"{name}_m{mode}" if len(c["einsums"]) > 1 else name
            ops = c2_inputs(mode, ext) if name == "C2" else seeded(e, ext, 0)
            t = time.time()
            out, secs, comm = oracle.ref_run(e, ext, P, ops)
            wall = time.time() - t
            del ops
            if out.size <= 65536:
                np.save(os.path.join(GOLD, f"{tag}_out.npy"), out)
            with open(os.path.join(GOLD, f"{tag}_summary.json"), "w") as f:
                json.dump(summary(out), f)
            meta[tag] = {"einsum": e, "extents": ext, "procs": P, "run_seconds": secs,
                         "wall_seconds": wall, "comm": list(comm), "threads": 1}
            json.dump(meta, open(meta_path, "w"), indent=1)
            print(tag, f"run() {secs:.1f}s", flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "plans":
        plans()
    else:
        outputs(sys.argv[2:] or ["C1", "C3", "C5", "C2", "C4"])
