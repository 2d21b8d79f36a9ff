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


def c5_slabs(slabs):
    """C5 goldens for P = 2, 4, 8 (global X = random_tensor(
    (64P, 64, 64, 64, 64), 0), one row-major stream).  Mode-0 TTMc rows
    depend only on X[i], so output rows [64p, 64p + 64) of every P > p are the
    reference run() at P = 1 on the 64-row slab p of the seed-0 stream (stream
    elements [p*64^5, (p+1)*64^5)) with the same four 64x16 factors (seeds
    1..4).  Slab 0 is the P = 1 golden (C5_summary.json)."""
    meta_path = os.path.join(GOLD, "reference_runs.json")
    meta = json.load(open(meta_path)) if os.path.exists(meta_path) else {}
    c = CONFIGS["C5"]
    e = c["einsums"][0]
    ext = c["extents"](1)
    ins, _ = oracle.parse(e)
    n = 64 ** 5
    for p in slabs:
        tag = f"C5_slab{p}"
        if os.path.exists(os.path.join(GOLD, f"{tag}_summary.json")):
            continue
        t = time.time()
        ops = [oracle.random_tensor(oracle.shape_of(ins[0], ext), 0, skip=p * n)]
        ops += [oracle.random_tensor(oracle.shape_of(s, ext), k + 1) for k, s in enumerate(ins[1:])]
        out, secs, comm = oracle.ref_run(e, ext, 1, ops)
        wall = time.time() - t
        del ops
        with open(os.path.join(GOLD, f"{tag}_summary.json"), "w") as f:
            json.dump(summary(out), f)
        meta[tag] = {"einsum": e, "extents": ext, "procs": 1, "x_stream_skip": p * n,
                     "run_seconds": secs, "wall_seconds": wall, "comm": list(comm), "threads": 1}
        json.dump(meta, open(meta_path, "w"), indent=1)
        print(tag, f"run() {secs:.1f}s wall {wall:.1f}s", flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "plans":
        plans()
    elif sys.argv[1] == "c5slabs":
        c5_slabs([int(x) for x in sys.argv[2:]] or list(range(1, 8)))
    else:
        outputs(sys.argv[2:] or ["C1", "C3", "C5", "C2", "C4"])
