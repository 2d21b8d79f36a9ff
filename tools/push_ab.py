"""A/B of the fused redistribution (TTM epilogue push, eb_scatter) against
the separate apply_plan copy, on virtual ranks at BASELINE size:
C4 at P = 2, 4, 8 and C5 at P = 4 (the configs whose schedules move data).
Device time per run (CUDA events on the executor stream, after warm-up)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2206_08301_b200 as eb  # noqa: E402
from tests.configs import CONFIGS  # noqa: E402


def stage_c4(ex, ext):
    X = np.empty((1024, 1024, 1024))
    eb.RandomStream(0).fill(X.reshape(-1))
    ex.stage_region(0, [0, 0, 0], X)
    del X
    for k, t in enumerate(("jb", "kc")):
        ex.stage_region(k + 1, [0, 0], eb.random_tensor((ext[t[0]], ext[t[1]]), k + 1))


def stage_c5(ex, ext, P, rows):
    rng = eb.RandomStream(0)
    region = np.empty((rows, 64, 64, 64, 64))
    for i0 in range(0, 64 * P, rows):
        rng.fill(region.reshape(-1))
        ex.stage_region(0, [i0, 0, 0, 0, 0], region)
    del region
    for k, t in enumerate(("jb", "kc", "ld", "me")):
        ex.stage_region(k + 1, [0, 0], eb.random_tensor((ext[t[0]], ext[t[1]]), k + 1))


def time_runs(ex, st, reps=5):
    for _ in range(2):
        ex.run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        ex.run()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    out = []
    cases = [("C4", P) for P in (2, 4, 8)] + [("C5", 4)]
    if os.environ.get("PUSH_AB_ONLY"):  # e.g. "C5:4"
        n, p = os.environ["PUSH_AB_ONLY"].split(":")
        cases = [(n, int(p))]
    for name, P in cases:
        c = CONFIGS[name]
        e, ext = c["einsums"][0], c["extents"](P)
        st = torch.cuda.Stream()
        ex = eb.Executor(e, ext, P, stream=st.cuda_stream)
        if name == "C4":
            stage_c4(ex, ext)
        else:
            plan = json.loads(eb.plan_json(e, ext, P))
            stage_c5(ex, ext, P, 64 * P // plan["schedule"]["terms"][0]["grid"]["i"])
        res = {"config": name, "P": P}
        outs = [None, None]
        times = {0: [], 1: []}
        for _ in range(3):  # interleaved A/B rounds (clock drift hits both alike)
            for fuse in (0, 1):
                eb.set_option("fuse_redistribution", fuse)
                times[fuse].append(time_runs(ex, st))
                s = ex.stats()
                outs[fuse] = ex.gather()
                res["fused" if fuse else "separate"] = {
                    "fused_redistributions": s["fused_redistributions"],
                    "redistribute_volume": s["redistribute_volume"]}
        for fuse in (0, 1):
            res["fused" if fuse else "separate"]["ms_per_run"] = sorted(times[fuse])[1]
            res["fused" if fuse else "separate"]["ms_rounds"] = times[fuse]
        res["bitwise_equal"] = bool(np.array_equal(outs[0], outs[1]))
        res["saved_ms"] = res["separate"]["ms_per_run"] - res["fused"]["ms_per_run"]
        print(json.dumps(res), flush=True)
        out.append(res)
        ex.close()
        torch.cuda.empty_cache()
    eb.set_option("fuse_redistribution", 1)
    if len(sys.argv) > 1 and not os.environ.get("PUSH_AB_ONLY"):
        with open(sys.argv[1], "w") as f:
            for r in out:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
