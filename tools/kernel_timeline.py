"""Warm per-kernel timeline of one BASELINE config at P virtual ranks
(torch.profiler / CUPTI activity records: real concurrent timings, no cache
flush, no serialisation — unlike an ncu launch list).  Prints, per kernel
name, the launch count and mean duration per run, then the busy time, the
span and the idle gaps of one run.

    python tools/kernel_timeline.py C1 8 [--reps 5] [--out f.json]
"""
import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

import paper_2206_08301_b200 as eb  # noqa: E402
from scaling_proxy import stage  # noqa: E402
from tests.configs import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("P", type=int)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    c = CONFIGS[a.config]
    ext = c["extents"](a.P)
    st = torch.cuda.Stream()
    exs = []
    X1024 = None
    if a.config in ("C2", "C4"):
        import numpy as np
        X1024 = np.empty((1024, 1024, 1024))
        eb.RandomStream(0).fill(X1024.reshape(-1))
    for e in c["einsums"]:
        ex = eb.Executor(e, ext, a.P, stream=st.cuda_stream)
        stage(ex, a.config, e, ext, a.P, X1024)
        exs.append(ex)
    for _ in range(3):
        for ex in exs:
            ex.run()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.reps):
            for ex in exs:
                ex.run()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    by = collections.OrderedDict()
    for e in evs:
        k = e.name.replace("(anonymous namespace)::", "").split("(")[0][:90]
        n, t = by.get(k, (0, 0.0))
        by[k] = (n + 1, t + e.time_range.elapsed_us())
    busy = sum(e.time_range.elapsed_us() for e in evs)
    span = evs[-1].time_range.end - evs[0].time_range.start
    gaps = []
    for x, y in zip(evs, evs[1:]):
        gaps.append(y.time_range.start - x.time_range.end)
    res = {"config": a.config, "P": a.P, "reps": a.reps,
           "kernels": {k: {"launches_per_run": n / a.reps, "us_per_run": t / a.reps,
                           "us_per_launch": t / n} for k, (n, t) in by.items()},
           "busy_us_per_run": busy / a.reps, "span_us_per_run": span / a.reps,
           "gap_us_per_run": sum(g for g in gaps if g > 0) / a.reps,
           "overlap_us_per_run": -sum(g for g in gaps if g < 0) / a.reps}
    print(json.dumps(res, indent=1))
    if a.out:
        with open(a.out, "a") as f:
            f.write(json.dumps(res) + "\n")


if __name__ == "__main__":
    main()
