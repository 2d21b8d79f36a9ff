"""Multi-GPU scaling proxy on one B200: every BASELINE config at P = 1, 2,
4, 8 with the P ranks virtual on the one device (the same per-rank blocks,
kernels, reductions and fused redistributions a P-GPU run executes, one rank
after the other).  Device time per run T_P (CUDA events); per-GPU time =
T_P / P.  Efficiency proxies:
  strong scaling (C1-C4): T_1 / T_P          (= T_1 / (P x per-GPU time))
  weak scaling (C5):      T_1 / (T_P / P)
They include everything a rank computes and copies locally but no
interconnect time (NVLink transfers, collective latency): an upper bound on
the real efficiency, and the per-rank work balance it depends on.

    python tools/scaling_proxy.py [out.jsonl]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2206_08301_b200 as eb  # noqa: E402
from tests.configs import CONFIGS, C2_FACTOR_SEED  # noqa: E402


def stage(ex, name, e, ext, P, X1024=None):
    ins = e.split("->")[0].split(",")
    if name in ("C2", "C4") and X1024 is not None:
        ex.stage_region(0, [0, 0, 0], X1024)
    elif name == "C5":
        plan = json.loads(eb.plan_json(e, ext, P))
        rows = 64 * P // plan["schedule"]["terms"][0]["grid"]["i"]
        rng = eb.RandomStream(0)
        region = np.empty((rows, 64, 64, 64, 64))
        for i0 in range(0, 64 * P, rows):
            rng.fill(region.reshape(-1))
            ex.stage_region(0, [i0, 0, 0, 0, 0], region)
        del region
    else:
        X = eb.random_tensor(tuple(ext[c] for c in ins[0]), 0)
        ex.stage_region(0, [0] * X.ndim, X)
    for k, t in enumerate(ins[1:]):
        seed = C2_FACTOR_SEED[t[0]] if name == "C2" else k + 1
        f = eb.random_tensor((ext[t[0]], ext[t[1]]), seed)
        ex.stage_region(k + 1, [0, 0], f)


def time_run(exs, st, reps=5):
    for _ in range(2):
        for ex in exs:
            ex.run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        for ex in exs:
            ex.run()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    out = []
    X1024 = np.empty((1024, 1024, 1024))
    eb.RandomStream(0).fill(X1024.reshape(-1))
    for name in ("C1", "C2", "C3", "C4", "C5"):
        c = CONFIGS[name]
        T1 = None
        for P in (1, 2, 4, 8):
            ext = c["extents"](P)
            st = torch.cuda.Stream()
            exs = []
            for mi, e in enumerate(c["einsums"]):
                ex = eb.Executor(e, ext, P, stream=st.cuda_stream)
                stage(ex, name, e, ext, P, X1024)
                exs.append(ex)
            ms = time_run(exs, st)
            stats = [ex.stats() for ex in exs]
            if P == 1:
                T1 = ms
            eff = T1 / ms if name != "C5" else T1 / (ms / P)
            line = {"config": name, "P": P, "ms_virtual_total": ms, "ms_per_gpu": ms / P,
                    "efficiency_proxy": eff,
                    "scaling": "weak" if name == "C5" else "strong",
                    "allreduce_volume": sum(s["allreduce_volume"] for s in stats),
                    "redistribute_volume": sum(s["redistribute_volume"] for s in stats),
                    "fused_redistributions": sum(s["fused_redistributions"] for s in stats)}
            print(json.dumps(line), flush=True)
            out.append(line)
            for ex in exs:
                ex.close()
            del exs
            torch.cuda.empty_cache()
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            for l in out:
                f.write(json.dumps(l) + "\n")


if __name__ == "__main__":
    main()
