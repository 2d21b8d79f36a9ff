"""Table-III GEMM chains (reference fixtures bench.cpp:27-30 at
scale 1: 4096 extents) through the executor at P = 1: which kernels run, the
device time (CUDA events on the executor's stream, after warm-up), the FP64
roofline fraction, and a spot check of two output rows against numpy.

    python tools/gemm_chain_check.py [--out profiles/gemm_chain_r02.jsonl]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2206_08301_b200 as eb  # noqa: E402
from paper_2206_08301_b200 import _capi  # noqa: E402

FP64_PEAK = 37.05  # measured DMMA peak (profiles/fp64_peak_r01.jsonl)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default=None, help="1MM / 2MM / 3MM")
    a = ap.parse_args()
    n = a.n
    lines = []
    for name, e in [("1MM", "ij,jk->ik"), ("2MM", "ij,jk,kl->il"), ("3MM", "ij,jk,kl,lm->im")]:
        if a.only and name != a.only:
            continue
        ins = e.split("->")[0].split(",")
        ext = {c: n for t in ins for c in t}
        ops = [eb.random_tensor(tuple(ext[c] for c in t), k) for k, t in enumerate(ins)]
        st = torch.cuda.Stream()
        ex = eb.Executor(e, ext, 1, stream=st.cuda_stream)
        ex.stage(ops)
        for _ in range(2):
            ex.run()
        torch.cuda.synchronize()
        L = _capi.lib()
        L.eb_timer_enable(1)
        L.eb_timer_collect(None, None)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(a.reps):
            ex.run()
        e1.record(st)
        torch.cuda.synchronize()
        import ctypes
        kms, kn = ctypes.c_double(0), ctypes.c_longlong(0)
        L.eb_timer_collect(ctypes.byref(kms), ctypes.byref(kn))
        L.eb_timer_enable(0)
        ms = e0.elapsed_time(e1) / a.reps
        s = ex.stats()
        out = ex.gather().reshape(n, n)
        err = 0.0
        for r in (5, n - 3):
            ref = ops[0][r:r + 1]
            for o in ops[1:]:
                ref = ref @ o
            err = max(err, float(np.linalg.norm(out[r] - ref[0]) / np.linalg.norm(ref[0])))
        tf = s["tree_flops"] / (ms * 1e-3) / 1e12
        line = {"kernel": name, "einsum": e, "n": n, "ms_per_run": ms, "tflops": tf,
                "frac_fp64_peak": tf / FP64_PEAK, "main_kernel_ms_per_run": kms.value / a.reps,
                "main_kernel_launches_per_run": kn.value / a.reps, "row_rel_err": err,
                **{k: s[k] for k in ("fused_launches", "ttm_launches", "generic_launches",
                                     "tree_flops")}}
        print(json.dumps(line), flush=True)
        lines.append(line)
        ex.close()
        del ops
    if a.out:
        with open(a.out, "w") as f:
            for l in lines:
                f.write(json.dumps(l) + "\n")


if __name__ == "__main__":
    main()
