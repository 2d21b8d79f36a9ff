"""A/B timing of eb_ttm2 on the C5 term shapes (CUDA events, inputs resident).

term0: X[i=64][j=64][k=64][lm=4096] -> out[64][4096][16][16]
term1: t1[i=64][l=64][m=64][bc=256] -> out[64][256][16][16]

usage: python tools/ttm2_bench.py REPS [ENV=VAL,ENV=VAL ...]   (one arg per variant;
variants are interleaved round-robin, 3 rounds, so box drift hits all of them)
"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_08301_b200 import _capi as C  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
variants = sys.argv[2:] or [""]
try:
    import pynvml
    pynvml.nvmlInit()
    H = pynvml.nvmlDeviceGetHandleByIndex(0)
except Exception:
    H = None

dev = torch.device("cuda:0")
L = C.lib()
st = torch.cuda.current_stream()
s = ctypes.c_void_p(st.cuda_stream)
shapes = {"term0": (64, 64, 64, 4096), "term1": (64, 64, 64, 256)}
bufs = {}
for name, (P, Q1, Q2, M) in shapes.items():
    X = torch.rand(P, Q1, Q2, M, dtype=torch.float64, device=dev)
    U1 = torch.rand(Q1, 16, dtype=torch.float64, device=dev)
    U2 = torch.rand(Q2, 16, dtype=torch.float64, device=dev)
    out = torch.empty(P, M, 16, 16, dtype=torch.float64, device=dev)
    d = C.Ttm2Desc(P, Q1, Q2, M, 16, 16, X.data_ptr(), U1.data_ptr(), 16, U2.data_ptr(), 16,
                   out.data_ptr())
    bufs[name] = (X, U1, U2, out, d)


def set_env(v):
    for kv in filter(None, v.split(",")):
        k, val = kv.split("=")
        os.environ[k] = val


res = {}
for rnd in range(3):
    for v in variants:
        set_env(v)
        for name, (P, Q1, Q2, M) in shapes.items():
            X, U1, U2, out, d = bufs[name]
            for _ in range(2):
                C.check(L.eb_ttm2(ctypes.byref(d), s))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            for _ in range(reps):
                C.check(L.eb_ttm2(ctypes.byref(d), s))
            e1.record(st)
            clk = pynvml.nvmlDeviceGetClockInfo(H, pynvml.NVML_CLOCK_SM) if H else None
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            res.setdefault((v, name), []).append((ms, clk))
        for kv in filter(None, v.split(",")):
            os.environ.pop(kv.split("=")[0], None)

for (v, name), runs in res.items():
    P, Q1, Q2, M = shapes[name]
    X, U1, U2, out, d = bufs[name]
    ms = min(r[0] for r in runs)
    flops = 2.0 * P * Q1 * Q2 * M * 16 + 2.0 * P * Q2 * M * 16 * 16
    byts = 8.0 * (X.numel() + out.numel())
    print(json.dumps({"variant": v, "shape": name, "ms_best": round(ms, 4),
                      "ms_all": [round(r[0], 4) for r in runs], "sm_mhz": [r[1] for r in runs],
                      "TFLOPs": round(flops / ms / 1e9, 2), "GBs": round(byts / ms / 1e6, 1)}))
# correctness spot check of the last variant run
X, U1, U2, out, d = bufs["term1"]
C.check(L.eb_ttm2(ctypes.byref(d), s))
torch.cuda.synchronize()
ref = torch.einsum("pjkm,jb,kc->pmbc", X[:2], U1, U2)
print(json.dumps({"normwise_err_term1": ((out[:2] - ref).norm() / ref.norm()).item()}))
