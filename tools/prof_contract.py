"""Run eb_contract on a BASELINE term shape: a few launches (for ncu captures),
or timed A/B variants with CUDA events.

usage: python tools/prof_contract.py CFG [REPS] [ENV=VAL,... ...]
  CFG in c1, c2m0, c2m1, c2m2, c2pair (eb_mttkrp2: modes 0+1 in one pass), c3,
  p8m0/p8m1/p8m2 (C2's per-GPU 512^3 block at P = 8).  With variant args, the variants are run
  round-robin (3 rounds) and the best ms / TFLOP/s of each is printed; a variant is
  NAME=VAL,... where lower-case names are eb_set_option options (e.g. row_tile=1).
"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_08301_b200 import _capi as C  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2m0"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
variants = sys.argv[3:]
dev = torch.device("cuda:0")


def fac(t):
    return C.Factor(t.data_ptr(), t.shape[0], t.shape[1])


def desc(variant, P, M, Q, L, R, X, U, pre, mid, out, mode=C.EB_REDUCE):
    d = C.ContractDesc()
    d.variant, d.mode, d.P, d.M, d.Q, d.L, d.R = variant, mode, P, M, Q, L, R
    d.X, d.U, d.ldu = X.data_ptr(), U.data_ptr(), U.shape[1]
    d.n_pre = len(pre)
    for i, f in enumerate(pre): d.pre[i] = fac(f)
    d.n_mid = len(mid)
    for i, f in enumerate(mid): d.mid[i] = fac(f)
    d.out = out.data_ptr()
    return d


r = lambda *s: torch.rand(*s, dtype=torch.float64, device=dev)
if cfg.startswith("c2"):
    X = r(1024, 1024, 1024); A, B, Cm = r(1024, 32), r(1024, 32), r(1024, 32)
    out = torch.zeros(1024, 32, dtype=torch.float64, device=dev)
    out1 = torch.zeros(1024, 32, dtype=torch.float64, device=dev)
    d = {"c2m0": lambda: desc(C.EB_ROW, 1, 1024, 1024, 1024, 32, X, Cm, [], [B], out),
         "c2pair": lambda: desc(C.EB_ROW, 1, 1024, 1024, 1024, 32, X, Cm, [], [B], out),
         "c2m1": lambda: desc(C.EB_ROW, 1024, 1024, 1, 1024, 32, X, Cm, [A], [], out),
         "c2m2": lambda: desc(C.EB_COL, 1024, 1024, 1024, 0, 32, X, B, [A], [], out)}[cfg]()
    flops = 2.0 * 1024 ** 3 * 32
elif cfg.startswith("p8"):  # C2's per-GPU block at P=8 (grid i2 j2 k2): 512^3, R = 32
    X = r(512, 512, 512); A, B, Cm = r(512, 32), r(512, 32), r(512, 32)
    out = torch.zeros(512, 32, dtype=torch.float64, device=dev)
    d = {"p8m0": lambda: desc(C.EB_ROW, 1, 512, 512, 512, 32, X, Cm, [], [B], out),
         "p8m1": lambda: desc(C.EB_ROW, 512, 512, 1, 512, 32, X, Cm, [A], [], out),
         "p8m2": lambda: desc(C.EB_COL, 512, 512, 512, 0, 32, X, B, [A], [], out)}[cfg]()
    flops = 2.0 * 512 ** 3 * 32
elif cfg == "c1":
    X = r(512, 512, 512); B, Cm = r(512, 24), r(512, 24)
    out = torch.zeros(512, 24, dtype=torch.float64, device=dev)
    d = desc(C.EB_ROW, 1, 512, 512, 512, 24, X, Cm, [], [B], out)
    flops = 2.0 * 512 ** 3 * 24
elif cfg == "c3":
    X = r(64, 64, 64, 64, 64); F = [r(64, 24) for _ in range(4)]
    out = torch.zeros(64, 24, dtype=torch.float64, device=dev)
    d = desc(C.EB_ROW, 1, 64, 64 ** 3, 64, 24, X, F[3], [], F[:3], out)
    flops = 2.0 * 64 ** 5 * 24
L = C.lib()
pair = cfg == "c2pair"
wsfn = L.eb_mttkrp2_workspace if pair else L.eb_contract_workspace
wsb = wsfn(ctypes.byref(d))
ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=dev)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def launch():
    global ws, wsb
    need = wsfn(ctypes.byref(d))  # the tiling may depend on EB_* knobs
    if need > wsb:
        wsb, ws = need, torch.empty(need, dtype=torch.uint8, device=dev)
    if pair:
        C.check(L.eb_mttkrp2(ctypes.byref(d), ctypes.c_void_p(A.data_ptr()), 32,
                             ctypes.c_void_p(out1.data_ptr()), ctypes.c_void_p(ws.data_ptr()), wsb, st))
    else:
        C.check(L.eb_contract(ctypes.byref(d), ctypes.c_void_p(ws.data_ptr()), wsb, st))


if not variants:
    for _ in range(reps):
        launch()
    torch.cuda.synchronize()
    print("done", cfg)
    sys.exit(0)

res = {}
for rnd in range(3):
    for v in variants:
        kv = [x.split("=") for x in v.split(",") if x]
        for k, val in kv:  # lower-case names are eb_set_option options
            if k.islower():
                C.check(L.eb_set_option(k.encode(), val.encode()))
            else:
                os.environ[k] = val
        launch(); launch()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            launch()
        e1.record()
        torch.cuda.synchronize()
        res.setdefault(v, []).append(e0.elapsed_time(e1) / reps)
        for k, _ in kv:
            os.environ.pop(k, None)
for v, ms in res.items():
    print(json.dumps({"cfg": cfg, "variant": v, "ms_best": round(min(ms), 4),
                      "ms_all": [round(x, 4) for x in ms],
                      "TFLOPs": round(flops / min(ms) / 1e9, 2)}))
