"""C5 (TTMc order 5) at P = 1: both fused TTM-pair terms over the whole i
range (t1 = 537 MB round-trips HBM) vs interleaved over i-chunks with one
reused t1 chunk buffer (L2 residency of the intermediate).

usage: python tools/c5_chunk_exp.py REPS CHUNK [CHUNK ...]   (CHUNK 64 = unchunked)
"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_08301_b200 import _capi as C  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
chunks = [int(c) for c in sys.argv[2:]] or [64, 16, 8, 4]
dev = torch.device("cuda:0")
L = C.lib()
st = torch.cuda.current_stream()
s = ctypes.c_void_p(st.cuda_stream)
n = 64
X = torch.rand(n, n, n, n, n, dtype=torch.float64, device=dev)
U = [torch.rand(n, 16, dtype=torch.float64, device=dev) for _ in range(4)]
out = torch.empty(n, 16, 16, 16, 16, dtype=torch.float64, device=dev)
t1_full = torch.empty(n, n, n, 16, 16, dtype=torch.float64, device=dev)


def run(pc):
    t1 = t1_full if pc == n else t1_full[:pc]
    for i0 in range(0, n, pc):
        d0 = C.Ttm2Desc(pc, n, n, n * n, 16, 16, X[i0].data_ptr(), U[0].data_ptr(), 16,
                        U[1].data_ptr(), 16, t1.data_ptr())
        C.check(L.eb_ttm2(ctypes.byref(d0), s))
        d1 = C.Ttm2Desc(pc, n, n, 256, 16, 16, t1.data_ptr(), U[2].data_ptr(), 16,
                        U[3].data_ptr(), 16, out[i0].data_ptr())
        C.check(L.eb_ttm2(ctypes.byref(d1), s))


run(n)
torch.cuda.synchronize()
ref = out.clone()
res = {}
for rnd in range(3):
    for pc in chunks:
        run(pc)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            run(pc)
        e1.record(st)
        torch.cuda.synchronize()
        res.setdefault(pc, []).append(e0.elapsed_time(e1) / reps)
        assert (out - ref).norm() <= 1e-13 * ref.norm(), pc  # JP variant may change with the chunk
for pc, ms in res.items():
    print(json.dumps({"chunk_i": pc, "ms_best": round(min(ms), 4), "ms_all": [round(x, 4) for x in ms]}))
