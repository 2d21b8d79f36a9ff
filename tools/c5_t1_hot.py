"""C5 term 1 (eb_ttm2 on t1) timed right after term 0 wrote t1 (L2-hot) and
after an L2 flush (cold), for i-chunks of t1: the bound on what keeping t1
in L2 could save.  usage: python tools/c5_t1_hot.py CHUNK_I"""
import ctypes, os, sys, json, torch
sys.path.insert(0, "/root/repo")
from paper_2206_08301_b200 import _capi as C
L = C.lib(); st = torch.cuda.current_stream(); s = ctypes.c_void_p(st.cuda_stream)
n = 64; pc = int(sys.argv[1]) if len(sys.argv) > 1 else 8
X = torch.rand(pc, n, n, n, n, dtype=torch.float64, device="cuda")
U = [torch.rand(n, 16, dtype=torch.float64, device="cuda") for _ in range(4)]
t1 = torch.empty(pc, n, n, 16, 16, dtype=torch.float64, device="cuda")
out = torch.empty(pc, 16, 16, 16, 16, dtype=torch.float64, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
d0 = C.Ttm2Desc(pc, n, n, n * n, 16, 16, X.data_ptr(), U[0].data_ptr(), 16, U[1].data_ptr(), 16, t1.data_ptr())
d1 = C.Ttm2Desc(pc, n, n, 256, 16, 16, t1.data_ptr(), U[2].data_ptr(), 16, U[3].data_ptr(), 16, out.data_ptr())
def ev(): return torch.cuda.Event(enable_timing=True)
res = {"hot": [], "cold": []}
for _ in range(5):
    C.check(L.eb_ttm2(ctypes.byref(d0), s))
    a, b = ev(), ev(); a.record(st); C.check(L.eb_ttm2(ctypes.byref(d1), s)); b.record(st)
    torch.cuda.synchronize(); res["hot"].append(a.elapsed_time(b))
    flush.zero_(); torch.cuda.synchronize()
    a, b = ev(), ev(); a.record(st); C.check(L.eb_ttm2(ctypes.byref(d1), s)); b.record(st)
    torch.cuda.synchronize(); res["cold"].append(a.elapsed_time(b))
print(json.dumps({"chunk_i": pc, "t1_MB": t1.numel() * 8 / 1e6, "term1_hot_ms": min(res["hot"]), "term1_cold_ms": min(res["cold"])}))
