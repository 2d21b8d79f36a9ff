"""First on-GPU check of eb_contract: parity vs the C oracle on small cases,
then device timing of the BASELINE configs' hot steps."""
import ctypes, json, sys, time
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import oracle
from paper_2206_08301_b200 import _capi as C

dev = torch.device("cuda:0")


def run_desc(d, out):
    L = C.lib()
    ws_bytes = L.eb_contract_workspace(ctypes.byref(d))
    ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device=dev)
    C.check(L.eb_contract(ctypes.byref(d), ctypes.c_void_p(ws.data_ptr()), ws_bytes,
                          ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return ws


def fac(t):
    return C.Factor(t.data_ptr(), t.shape[0], t.shape[1])


def mttkrp(variant, P, M, Q, L, R, X, U, pre, mid, out, mode=C.EB_REDUCE):
    d = C.ContractDesc()
    d.variant, d.mode, d.P, d.M, d.Q, d.L, d.R = variant, mode, P, M, Q, L, R
    d.X, d.U, d.ldu = X.data_ptr(), U.data_ptr(), U.shape[1]
    d.n_pre = len(pre)
    for i, f in enumerate(pre): d.pre[i] = fac(f)
    d.n_mid = len(mid)
    for i, f in enumerate(mid): d.mid[i] = fac(f)
    d.out = out.data_ptr()
    return d


def g(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


results = []
def check(name, got, want):
    e = oracle.normwise_error(got, want)
    results.append((name, e))
    print(json.dumps({"case": name, "normwise": e, "maxrel": oracle.max_rel_error(got, want)}), flush=True)

# 1. order-3 mode 0
for (I, J, K, R) in [(40, 36, 50, 24), (130, 20, 34, 32), (64, 64, 64, 64), (20, 9, 18, 70)]:
    ext = dict(i=I, j=J, k=K, a=R)
    e = "ijk,ja,ka->ia"
    X, B, Cm = oracle.seeded_inputs(e, ext, 5)
    want = oracle.naive_evaluate(e, ext, [X, B, Cm])
    out = torch.zeros(I, R, dtype=torch.float64, device=dev)
    d = mttkrp(C.EB_ROW, 1, I, J, K, R, g(X), g(Cm), [], [g(B)], out); dX=[g(X), g(Cm), g(B)]
    d = mttkrp(C.EB_ROW, 1, I, J, K, R, dX[0], dX[1], [], [dX[2]], out)
    run_desc(d, out); torch.cuda.synchronize()
    check(f"m0 {ext}", out.cpu().numpy(), want)
    # mode 1
    e = "ijk,ia,ka->ja"
    X, A, Cm = oracle.seeded_inputs(e, ext, 7)
    want = oracle.naive_evaluate(e, ext, [X, A, Cm])
    out = torch.zeros(J, R, dtype=torch.float64, device=dev)
    dX = [g(X), g(Cm), g(A)]
    d = mttkrp(C.EB_ROW, I, J, 1, K, R, dX[0], dX[1], [dX[2]], [], out)
    run_desc(d, out); torch.cuda.synchronize()
    check(f"m1 {ext}", out.cpu().numpy(), want)
    # mode 2
    e = "ijk,ia,ja->ka"
    X, A, Bm = oracle.seeded_inputs(e, ext, 9)
    want = oracle.naive_evaluate(e, ext, [X, A, Bm])
    out = torch.zeros(K, R, dtype=torch.float64, device=dev)
    dX = [g(X), g(Bm), g(A)]
    d = mttkrp(C.EB_COL, I, K, J, 0, R, dX[0], dX[1], [dX[2]], [], out)
    run_desc(d, out); torch.cuda.synchronize()
    check(f"m2 {ext}", out.cpu().numpy(), want)

# order 5 mode 0
ext = dict(i=8, j=6, k=7, l=5, m=10, a=24)
e = "ijklm,ja,ka,la,ma->ia"
X, B, Cm, D, E = oracle.seeded_inputs(e, ext, 11)
want = oracle.naive_evaluate(e, ext, [X, B, Cm, D, E])
out = torch.zeros(8, 24, dtype=torch.float64, device=dev)
dX = [g(X), g(E), g(B), g(Cm), g(D)]
d = mttkrp(C.EB_ROW, 1, 8, 6 * 7 * 5, 10, 24, dX[0], dX[1], [], dX[2:], out)
run_desc(d, out); torch.cuda.synchronize()
check("o5m0", out.cpu().numpy(), want)

# TTM batched: ijk,jb->ikb
for (I, J, K, Bn) in [(5, 40, 34, 64), (3, 70, 130, 16), (4, 33, 64, 24)]:
    ext = dict(i=I, j=J, k=K, b=Bn)
    e = "ijk,jb->ikb"
    X, U = oracle.seeded_inputs(e, ext, 13)
    want = oracle.naive_evaluate(e, ext, [X, U])
    out = torch.zeros(I, K, Bn, dtype=torch.float64, device=dev)
    dX = [g(X), g(U)]
    d = mttkrp(C.EB_COL, I, K, J, 0, Bn, dX[0], dX[1], [], [], out, mode=C.EB_BATCHED)
    run_desc(d, out); torch.cuda.synchronize()
    check(f"ttm {ext}", out.cpu().numpy(), want)

bad = [r for r in results if not (r[1] <= 1e-12)]
print(json.dumps({"parity_cases": len(results), "failed": bad}), flush=True)


def timeit(name, d, flops, bytes_, reps=10):
    L = C.lib()
    ws_bytes = L.eb_contract_workspace(ctypes.byref(d))
    ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device=dev)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for _ in range(3):
        C.check(L.eb_contract(ctypes.byref(d), ctypes.c_void_p(ws.data_ptr()), ws_bytes, st))
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        C.check(L.eb_contract(ctypes.byref(d), ctypes.c_void_p(ws.data_ptr()), ws_bytes, st))
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"time": name, "ms": round(ms, 4), "tflops": round(flops / ms / 1e9, 2),
                      "gbs": round(bytes_ / ms / 1e6, 1), "frac_fp64_37.1": round(flops / ms / 1e9 / 37.1, 3)}), flush=True)

torch.manual_seed(0)
# C1
X = torch.rand(512, 512, 512, dtype=torch.float64, device=dev) * 2 - 1
B = torch.rand(512, 24, dtype=torch.float64, device=dev); Cm = torch.rand(512, 24, dtype=torch.float64, device=dev)
out = torch.zeros(512, 24, dtype=torch.float64, device=dev)
timeit("C1 m0", mttkrp(C.EB_ROW, 1, 512, 512, 512, 24, X, Cm, [], [B], out), 2 * 512**3 * 24, 8 * 512**3)
del X
# C2
X = torch.rand(1024, 1024, 1024, dtype=torch.float64, device=dev) * 2 - 1
A = torch.rand(1024, 32, dtype=torch.float64, device=dev); B = torch.rand(1024, 32, dtype=torch.float64, device=dev)
Cm = torch.rand(1024, 32, dtype=torch.float64, device=dev)
out = torch.zeros(1024, 32, dtype=torch.float64, device=dev)
fl = 2 * 1024**3 * 32; by = 8 * 1024**3
timeit("C2 m0", mttkrp(C.EB_ROW, 1, 1024, 1024, 1024, 32, X, Cm, [], [B], out), fl, by, reps=5)
timeit("C2 m1", mttkrp(C.EB_ROW, 1024, 1024, 1, 1024, 32, X, Cm, [A], [], out), fl, by, reps=5)
timeit("C2 m2", mttkrp(C.EB_COL, 1024, 1024, 1024, 0, 32, X, B, [A], [], out), fl, by, reps=5)
U1 = torch.rand(1024, 64, dtype=torch.float64, device=dev)
t0 = torch.zeros(1024, 1024, 64, dtype=torch.float64, device=dev)
timeit("C4 ttm0", mttkrp(C.EB_COL, 1024, 1024, 1024, 0, 64, X, U1, [], [], t0, mode=C.EB_BATCHED), 2 * 1024**3 * 64, by, reps=3)
del X, t0
# C3
X = torch.rand(64, 64, 64, 64, 64, dtype=torch.float64, device=dev) * 2 - 1
F = [torch.rand(64, 24, dtype=torch.float64, device=dev) for _ in range(4)]
out = torch.zeros(64, 24, dtype=torch.float64, device=dev)
timeit("C3 o5m0", mttkrp(C.EB_ROW, 1, 64, 64**3, 64, 24, X, F[3], [], F[:3], out), 2 * 64**5 * 24, 8 * 64**5, reps=5)
# C5 step 0: ijklm,jb->iklmb
U = torch.rand(64, 16, dtype=torch.float64, device=dev)
t0 = torch.zeros(64, 64**3, 16, dtype=torch.float64, device=dev)
timeit("C5 ttm0", mttkrp(C.EB_COL, 64, 64**3, 64, 0, 16, X, U, [], [], t0, mode=C.EB_BATCHED), 2 * 64**5 * 16, 8 * 64**5 + 8 * t0.numel(), reps=3)
