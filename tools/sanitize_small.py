"""Small end-to-end exercise of every kernel, for compute-sanitizer runs
(memcheck / racecheck / synccheck, one tool per call):
fused MTTKRP ROW/COL (REDUCE, OS = 1/2), the resident-factor MTTKRP, the
dimension-tree pair, CP-ALS, TTM (BATCHED), the fused TTM pair (eb_ttm2),
the GEMM mode, generic steps, group sums, redistribution boxes (vectorised
and scalar) at P = 1, 2, 4, and the peer transport between rank threads
(einplan_run_json with EINPLAN_DEVICES=0,0,...)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2206_08301_b200 as eb  # noqa: E402

cases = [
    ("ijk,ja,ka->ia", dict(i=24, j=20, k=18, a=8), (1, 4)),
    ("ijk,ia,ka->ja", dict(i=130, j=132, k=18, a=8), (1, 2)),
    ("ijk,ia,ja->ka", dict(i=12, j=10, k=136, a=24), (1, 4)),
    ("ijklm,ja,ka,la,ma->ia", dict(i=8, j=4, k=4, l=4, m=6, a=6), (1, 2)),
    ("ijklm,ja,ka,la,ma->ia", dict(i=8, j=4, k=4, l=8, m=16, a=6), (1, 2)),  # resident factor
    ("ijk,jb,kc->ibc", dict(i=8, j=8, k=8, b=3, c=3), (1, 2)),
    ("ijk,jb,kc->ibc", dict(i=96, j=96, k=96, b=24, c=24), (2, 4)),  # redistribution boxes
    ("ijklm,jb,kc,ld,me->ibcde", dict(i=16, j=16, k=16, l=16, m=16, b=12, c=12, d=12, e=12),
     (1, 4)),  # eb_ttm2
    ("ij,jk,kl->il", dict(i=12, j=10, k=8, l=6), (1, 4)),
    ("ij,jk->ik", dict(i=256, j=64, k=200), (1,)),  # GEMM mode (forced below)
]
eb.set_option("gemm", 1)
worst = 0.0
for e, ext, Ps in cases:
    ops = oracle.seeded_inputs(e, ext, 9)
    want = oracle.naive_evaluate(e, ext, ops)
    for P in Ps:
        fm = 16.0 if e == "ijk,jb,kc->ibc" and ext["i"] == 8 else 1024.0
        ex = eb.Executor(e, ext, P, fm)
        ex.stage(ops)
        ex.run()
        got = ex.gather().reshape(want.shape)
        worst = max(worst, oracle.normwise_error(got, want))
        ex.close()
eb.set_option("gemm", 0)

# dimension-tree pair and one CP-ALS sweep
import torch  # noqa: E402
ext = dict(i=160, j=24, k=34, a=8)
X = oracle.random_tensor((160, 24, 34), 0)
F = {c: oracle.random_tensor((ext[c], 8), s) for c, s in (("i", 1), ("j", 2), ("k", 3))}
m0 = eb.Executor("ijk,ja,ka->ia", ext, 1)
m0.stage([X, F["j"], F["k"]])
m1 = eb.Executor("ijk,ia,ka->ja", ext, like=m0)
m1.share_input(0, m0, 0)
m1.share_input(2, m0, 2)
m1.stage([None, F["i"], None])
assert m0.run_pair(m1)
worst = max(worst, oracle.normwise_error(m0.gather().reshape(160, 8),
                                         oracle.naive_evaluate("ijk,ja,ka->ia", ext,
                                                               [X, F["j"], F["k"]])))
Xd = torch.from_numpy(X).cuda()
A, B, C = (torch.from_numpy(F[c]).cuda() for c in "ijk")
eb.cp3_als_sweep(Xd, A, B, C)
torch.cuda.synchronize()
assert bool(torch.isfinite(A).all())

# the peer transport between rank threads on one GPU
os.environ["EINPLAN_DEVICES"] = "0,0,0,0"
os.environ["EINPLAN_MAX_POINTS"] = "1000000000"
st, rep = eb.Session("ijk,jb,kc->ibc", dict(i=96, j=96, k=96, b=24, c=24)).run_json(4, seed=2)
del os.environ["EINPLAN_DEVICES"]
r = json.loads(rep)
assert st == 0 and r["execution"]["transport"] == "peer", r.get("execution")
assert r["verification"]["pass"]
print("worst normwise", worst)
assert worst < 1e-12
print("SANITIZE_SMALL_OK")
