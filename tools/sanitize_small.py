"""Small end-to-end exercise of every kernel (for compute-sanitizer runs):
fused MTTKRP ROW/COL (REDUCE, OS=1/2), the resident-factor MTTKRP, TTM (BATCHED), generic steps, group
sums and redistribution boxes at P=1,2,4."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import oracle
import paper_2206_08301_b200 as eb

cases = [
    ("ijk,ja,ka->ia", dict(i=24, j=20, k=18, a=8), (1, 4)),
    ("ijk,ia,ka->ja", dict(i=130, j=132, k=18, a=8), (1, 2)),
    ("ijk,ia,ja->ka", dict(i=12, j=10, k=136, a=24), (1, 4)),
    ("ijklm,ja,ka,la,ma->ia", dict(i=8, j=4, k=4, l=4, m=6, a=6), (1, 2)),
    ("ijklm,ja,ka,la,ma->ia", dict(i=8, j=4, k=4, l=8, m=16, a=6), (1, 2)),  # resident factor
    ("ijk,jb,kc->ibc", dict(i=8, j=8, k=8, b=3, c=3), (1, 2)),
    ("ij,jk,kl->il", dict(i=12, j=10, k=8, l=6), (1, 4)),
]
worst = 0.0
for e, ext, Ps in cases:
    ops = oracle.seeded_inputs(e, ext, 9)
    want = oracle.naive_evaluate(e, ext, ops)
    for P in Ps:
        fm = 16.0 if e.startswith("ijk,jb") else 1024.0
        ex = eb.Executor(e, ext, P, fm)
        ex.stage(ops)
        ex.run()
        got = ex.gather().reshape(want.shape)
        worst = max(worst, oracle.normwise_error(got, want))
print("worst normwise", worst)
assert worst < 1e-12
