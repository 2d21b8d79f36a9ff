import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import oracle
import paper_2206_08301_b200 as eb
CASES = {"c5": ("ijklm,jb,kc,ld,me->ibcde", dict(i=128, j=32, k=32, l=32, m=32, b=16, c=16, d=16, e=16), 4),
         "c4": ("ijk,jb,kc->ibc", dict(i=256, j=256, k=256, b=64, c=64), 8),
         "c5b": ("ijklm,jb,kc,ld,me->ibcde", dict(i=256, j=32, k=32, l=32, m=32, b=16, c=16, d=16, e=16), 4)}
e, ext, P = CASES[os.environ.get("CASE", "c5")]
ops = oracle.seeded_inputs(e, ext, 81)
for fuse in (int(os.environ.get("FUSE", "1")),):
    eb.set_option("fuse_redistribution", fuse)
    ex = eb.Executor(e, ext, P)
    ex.stage(ops)
    ex.run(); torch.cuda.synchronize(); ref = ex.gather().copy()
    nbad = 0
    for rnd in range(int(os.environ.get("ROUNDS", "20"))):
        for _ in range(5): ex.run()
        out = ex.gather()
        if not np.array_equal(out, ref):
            nbad += 1
            d = np.nonzero(out.reshape(ext["i"], -1) != ref.reshape(ext["i"], -1))
            ii = np.unique(d[0])
            print("fuse", fuse, "round", rnd, "ndiff", len(d[0]), "i values", ii[:10])
            o = out.reshape(ext["i"], -1); rf = ref.reshape(ext["i"], -1)
            for i in ii[:2]:
                w = o[i]
                print("  wrong norm", np.linalg.norm(w), "ref norm", np.linalg.norm(rf[i]), "ratio", np.linalg.norm(w) / np.linalg.norm(rf[i]))
                dists = [np.linalg.norm(w - rf[j]) / np.linalg.norm(rf[j]) for j in range(ext["i"])]
                print("  closest ref row", int(np.argmin(dists)), min(dists), "diff-to-ref2", dists[i])
    print("fuse", fuse, "bad rounds", nbad)
