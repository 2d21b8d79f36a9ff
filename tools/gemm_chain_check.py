"""Table-III GEMM chains through the executor: which kernels
run and how fast (P = 1, full 4096 extents)."""
import json, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2206_08301_b200 as eb
import oracle
for name, e, ext in [("1MM", "ij,jk->ik", dict(i=4096, j=4096, k=4096)),
                     ("2MM", "ij,jk,kl->il", dict(i=4096, j=4096, k=4096, l=4096)),
                     ("3MM", "ij,jk,kl,lm->im", dict(i=4096, j=4096, k=4096, l=4096, m=4096))]:
    ins, _ = oracle.parse(e)
    ops = [eb.random_tensor(tuple(ext[c] for c in t), k) for k, t in enumerate(ins)]
    ex = eb.Executor(e, ext, 1)
    ex.stage(ops)
    ex.run(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3): ex.run()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 3 * 1e3
    st = ex.stats()
    out = ex.gather()
    # spot-check one output row against numpy (float64)
    ref_row = ops[0][5:6]
    for o in ops[1:]:
        ref_row = ref_row @ o
    err = np.linalg.norm(out.reshape(4096, 4096)[5] - ref_row[0]) / np.linalg.norm(ref_row[0])
    print(json.dumps({"kernel": name, "ms": round(ms, 2), "tflops": round(st["tree_flops"] / ms / 1e9, 2),
                      "row_err": err, **{k: st[k] for k in ("fused_launches", "ttm_launches", "generic_launches")}}), flush=True)
