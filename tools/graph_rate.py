"""Host time and device wall time per run, eager execute() vs the captured
CUDA graph (eb_exec_replay), for launch-heavy schedules: C1 at P = 1 and 8
virtual ranks, a 96^3 TTMc at P = 4, a 64^3 MTTKRP at P = 8.

    python tools/graph_rate.py [out.jsonl]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2206_08301_b200 as eb  # noqa: E402

CASES = [("C1", "ijk,ja,ka->ia", dict(i=512, j=512, k=512, a=24), 1),
         ("C1", "ijk,ja,ka->ia", dict(i=512, j=512, k=512, a=24), 8),
         ("ttmc96", "ijk,jb,kc->ibc", dict(i=96, j=96, k=96, b=24, c=24), 4),
         ("mttkrp64", "ijk,ja,ka->ia", dict(i=64, j=64, k=64, a=16), 8)]


def rate(fn, st, n=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return (t1 - t0) / n * 1e6, (t2 - t0) / n * 1e6


out = []
for name, e, ext, P in CASES:
    st = torch.cuda.Stream()
    ex = eb.Executor(e, ext, P, stream=st.cuda_stream)
    ex.stage(oracle.seeded_inputs(e, ext, 0) if name != "C1" else
             [eb.random_tensor((512, 512, 512), 0), eb.random_tensor((512, 24), 1),
              eb.random_tensor((512, 24), 2)])
    h_e, w_e = rate(ex.run, st)
    a = ex.gather()
    ex.capture()
    h_g, w_g = rate(ex.replay, st)
    assert (ex.gather() == a).all()
    line = {"case": name, "P": P, "eager_host_us": round(h_e, 1), "eager_wall_us": round(w_e, 1),
            "graph_host_us": round(h_g, 1), "graph_wall_us": round(w_g, 1)}
    print(json.dumps(line), flush=True)
    out.append(line)
    ex.close()
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        for l in out:
            f.write(json.dumps(l) + "\n")
