import sys, time, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import torch
import paper_2206_08301_b200 as eb
from scaling_proxy import stage
from tests.configs import CONFIGS
for cfg, P in (("C1", 1), ("C1", 8), ("C5", 1), ("C3", 1)):
    c = CONFIGS[cfg]; ext = c["extents"](P)
    st = torch.cuda.Stream()
    ex = eb.Executor(c["einsums"][0], ext, P, stream=st.cuda_stream)
    stage(ex, cfg, c["einsums"][0], ext, P)
    for _ in range(3): ex.run()
    torch.cuda.synchronize()
    n = 50
    t0 = time.perf_counter()
    for _ in range(n): ex.run()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(cfg, P, "host us/run %.1f" % ((t1 - t0) / n * 1e6), "wall us/run %.1f" % ((t2 - t0) / n * 1e6))
    ex.close()
