"""Run CP-ALS sweeps on a random order-3 tensor (for ncu launch lists / timing)."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2206_08301_b200 as eb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
R = int(sys.argv[2]) if len(sys.argv) > 2 else 32
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
X = torch.rand(n, n, n, dtype=torch.float64, device="cuda") * 2 - 1
A, B, C = (torch.rand(n, R, dtype=torch.float64, device="cuda") * 2 - 1 for _ in range(3))
ws = eb.cp3_als_sweep(X, A, B, C)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    eb.cp3_als_sweep(X, A, B, C, workspace=ws)
e1.record()
torch.cuda.synchronize()
print("ms per sweep", e0.elapsed_time(e1) / reps)
