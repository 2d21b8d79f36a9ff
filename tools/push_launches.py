"""One run of C4 (P=2) with the fused and with the separate redistribution,
for an ncu launch list (which kernel carries the cost)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2206_08301_b200 as eb
from tests.configs import CONFIGS
from tools.push_ab import stage_c4
c = CONFIGS["C4"]
P = int(sys.argv[1]) if len(sys.argv) > 1 else 2
e, ext = c["einsums"][0], c["extents"](P)
ex = eb.Executor(e, ext, P)
stage_c4(ex, ext)
for fuse in (1, 0):
    eb.set_option("fuse_redistribution", fuse)
    ex.run()
    torch.cuda.synchronize()
print("done")
