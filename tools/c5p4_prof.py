"""C5 at P = 4 on virtual ranks, one run with the fused redistribution and
one without (for ncu: the term-0 ttm2 kernel with and without the scatter
epilogue)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2206_08301_b200 as eb
from tests.configs import CONFIGS
from tools.push_ab import stage_c5
c = CONFIGS["C5"]; P = 4
e, ext = c["einsums"][0], c["extents"](P)
ex = eb.Executor(e, ext, P)
plan = json.loads(eb.plan_json(e, ext, P))
stage_c5(ex, ext, P, 64 * P // plan["schedule"]["terms"][0]["grid"]["i"])
for fuse in (1, 0):
    eb.set_option("fuse_redistribution", fuse)
    ex.run()
    torch.cuda.synchronize()
print("ok")
