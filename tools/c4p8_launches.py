import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, numpy as np
import paper_2206_08301_b200 as eb
from tests.configs import CONFIGS
from tools.push_ab import stage_c4
P = int(sys.argv[1]); c = CONFIGS["C4"]; e, ext = c["einsums"][0], c["extents"](P)
ex = eb.Executor(e, ext, P); stage_c4(ex, ext)
for _ in range(3): ex.run()
torch.cuda.synchronize(); print("ok")
