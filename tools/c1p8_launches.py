import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2206_08301_b200 as eb
import oracle
from tests.configs import CONFIGS
P = int(sys.argv[1]); c = CONFIGS["C1"]; e, ext = c["einsums"][0], c["extents"](P)
ex = eb.Executor(e, ext, P); ex.stage(oracle.seeded_inputs(e, ext, 0))
for _ in range(3): ex.run()
torch.cuda.synchronize(); print("ok")
