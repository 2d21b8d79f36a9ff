import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2206_08301_b200 as eb
from tests.configs import CONFIGS
from tools.push_ab import stage_c5
c = CONFIGS["C5"]; P = 4
e, ext = c["einsums"][0], c["extents"](P)
st = torch.cuda.Stream()
ex = eb.Executor(e, ext, P, stream=st.cuda_stream)
plan = json.loads(eb.plan_json(e, ext, P))
stage_c5(ex, ext, P, 64 * P // plan["schedule"]["terms"][0]["grid"]["i"])
ref = {}
for fuse in (0, 1):
    eb.set_option("fuse_redistribution", fuse)
    ex.run(); torch.cuda.synchronize(); ref[fuse] = ex.gather().copy()
print("ref equal", np.array_equal(ref[0], ref[1]))
for rnd in range(int(os.environ.get('ROUNDS', '4'))):
    for fuse in (0, 1):
        eb.set_option("fuse_redistribution", fuse)
        for _ in range(7): ex.run()
        out = ex.gather()
        bad = not np.array_equal(out, ref[fuse])
        if bad:
            d = np.abs(out - ref[fuse]); print("round", rnd, "fuse", fuse, "DIFF ndiff", int((d > 0).sum()), "max", d.max(), "first", int(np.argmax(d > 0)))
        else:
            print("round", rnd, "fuse", fuse, "ok")
