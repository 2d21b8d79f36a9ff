import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2206_08301_b200 as eb
from tests.configs import CONFIGS
from tools.push_ab import stage_c5
c = CONFIGS["C5"]; P = 4
e, ext = c["einsums"][0], c["extents"](P)
ex = eb.Executor(e, ext, P)
plan = json.loads(eb.plan_json(e, ext, P))
stage_c5(ex, ext, P, 64 * P // plan["schedule"]["terms"][0]["grid"]["i"])
outs = {}
for tag, fuse in (("f1", 1), ("s1", 0), ("f2", 1), ("s2", 0)):
    eb.set_option("fuse_redistribution", fuse)
    ex.run(); outs[tag] = ex.gather().copy()
for a, b in (("f1", "f2"), ("s1", "s2"), ("f1", "s1")):
    d = np.abs(outs[a] - outs[b]); i = int(d.argmax())
    print(a, b, "equal" if np.array_equal(outs[a], outs[b]) else f"maxdiff {d.max():.3e} at {i} ndiff {int((d>0).sum())} rel {np.linalg.norm(outs[a]-outs[b])/np.linalg.norm(outs[b]):.3e}")
