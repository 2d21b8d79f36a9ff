"""Where the C1 bench step's time goes beyond the kernels: CUDA-event time of
K back-to-back executor runs (C1, P = 1) with and without join(), async
reduce, the NVML clock-sampler thread and graph replay.

    python tools/c1_step_gap.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2206_08301_b200 as eb  # noqa: E402

e, ext = "ijk,ja,ka->ia", dict(i=512, j=512, k=512, a=24)
st = torch.cuda.Stream()
ex = eb.Executor(e, ext, 1, stream=st.cuda_stream)
ex.stage([eb.random_tensor((512, 512, 512), 0), eb.random_tensor((512, 24), 1),
          eb.random_tensor((512, 24), 2)])


def timed(fn, k):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(k):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k * 1e3


def run_join():
    ex.run()
    ex.join()


def run_replay():
    ex.replay()


res = {}
plain = eb.Executor(e, ext, 1, stream=st.cuda_stream)
plain.stage([eb.random_tensor((512, 512, 512), 0), eb.random_tensor((512, 24), 1),
             eb.random_tensor((512, 24), 2)])
ex.capture()
# interleaved rounds (the GPU warms up over the script: no variant gets the cold GPU)
for rnd in range(4):
    for name, fn in (("run", plain.run), ("replay", run_replay)):
        res.setdefault(name, []).append(round(timed(fn, 50), 2))
    cs = bench.ClockSampler(0)
    cs.start()
    res.setdefault("run_with_sampler", []).append(round(timed(plain.run, 50), 2))
    c = cs.stop()
    res.setdefault("sampler_mhz", []).append(c.get("sm_mhz"))
    res.setdefault("reasons", []).append(c.get("reasons"))
print(json.dumps(res))
