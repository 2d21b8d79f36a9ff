"""CUDA-graph replay of an executor run (eb_exec_capture / eb_exec_replay):
bitwise the eager run's output on every schedule shape the executor has —
fused MTTKRP with device group sums (async reduce on a side stream), the
resident-factor kernel, TTM terms with the fused redistribution push, TTM
pairs, GEMM chains with box-copy redistributions — across repeated replays
and after re-staging new inputs; the peer transport refuses to be captured.
"""
import uuid

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

CASES = [
    ("ijk,ja,ka->ia", dict(i=96, j=64, k=80, a=24), 1),
    ("ijk,ja,ka->ia", dict(i=96, j=64, k=80, a=24), 4),
    ("ijk,ia,ja->ka", dict(i=64, j=48, k=136, a=16), 8),
    ("ijklm,ja,ka,la,ma->ia", dict(i=16, j=8, k=8, l=8, m=64, a=24), 2),
    ("ijk,jb,kc->ibc", dict(i=96, j=96, k=96, b=24, c=24), 4),
    ("ijklm,jb,kc,ld,me->ibcde", dict(i=16, j=16, k=16, l=16, m=16, b=12, c=12, d=12, e=12), 2),
    ("ij,jk,kl->il", dict(i=64, j=48, k=40, l=32), 4),
]


def _eager(eb, e, ext, P, ops):
    ex = eb.Executor(e, ext, P)
    ex.stage(ops)
    ex.run()
    out = ex.gather()
    st = ex.stats()
    ex.close()
    return out, st


@pytest.mark.parametrize("e,ext,P", CASES, ids=[f"{c[0]}-P{c[2]}" for c in CASES])
def test_replay_matches_eager(eb, e, ext, P):
    import torch
    ops = oracle.seeded_inputs(e, ext, 5)
    want, want_st = _eager(eb, e, ext, P, ops)
    st = torch.cuda.Stream()
    ex = eb.Executor(e, ext, P, stream=st.cuda_stream)
    ex.set_async_reduce(True)
    ex.stage(ops)
    ex.capture()
    n0 = eb.launch_count()
    for _ in range(3):
        ex.replay()
        assert np.array_equal(ex.gather(), want)
    assert eb.launch_count() > n0  # replays count their captured launches
    got_st = ex.stats()
    for k in ("allreduce_volume", "redistribute_volume", "fused_launches", "generic_launches"):
        assert got_st[k] == want_st[k], (k, got_st, want_st)
    # new inputs into the same device blocks: the graph computes on them
    ops2 = oracle.seeded_inputs(e, ext, 6)
    want2, _ = _eager(eb, e, ext, P, ops2)
    ex.stage(ops2)
    ex.replay()
    assert np.array_equal(ex.gather(), want2)
    if np.prod(list(ext.values()), dtype=float) < 1e9:  # the n-ary loop finishes in seconds
        assert oracle.normwise_error(want2, oracle.naive_evaluate(e, ext, ops2).ravel()) <= 1e-12
    ex.close()


def test_peer_transport_is_not_captured(eb):
    import torch
    e, ext = "ijk,ja,ka->ia", dict(i=32, j=16, k=16, a=8)
    st = torch.cuda.Stream()
    ex = eb.Executor(e, ext, 1, rank=0, transport="peer", group=f"/eb_g{uuid.uuid4().hex[:12]}",
                     stream=st.cuda_stream)
    ex.stage(oracle.seeded_inputs(e, ext, 1))
    with pytest.raises(eb.EinplanError, match="peer transport"):
        ex.capture()
    with pytest.raises(eb.EinplanError, match="no captured run"):
        ex.replay()
    ex.close()
