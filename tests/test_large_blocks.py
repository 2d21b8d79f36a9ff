"""Maximum-size edge case: one rank block of more than 2^31 elements (X of
2100 x 1024 x 1024 doubles = 17.6 GB; 2100 rows also leave a ragged last row
tile).  Every 64-bit offset of the contraction, TTM, reduction and
redistribution paths is exercised past the int32 range.

The oracle's loop nest would take hours at this size, so the check is the
size-independent closed form of a rank-1 tensor X = f ∘ g ∘ h:
  MTTKRP mode 0:  out[i, a] = f_i (gᵀB)_a (hᵀC)_a   (and modes 1, 2 alike)
  TTMc:           out[i, b, c] = f_i (gᵀU1)_b (hᵀU2)_c
which restates naive_evaluate (evaluate.cpp:7-63) summed in closed form; the
tolerance is the north-star normwise 1e-12.
"""
import gc

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
I, J, K = 2100, 1024, 1024
TOL = 1e-12


@pytest.fixture(scope="module")
def rank1():
    rng = np.random.default_rng(2026)
    f, g, h = (rng.uniform(0.5, 1.5, n) for n in (I, J, K))
    X = np.empty((I, J, K))
    np.multiply(np.multiply.outer(f, g)[:, :, None], h[None, None, :], out=X)
    assert X.size > 2**31
    yield f, g, h, X
    del X
    gc.collect()


def _run(eb, e, ext, ops, P=1):
    ex = eb.Executor(e, ext, P)
    ex.stage(ops)
    ex.run()
    out = ex.gather()
    st = ex.stats()
    ex.close()
    return out, st


@pytest.mark.parametrize("mode,P", [(0, 1), (1, 1), (2, 1), (0, 2)])
def test_mttkrp_block_past_int32(eb, rank1, mode, P):
    f, g, h, X = rank1
    R = 24
    A, B, C = (oracle.random_tensor((n, R), s) for n, s in ((I, 1), (J, 2), (K, 3)))
    e = ["ijk,ja,ka->ia", "ijk,ia,ka->ja", "ijk,ia,ja->ka"][mode]
    ops = [X] + [[B, C], [A, C], [A, B]][mode]
    vec = {"i": f @ A, "j": g @ B, "k": h @ C}
    lead = {0: ("i", f), 1: ("j", g), 2: ("k", h)}[mode]
    others = [c for c in "ijk" if c != lead[0]]
    want = lead[1][:, None] * (vec[others[0]] * vec[others[1]])[None, :]
    out, st = _run(eb, e, dict(i=I, j=J, k=K, a=R), ops, P)
    assert st["generic_launches"] == 0, st
    assert oracle.normwise_error(out.reshape(want.shape), want) <= TOL


def test_ttmc_block_past_int32(eb, rank1):
    f, g, h, X = rank1
    U1, U2 = oracle.random_tensor((J, 64), 1), oracle.random_tensor((K, 32), 2)
    want = f[:, None, None] * np.multiply.outer(g @ U1, h @ U2)[None]
    out, st = _run(eb, "ijk,jb,kc->ibc", dict(i=I, j=J, k=K, b=64, c=32), [X, U1, U2])
    assert st["generic_launches"] == 0, st
    assert oracle.normwise_error(out.reshape(want.shape), want) <= TOL


@pytest.fixture(scope="module")
def rank1_o5():
    """Order 5: X = f ∘ g ∘ h ∘ u ∘ v, 130 x 64^4 = 2.18e9 elements."""
    rng = np.random.default_rng(2027)
    vs = [rng.uniform(0.5, 1.5, n) for n in (130, 64, 64, 64, 64)]
    X = np.empty((130, 64, 64, 64, 64))
    inner = np.multiply.outer(np.multiply.outer(vs[1], vs[2]), np.multiply.outer(vs[3], vs[4]))
    np.multiply(vs[0][:, None, None, None, None], inner[None], out=X)
    assert X.size > 2**31
    yield vs, X
    del X
    gc.collect()


def test_ttmc_o5_block_past_int32(eb, rank1_o5):
    """TTMc order 5 (the C5 chain: both terms on the fused TTM-pair kernel)."""
    vs, X = rank1_o5
    Us = [oracle.random_tensor((64, 16), s) for s in (1, 2, 3, 4)]
    p = [v @ U for v, U in zip(vs[1:], Us)]
    want = vs[0][:, None, None, None, None] * np.einsum("b,c,d,e->bcde", *p)[None]
    out, st = _run(eb, "ijklm,jb,kc,ld,me->ibcde",
                   dict(i=130, j=64, k=64, l=64, m=64, b=16, c=16, d=16, e=16), [X, *Us])
    assert st["generic_launches"] == 0, st
    assert oracle.normwise_error(out.reshape(want.shape), want) <= TOL


def test_mttkrp_o5_block_past_int32(eb, rank1_o5):
    """Order-5 MTTKRP mode 0 (the C3 shape: resident-factor kernel)."""
    vs, X = rank1_o5
    Us = [oracle.random_tensor((64, 24), s) for s in (1, 2, 3, 4)]
    prod = np.ones(24)
    for v, U in zip(vs[1:], Us):
        prod *= v @ U
    want = vs[0][:, None] * prod[None, :]
    out, st = _run(eb, "ijklm,ja,ka,la,ma->ia",
                   dict(i=130, j=64, k=64, l=64, m=64, a=24), [X, *Us])
    assert st["generic_launches"] == 0, st
    assert oracle.normwise_error(out.reshape(want.shape), want) <= TOL
