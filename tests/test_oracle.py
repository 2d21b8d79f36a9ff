"""The CPU oracle (oracle/oracle.c) pinned against the reference itself
(oracle/_ref, compiled from /root/reference) and against committed golden
vectors produced by the reference (tests/golden, tools/make_golden.py)."""
import json
import os

import numpy as np
import pytest

import oracle
from tests.configs import CONFIGS

GOLD = os.path.join(os.path.dirname(__file__), "golden")
needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")

DESK = [  # acceptance.cpp:111-133 (desk-scale Table-III kernels)
    ("1MM", "ij,jk->ik", dict(i=63, j=64, k=61)),
    ("2MM", "ij,jk,kl->il", dict(i=40, j=40, k=40, l=40)),
    ("3MM", "ij,jk,kl,lm->im", dict(i=32, j=32, k=32, l=32, m=32)),
    ("MTTKRP-O3-M0", "ijk,ja,ka->ia", dict(i=22, j=24, k=23, a=12)),
    ("MTTKRP-O3-M1", "ijk,ia,ka->ja", dict(i=24, j=24, k=24, a=16)),
    ("MTTKRP-O3-M2", "ijk,ia,ja->ka", dict(i=24, j=22, k=24, a=16)),
    ("MTTKRP-O5-M0", "ijklm,ja,ka,la,ma->ia", dict(i=8, j=8, k=8, l=8, m=8, a=6)),
    ("MTTKRP-O5-M2", "ijklm,ia,ja,la,ma->ka", dict(i=7, j=8, k=8, l=7, m=8, a=5)),
    ("MTTKRP-O5-M4", "ijklm,ia,ja,ka,la->ma", dict(i=8, j=8, k=8, l=8, m=8, a=6)),
    ("TTMc-O5-M0", "ijklm,jb,kc,ld,me->ibcde",
     dict(i=8, j=8, k=8, l=8, m=8, b=6, c=6, d=6, e=6)),
]


def test_mt19937_64_known_answer():
    # The C++ standard pins mt19937_64 with default seed 5489: the 10000th
    # output is 9981545732273789042.  random_tensor maps (x >> 11) * 2^-53.
    v = oracle.random_tensor((10000,), 5489)
    x = 9981545732273789042
    assert v[-1] == 2.0 * ((x >> 11) * 2.0 ** -53) - 1.0


def test_random_stream_skip_matches_prefix():
    a = oracle.random_tensor((5000,), 7)
    b = oracle.random_tensor((1000,), 7, skip=4000)
    assert np.array_equal(a[4000:], b)


@needs_ref
@pytest.mark.parametrize("seed", [0, 1, 42, 2**40 + 3])
def test_random_tensor_matches_reference(seed):
    a = oracle.random_tensor((4096,), seed)
    b = np.empty(4096)
    oracle.ref().ref_random_fill(oracle._ptr(b), 4096, seed)
    assert np.array_equal(a, b)


@needs_ref
@pytest.mark.parametrize("name,einsum,ext", DESK, ids=[d[0] for d in DESK])
def test_naive_evaluate_bitwise_matches_reference(name, einsum, ext):
    ops = oracle.seeded_inputs(einsum, ext, 1000)
    assert np.array_equal(oracle.naive_evaluate(einsum, ext, ops),
                          oracle.ref_naive_evaluate(einsum, ext, ops))


@needs_ref
@pytest.mark.parametrize("name,einsum,ext", DESK, ids=[d[0] for d in DESK])
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_reference_run_agrees_with_oracle(name, einsum, ext, P):
    # acceptance.cpp:347-361: every kernel at P in {1,2,4,8} within 1e-10.
    ops = oracle.seeded_inputs(einsum, ext, 1000)
    want = oracle.naive_evaluate(einsum, ext, ops)
    got, _, _ = oracle.ref_run(einsum, ext, P, ops)
    assert oracle.max_rel_error(got, want) <= 1e-10


def test_allreduce_known_answer():
    # test_executor.cpp:69-94: [1,2,3,4] + [10,20,30,40] = [11,22,33,44]
    acc = oracle.group_sum([np.array([1.0, 2, 3, 4]), np.array([10.0, 20, 30, 40])])
    assert acc.tolist() == [11, 22, 33, 44]


def test_mttkrp_is_krp_then_contract():
    # test_einsum.cpp:150-166: MTTKRP == KRP followed by the contraction.
    ext = dict(i=5, j=6, k=7, a=3)
    X, B, C = oracle.seeded_inputs("ijk,ja,ka->ia", ext, 3)
    krp = oracle.naive_evaluate("ja,ka->jka", dict(j=6, k=7, a=3), [B, C])
    two = oracle.naive_evaluate("ijk,jka->ia", ext, [X, krp])
    one = oracle.naive_evaluate("ijk,ja,ka->ia", ext, [X, B, C])
    assert oracle.normwise_error(two, one) < 1e-14


def test_golden_small_outputs_pin_oracle():
    """Reference outputs of C1 / C3 (full BASELINE sizes) are committed; the
    oracle must reproduce a C1 row exactly as the reference computed it."""
    path = os.path.join(GOLD, "C1_out.npy")
    if not os.path.exists(path):
        pytest.skip("golden C1 output not generated yet")
    gold = np.load(path)
    ext = CONFIGS["C1"]["extents"](1)
    # Row i of out for a few i, via the oracle on the i-slice of X.
    X = oracle.random_tensor((512, 512, 512), 0)
    B = oracle.random_tensor((512, 24), 1)
    C = oracle.random_tensor((512, 24), 2)
    for i in (0, 311):
        row = oracle.naive_evaluate("jk,ja,ka->a", dict(j=512, k=512, a=24),
                                    [np.ascontiguousarray(X[i]), B, C])
        assert oracle.normwise_error(row, gold[i]) < 1e-13
    assert gold.shape == (512, 24)
    meta = json.load(open(os.path.join(GOLD, "reference_runs.json")))
    assert meta["C1"]["extents"] == ext
