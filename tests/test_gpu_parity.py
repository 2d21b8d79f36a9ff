"""GPU parity of the CUDA path against the CPU oracle / reference goldens.

Every comparison here runs the product path (libeinplan_b200.so: DMMA/TMA
kernels, device reductions and redistributions) and checks it against the
oracle (oracle/oracle.c) or against outputs the reference itself produced
(tests/golden, tools/make_golden.py).  Tolerance: <= 1e-12 normwise
(||got - want||_2 / ||want||_2), the north-star bound; the reference's own
elementwise metric (max |d| / max(1,|want|)) is additionally held to 1e-10
as in acceptance.cpp:347-361.
"""
import ctypes
import json
import os

import numpy as np
import pytest

import oracle
from tests.configs import CONFIGS, c2_inputs, seeded
from tests.test_oracle import DESK

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL = 1e-12


def _torch():
    import torch
    return torch


def check(got, want, tol=TOL):
    got = np.asarray(got).reshape(np.shape(want))
    nw = oracle.normwise_error(got, want)
    mr = oracle.max_rel_error(got, want)
    assert nw <= tol and mr <= 1e-10, (nw, mr)


# ------------------------------------------------------------------ kernel --

def _contract(eb, variant, mode, P, M, Q, L, R, X, U, pre, mid, out):
    from paper_2206_08301_b200 import _capi as C
    torch = _torch()
    d = C.ContractDesc()
    d.variant, d.mode, d.P, d.M, d.Q, d.L, d.R = variant, mode, P, M, Q, L, R
    d.X, d.U, d.ldu = X.data_ptr(), U.data_ptr(), U.shape[1]
    d.n_pre = len(pre)
    for i, f in enumerate(pre):
        d.pre[i] = C.Factor(f.data_ptr(), f.shape[0], f.shape[1])
    d.n_mid = len(mid)
    for i, f in enumerate(mid):
        d.mid[i] = C.Factor(f.data_ptr(), f.shape[0], f.shape[1])
    d.out = out.data_ptr()
    L_ = C.lib()
    wb = L_.eb_contract_workspace(ctypes.byref(d))
    assert wb > 0, L_.eb_last_error()
    ws = torch.empty(wb, dtype=torch.uint8, device="cuda")
    C.check(L_.eb_contract(ctypes.byref(d), ctypes.c_void_p(ws.data_ptr()), wb,
                           ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    return out.cpu().numpy()


SHAPES3 = [(40, 36, 50, 24), (130, 20, 34, 32), (64, 64, 64, 64), (20, 9, 18, 70), (257, 3, 6, 8),
           (8, 200, 2, 1), (1, 1, 2, 3)]


@pytest.mark.parametrize("I,J,K,R", SHAPES3)
@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("fused_tma", [True, False])
def test_contract_mttkrp_order3(eb, I, J, K, R, mode, fused_tma, opts):
    from paper_2206_08301_b200 import _capi as C
    torch = _torch()
    if not fused_tma:  # one TMA box per 16-wide block instead of one per operand
        opts("no_fused_tma", 1)
    ext = dict(i=I, j=J, k=K, a=R)
    e = ["ijk,ja,ka->ia", "ijk,ia,ka->ja", "ijk,ia,ja->ka"][mode]
    ops = oracle.seeded_inputs(e, ext, 17 + mode)
    want = oracle.naive_evaluate(e, ext, ops)
    g = [torch.from_numpy(o).cuda() for o in ops]
    if mode == 2 and K % 2:
        pytest.skip("COL variant needs an even contiguous extent (executor uses the generic path)")
    if mode < 2 and K % 2:
        pytest.skip("ROW variant needs an even contiguous extent")
    out = torch.zeros(want.shape, dtype=torch.float64, device="cuda")
    if mode == 0:
        got = _contract(eb, C.EB_ROW, C.EB_REDUCE, 1, I, J, K, R, g[0], g[2], [], [g[1]], out)
    elif mode == 1:
        got = _contract(eb, C.EB_ROW, C.EB_REDUCE, I, J, 1, K, R, g[0], g[2], [g[1]], [], out)
    else:
        got = _contract(eb, C.EB_COL, C.EB_REDUCE, I, K, J, 0, R, g[0], g[2], [g[1]], [], out)
    check(got, want)


@pytest.mark.parametrize("I,J,K,B", [(5, 40, 34, 64), (3, 70, 130, 16), (4, 33, 64, 24),
                                     (2, 9, 2, 100), (1, 256, 258, 8),
                                     # narrow M (K here): OS outer indices per tile
                                     (37, 64, 16, 64), (8, 100, 16, 24), (13, 40, 24, 16),
                                     (16, 32, 32, 64), (9, 20, 12, 8)])
@pytest.mark.parametrize("fused_tma", [True, False])
def test_contract_ttm(eb, I, J, K, B, fused_tma, opts):
    from paper_2206_08301_b200 import _capi as C
    torch = _torch()
    if not fused_tma:
        opts("no_fused_tma", 1)
    ext = dict(i=I, j=J, k=K, b=B)
    e = "ijk,jb->ikb"
    X, U = oracle.seeded_inputs(e, ext, 13)
    want = oracle.naive_evaluate(e, ext, [X, U])
    out = torch.zeros(want.shape, dtype=torch.float64, device="cuda")
    got = _contract(eb, C.EB_COL, C.EB_BATCHED, I, K, J, 0, B, torch.from_numpy(X).cuda(),
                    torch.from_numpy(U).cuda(), [], [], out)
    check(got, want)


TTM2_SHAPES = [(2, 64, 64, 64, 16, 16), (3, 40, 7, 50, 16, 16), (1, 64, 9, 18, 5, 11),
               (4, 3, 130, 2, 16, 1), (2, 33, 64, 34, 8, 16), (1, 1, 1, 2, 1, 1),
               (5, 64, 4, 16, 16, 16)]


@pytest.mark.parametrize("P,Q1,Q2,M,N1,N2", TTM2_SHAPES)
@pytest.mark.parametrize("variant", [0, 1, 2])
def test_ttm2_pair(eb, P, Q1, Q2, M, N1, N2, variant, opts):
    """eb_ttm2 = the two chained TTM steps pjkm,jb->pkmb ; pkmb,kc->pmbc of one
    term (TTMc-O5), ragged in every extent, against the oracle's n-ary loop —
    the automatic choice and each shipped warp-specialised kernel (JP = 1 / 2)
    forced with the ttm2_variant option."""
    from paper_2206_08301_b200 import _capi as C
    torch = _torch()
    opts("ttm2_variant", variant)
    e = "pjkm,jb,kc->pmbc"
    ext = dict(p=P, j=Q1, k=Q2, m=M, b=N1, c=N2)
    ops = oracle.seeded_inputs(e, ext, 23)
    want = oracle.naive_evaluate(e, ext, ops)
    X, U1, U2 = [torch.from_numpy(o).cuda() for o in ops]
    out = torch.full(want.shape, float("nan"), dtype=torch.float64, device="cuda")
    d = C.Ttm2Desc(P, Q1, Q2, M, N1, N2, X.data_ptr(), U1.data_ptr(), N1, U2.data_ptr(), N2,
                   out.data_ptr())
    C.check(C.lib().eb_ttm2(ctypes.byref(d),
                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    check(out.cpu().numpy(), want)


def test_ttm2_rejects_unsupported_shapes(eb):
    from paper_2206_08301_b200 import _capi as C
    d = C.Ttm2Desc(1, 65, 4, 16, 16, 16, 8, 8, 16, 8, 16, 8)
    assert C.lib().eb_ttm2(ctypes.byref(d), None) == 1  # EB_E_INVALID, nothing launched
    d = C.Ttm2Desc(1, 64, 4, 15, 16, 16, 8, 8, 16, 8, 16, 8)
    assert C.lib().eb_ttm2(ctypes.byref(d), None) == 1


def _ttmc_o5_chain(ext, ops):
    """The reference tree of TTMc-O5 evaluated step by step with the oracle
    (ijklm -> iklmb -> ilmbc -> imbcd -> ibcde, Appendix A of SURVEY)."""
    X, U1, U2, U3, U4 = ops
    t = oracle.naive_evaluate("ijklm,jb->iklmb", ext, [X, U1])
    t = oracle.naive_evaluate("iklmb,kc->ilmbc", ext, [t, U2])
    t = oracle.naive_evaluate("ilmbc,ld->imbcd", ext, [t, U3])
    return oracle.naive_evaluate("imbcd,me->ibcde", ext, [t, U4])


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_ttmc_o5_fused_terms(eb, P, opts):
    """Both TTMc-O5 terms ([t0,t1], [t2,out]: the C5 partition at these
    extents, with the i2m2 / i2c2 / i2l2m2 / i2b2c2 grids of P=4, 8) run on
    eb_ttm2 — two fused launches per rank — and match the oracle chain and
    the unfused two-launch path."""
    e = "ijklm,jb,kc,ld,me->ibcde"
    ext = dict(i=16 * P, j=16, k=16, l=16, m=16, b=12, c=12, d=12, e=12)
    plan = json.loads(eb.plan_json(e, ext, P))
    assert [t["output"] for t in plan["schedule"]["terms"]] == ["t1", "out"]
    ops = oracle.seeded_inputs(e, ext, 5)
    want = _ttmc_o5_chain(ext, ops)
    opts("chain_terms", 1)
    ex = eb.Executor(e, ext, P)
    ex.stage(ops)
    ex.run()
    st = ex.stats()
    # with chaining on, the two terms run as one eb_ttm2_chain launch per rank
    # where the t1 hand-over is a whole-block self message, else two
    plan_r = json.loads(eb.plan_json(e, ext, P, include_messages=True))
    selfonly = all(m["self"] for r in plan_r["schedule"]["redistributions"]
                   for m in r["plan"]["messages"])
    assert st["fused_launches"] == (P if selfonly else 2 * P) and st["ttm_launches"] == 0, st
    assert st["generic_launches"] == 0, st
    check(ex.gather(), want)
    opts("chain_terms", 0)
    ex = eb.Executor(e, ext, P)
    ex.stage(ops)
    ex.run()
    assert ex.stats()["fused_launches"] == 2 * P
    check(ex.gather(), want)
    opts("fuse_ttm2", 0)
    ex = eb.Executor(e, ext, P)
    ex.stage(ops)
    ex.run()
    assert ex.stats()["ttm_launches"] == 4 * P
    check(ex.gather(), want)


MTTKRP2_SHAPES = [(130, 20, 34, 32), (256, 64, 64, 24), (128, 9, 2, 8), (300, 40, 18, 64),
                  (257, 3, 6, 8), (128, 1, 2, 1), (512, 33, 130, 17)]


@pytest.mark.parametrize("I,J,K,R", MTTKRP2_SHAPES)
@pytest.mark.parametrize("fused_tma", [True, False])
def test_mttkrp2_dimension_tree_pair(eb, I, J, K, R, fused_tma, opts):
    """eb_mttkrp2: one pass over X gives the mode-0 and the mode-1 MTTKRP
    (T = X x_k C folded with B and with A), each equal to the oracle's own
    naive_evaluate of that mode's einsum."""
    if not fused_tma:
        opts("no_fused_tma", 1)
    from paper_2206_08301_b200 import _capi as C
    torch = _torch()
    ext = dict(i=I, j=J, k=K, a=R)
    X = oracle.random_tensor((I, J, K), 0)
    A, B, Cf = (oracle.random_tensor((n, R), s) for n, s in ((I, 1), (J, 2), (K, 3)))
    want0 = oracle.naive_evaluate("ijk,ja,ka->ia", ext, [X, B, Cf])
    want1 = oracle.naive_evaluate("ijk,ia,ka->ja", ext, [X, A, Cf])
    g = {n: torch.from_numpy(t).cuda() for n, t in (("X", X), ("A", A), ("B", B), ("C", Cf))}
    out0 = torch.full((I, R), float("nan"), dtype=torch.float64, device="cuda")
    out1 = torch.full((J, R), float("nan"), dtype=torch.float64, device="cuda")
    d = C.ContractDesc()
    d.variant, d.mode, d.P, d.M, d.Q, d.L, d.R = C.EB_ROW, C.EB_REDUCE, 1, I, J, K, R
    d.X, d.U, d.ldu = g["X"].data_ptr(), g["C"].data_ptr(), R
    d.n_mid = 1
    d.mid[0] = C.Factor(g["B"].data_ptr(), J, R)
    d.out = out0.data_ptr()
    L_ = C.lib()
    wb = L_.eb_mttkrp2_workspace(ctypes.byref(d))
    assert wb > 0, L_.eb_last_error()
    ws = torch.empty(wb, dtype=torch.uint8, device="cuda")
    C.check(L_.eb_mttkrp2(ctypes.byref(d), ctypes.c_void_p(g["A"].data_ptr()), R,
                          ctypes.c_void_p(out1.data_ptr()), ctypes.c_void_p(ws.data_ptr()), wb,
                          ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    check(out0.cpu().numpy(), want0)
    check(out1.cpu().numpy(), want1)


def test_mttkrp2_rejects_small_row_tiles(eb):
    from paper_2206_08301_b200 import _capi as C
    d = C.ContractDesc()
    d.variant, d.mode, d.P, d.M, d.Q, d.L, d.R = C.EB_ROW, C.EB_REDUCE, 1, 64, 8, 8, 8
    d.X = d.U = d.out = 8
    d.n_mid = 1
    d.mid[0] = C.Factor(8, 8, 8)
    assert C.lib().eb_mttkrp2_workspace(ctypes.byref(d)) == 0  # M < 128: not this kernel


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_exec_run_pair_cp_sweep(eb, P):
    """eb_exec_run_pair on the reference schedules of modes 0 and 1 (same grid
    at every P): fused on every rank, both outputs equal the
    oracle, and the reduction volumes equal those of two separate runs."""
    ext = dict(i=256, j=256, k=128, a=16)
    es = ["ijk,ja,ka->ia", "ijk,ia,ka->ja"]
    X = oracle.random_tensor((256, 256, 128), 0)
    F = {c: oracle.random_tensor((ext[c], 16), s) for c, s in (("i", 1), ("j", 2), ("k", 3))}
    ex0 = eb.Executor(es[0], ext, P)
    ex0.stage([X, F["j"], F["k"]])
    ex1 = eb.Executor(es[1], ext, P)
    ex1.share_input(0, ex0, 0)
    ex1.share_input(2, ex0, 2)
    ex1.stage([None, F["i"], None])
    assert ex0.run_pair(ex1)
    got0, got1 = ex0.gather(), ex1.gather()
    st0, st1 = ex0.stats(), ex1.stats()
    check(got0, oracle.naive_evaluate(es[0], ext, [X, F["j"], F["k"]]))
    check(got1, oracle.naive_evaluate(es[1], ext, [X, F["i"], F["k"]]))
    assert st0["fused_launches"] == P and st1["fused_launches"] == 0
    ex0.run()
    ex1.run()
    assert ex0.stats()["allreduce_volume"] == st0["allreduce_volume"]
    assert ex1.stats()["allreduce_volume"] == st1["allreduce_volume"]
    check(ex0.gather(), got0)
    check(ex1.gather(), got1)


@pytest.mark.parametrize("name,einsum,ext",
                         [d for d in DESK if d[0] in ("2MM", "3MM", "MTTKRP-O3-M1", "MTTKRP-O5-M0")],
                         ids=["2MM", "3MM", "MTTKRP-O3-M1", "MTTKRP-O5-M0"])
@pytest.mark.parametrize("P", [4, 8])
def test_async_reduce_matches_ordered(eb, name, einsum, ext, P):
    """Reductions on the side stream (eb_exec_set_async_reduce): a sweep of
    runs with joins must give the ordered run's output bit for bit, including
    multi-term schedules whose later terms consume a reduced output."""
    ops = oracle.seeded_inputs(einsum, ext, 9)
    ex = eb.Executor(einsum, ext, P)
    ex.stage(ops)
    ex.run()
    want = ex.gather()
    ex2 = eb.Executor(einsum, ext, P)
    ex2.stage(ops)
    ex2.set_async_reduce(True)
    for _ in range(3):
        ex2.run()
    ex2.join()
    got = ex2.gather()
    assert np.array_equal(got, want)
    assert ex2.stats()["allreduce_volume"] == ex.stats()["allreduce_volume"]


def test_exec_run_pair_falls_back_when_not_shared(eb):
    ext = dict(i=128, j=32, k=32, a=8)
    X = oracle.random_tensor((128, 32, 32), 0)
    F = {c: oracle.random_tensor((ext[c], 8), s) for c, s in (("i", 1), ("j", 2), ("k", 3))}
    ex0 = eb.Executor("ijk,ja,ka->ia", ext, 1)
    ex0.stage([X, F["j"], F["k"]])
    ex1 = eb.Executor("ijk,ia,ka->ja", ext, 1)
    ex1.stage([X, F["i"], F["k"]])  # own copy of X: not the same blocks
    assert not ex0.run_pair(ex1)
    check(ex1.gather(), oracle.naive_evaluate("ijk,ia,ka->ja", ext, [X, F["i"], F["k"]]))


def _np_als_sweep(X, A, B, C):
    """One CP-ALS sweep in numpy (float64): the textbook update order."""
    A = np.einsum("ijk,jr,kr->ir", X, B, C) @ np.linalg.inv((B.T @ B) * (C.T @ C))
    B = np.einsum("ijk,ir,kr->jr", X, A, C) @ np.linalg.inv((A.T @ A) * (C.T @ C))
    C = np.einsum("ijk,ir,jr->kr", X, A, B) @ np.linalg.inv((A.T @ A) * (B.T @ B))
    return A, B, C


@pytest.mark.parametrize("I,J,K,R", [(40, 36, 50, 8), (130, 20, 34, 16), (64, 64, 64, 32),
                                     (257, 3, 6, 4), (300, 40, 18, 24),
                                     (600, 512, 16, 8),  # T on the direct (tile-aligned) path
                                     (70, 50, 24, 64), (33, 17, 10, 1), (90, 130, 66, 13)])
def test_cp3_als_sweep(eb, I, J, K, R):
    """eb_cp3_als_sweep (dimension tree: T = X x3 C shared by modes 0 and 1,
    Gram/Hadamard/SPD-inverse updates on the device) = the numpy sweep, twice."""
    torch = _torch()
    rng = np.random.default_rng(I + J + K + R)
    X = rng.uniform(-1, 1, (I, J, K))
    F = [rng.uniform(-1, 1, (n, R)) for n in (I, J, K)]
    g = [torch.from_numpy(a.copy()).cuda() for a in [X] + F]
    ws = None
    want = F
    for _ in range(2):
        ws = eb.cp3_als_sweep(g[0], g[1], g[2], g[3], workspace=ws)
        want = _np_als_sweep(X, *want)
    torch.cuda.synchronize()
    for got, w in zip(g[1:], want):
        rel = np.linalg.norm(got.cpu().numpy() - w) / np.linalg.norm(w)
        assert rel <= 1e-9, rel


def test_contract_order5_all_krp_rows(eb):
    from paper_2206_08301_b200 import _capi as C
    torch = _torch()
    ext = dict(i=8, j=6, k=7, l=5, m=10, a=24)
    e = "ijklm,ja,ka,la,ma->ia"
    ops = oracle.seeded_inputs(e, ext, 11)
    want = oracle.naive_evaluate(e, ext, ops)
    g = [torch.from_numpy(o).cuda() for o in ops]
    out = torch.zeros(8, 24, dtype=torch.float64, device="cuda")
    got = _contract(eb, C.EB_ROW, C.EB_REDUCE, 1, 8, 6 * 7 * 5, 10, 24, g[0], g[4], [], g[1:4], out)
    check(got, want)


@pytest.mark.parametrize("cfg", ["64x1", "16x8"])
def test_resident_factor_measurement_tilings(eb, cfg, opts):
    """Both shipped resident-factor tilings (forced with the rf_cfg option)
    on the C3 term shape (L = 64, R = 24) give the oracle's result.  (The
    measurement-only tilings are compiled into EB_AB_VARIANTS builds only.)"""
    from paper_2206_08301_b200 import _capi as C
    torch = _torch()
    opts("rf_cfg", cfg)
    e = "ijklm,ja,ka,la,ma->ia"
    ext = dict(i=64, j=4, k=4, l=8, m=64, a=24)
    ops = oracle.seeded_inputs(e, ext, 21)
    want = oracle.naive_evaluate(e, ext, ops)
    g = [torch.from_numpy(o).cuda() for o in ops]
    out = torch.zeros(want.shape, dtype=torch.float64, device="cuda")
    got = _contract(eb, C.EB_ROW, C.EB_REDUCE, 1, 64, 4 * 4 * 8, 64, 24, g[0], g[4], [], g[1:4],
                    out)
    check(got, want)


@pytest.mark.parametrize("M,L", [(64, 64), (40, 32), (160, 64)])  # RF (x2) and general kernel
def test_contract_padded_factor_rows(eb, M, L):
    """Factors with a row pitch wider than R (ld = R + 5): the KRP loads, the
    resident B fragments and the staged U tiles all honour ld."""
    from paper_2206_08301_b200 import _capi as C
    torch = _torch()
    rng = np.random.default_rng(M + L)
    J, K, R, pad = 6, 7, 20, 5
    X = rng.uniform(-1, 1, (M, J, K, L))
    F = [rng.uniform(-1, 1, (n, R + pad)) for n in (J, K, L)]
    want = np.einsum("ijkl,ja,ka,la->ia", X, *(f[:, :R] for f in F))
    gX = torch.from_numpy(X).cuda()
    gF = [torch.from_numpy(f).cuda() for f in F]
    out = torch.zeros(M, R, dtype=torch.float64, device="cuda")
    d = C.ContractDesc()
    d.variant, d.mode, d.P, d.M, d.Q, d.L, d.R = C.EB_ROW, C.EB_REDUCE, 1, M, J * K, L, R
    d.X, d.U, d.ldu = gX.data_ptr(), gF[2].data_ptr(), R + pad
    d.n_mid = 2
    d.mid[0] = C.Factor(gF[0].data_ptr(), J, R + pad)
    d.mid[1] = C.Factor(gF[1].data_ptr(), K, R + pad)
    d.out = out.data_ptr()
    L_ = C.lib()
    wb = L_.eb_contract_workspace(ctypes.byref(d))
    ws = torch.empty(max(wb, 8), dtype=torch.uint8, device="cuda")
    C.check(L_.eb_contract(ctypes.byref(d), ctypes.c_void_p(ws.data_ptr()), wb,
                           ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    check(out.cpu().numpy(), want)


def test_back_to_back_contractions_share_workspace(eb):
    """Alternating contractions (general ROW, COL, resident-factor) reuse one
    workspace with no host sync between them: every kernel of the chain is
    launched with programmatic dependent launch, so this checks that none
    touches global memory before its grid-dependency wait (a staging kernel
    overwriting factors the previous contraction still reads would show)."""
    from paper_2206_08301_b200 import _capi as C
    torch = _torch()
    rng = np.random.default_rng(5)
    I, J, K, R = 160, 96, 64, 24
    X = rng.uniform(-1, 1, (I, J, K))
    gX = torch.from_numpy(X).cuda()
    L_ = C.lib()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    outs, wants = [], []
    for it in range(12):
        A, B, Cf = (rng.uniform(-1, 1, (n, R)) for n in (I, J, K))
        gA, gB, gC = (torch.from_numpy(a).cuda() for a in (A, B, Cf))
        out = torch.zeros(I if it % 3 != 2 else K, R, dtype=torch.float64, device="cuda")
        d = C.ContractDesc()
        if it % 3 == 0:    # mode 0, general ROW kernel (M = 160 >= 128)
            d.variant, d.mode, d.P, d.M, d.Q, d.L, d.R = C.EB_ROW, C.EB_REDUCE, 1, I, J, K, R
            d.U, d.n_mid = gC.data_ptr(), 1
            d.mid[0] = C.Factor(gB.data_ptr(), J, R)
            want = np.einsum("ijk,jr,kr->ir", X, B, Cf)
        elif it % 3 == 1:  # mode 0 on 64-row slab: resident-factor kernel (L = 64)
            d.variant, d.mode, d.P, d.M, d.Q, d.L, d.R = C.EB_ROW, C.EB_REDUCE, 1, 64, J, K, R
            d.U, d.n_mid = gC.data_ptr(), 1
            d.mid[0] = C.Factor(gB.data_ptr(), J, R)
            want = np.zeros((I, R))
            want[:64] = np.einsum("ijk,jr,kr->ir", X[:64], B, Cf)
        else:              # mode 2, COL kernel
            d.variant, d.mode, d.P, d.M, d.Q, d.L, d.R = C.EB_COL, C.EB_REDUCE, I, K, J, 0, R
            d.U, d.n_pre = gB.data_ptr(), 1
            d.pre[0] = C.Factor(gA.data_ptr(), I, R)
            want = np.einsum("ijk,ir,jr->kr", X, A, B)
        d.X, d.ldu, d.out = gX.data_ptr(), R, out.data_ptr()
        assert L_.eb_contract_workspace(ctypes.byref(d)) <= ws.numel()
        C.check(L_.eb_contract(ctypes.byref(d), ctypes.c_void_p(ws.data_ptr()), ws.numel(), st))
        outs.append((out, gA, gB, gC))  # keep the factors alive until the sync
        wants.append(want)
    torch.cuda.synchronize()
    for (out, *_), want in zip(outs, wants):
        check(out.cpu().numpy(), want)


RF_CASES = [  # (einsum, extents, P, M, Q, L, #pre, #mid): the resident-factor path
    ("ijklm,ja,ka,la,ma->ia", dict(i=40, j=6, k=7, l=5, m=64, a=24), 1, 40, 210, 64, 0, 3),
    ("ijkl,ja,ka,la->ia", dict(i=100, j=9, k=4, l=32, a=16), 1, 100, 36, 32, 0, 2),
    ("ijk,ia,ka->ja", dict(i=13, j=50, k=48, a=5), 13, 50, 1, 48, 1, 0),
    ("ijkl,ia,ka,la->ja", dict(i=7, j=64, k=11, l=16, a=20), 7, 64, 11, 16, 1, 1),
    ("ijk,ja,ka->ia", dict(i=1, j=300, k=64, a=24), 1, 1, 300, 64, 0, 1),
]


@pytest.mark.parametrize("case", range(len(RF_CASES)))
@pytest.mark.parametrize("knob", ["", "rf_cfg=64x1", "no_rf=1"])
def test_contract_resident_factor_path(eb, case, knob, opts):
    """Short contracted mode (L <= 64, L % 16 == 0), R <= 24, M < 128: the
    resident-factor kernel (mttkrp_rf.cu; the paired 16 x 8 tiling, or the
    64 x 1 one) and, with EB_NO_RF, the general kernel — all against the
    oracle."""
    from paper_2206_08301_b200 import _capi as C
    torch = _torch()
    e, ext, P, M, Q, L, npre, nmid = RF_CASES[case]
    if knob:
        k, v = knob.split("=")
        opts(k, v)
    ops = oracle.seeded_inputs(e, ext, 31 + case)
    want = oracle.naive_evaluate(e, ext, ops)
    g = [torch.from_numpy(o).cuda() for o in ops]
    facs = g[1:-1]
    out = torch.zeros(want.shape, dtype=torch.float64, device="cuda")
    got = _contract(eb, C.EB_ROW, C.EB_REDUCE, P, M, Q, L, ext["a"], g[0], g[-1], facs[:npre],
                    facs[npre:npre + nmid], out)
    check(got, want)


# ------------------------------------------------------- executor / C ABI --

@pytest.mark.parametrize("name,einsum,ext", DESK, ids=[d[0] for d in DESK])
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_run_json_desk_kernels(eb, name, einsum, ext, P):
    """einplan_run_json on the GPU (virtual ranks), verified on the device,
    and its output equal to the oracle at the same seed."""
    s = eb.Session(einsum, ext)
    path = f"/tmp/eb_out_{name}_{P}.jsonl"
    st, rep = s.run_json(P, 1024.0, seed=1000, verify=True, dump_output=path)
    j = json.loads(rep)
    assert st == 0 and j["verification"]["pass"], j["verification"]
    ops = oracle.seeded_inputs(einsum, ext, 1000)
    want = oracle.naive_evaluate(einsum, ext, ops)
    got = np.loadtxt(path, skiprows=1)
    check(got, want)


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_run_json_order5_resident_factor_blocks(eb, P):
    """Order-5 mode 0 with a 64-long last mode through einplan_run_json: the
    per-rank blocks of every grid the planner picks go to the resident-factor
    kernel (L = 64 or a 16-multiple slice of it) and the device reductions."""
    e = "ijklm,ja,ka,la,ma->ia"
    ext = dict(i=16, j=8, k=8, l=8, m=64, a=24)
    s = eb.Session(e, ext)
    path = f"/tmp/eb_out_rf_{P}.jsonl"
    st, rep = s.run_json(P, 1024.0, seed=77, verify=False, dump_output=path)
    assert st == 0, rep
    ops = oracle.seeded_inputs(e, ext, 77)
    check(np.loadtxt(path, skiprows=1), oracle.naive_evaluate(e, ext, ops))


def _random_case(rng):
    """A random MTTKRP (any mode, order 3-5) or TTMc (order 3-4) einsum with
    small, often odd / ragged extents and a random processor count."""
    order = int(rng.integers(3, 6))
    modes = "ijklm"[:order]
    ext = {c: int(rng.integers(2, 13 if order > 3 else 40)) for c in modes}
    if rng.random() < 0.6:
        m = int(rng.integers(0, order))
        R = int(rng.integers(1, 40))
        ext["a"] = R
        ins = [modes] + [c + "a" for c in modes if c != modes[m]]
        e = ",".join(ins) + "->" + modes[m] + "a"
    else:
        order = min(order, 4)
        modes = modes[:order]
        ext = {c: ext[c] for c in modes}
        ranks = "bcd"[:order - 1]
        for r in ranks:
            ext[r] = int(rng.integers(1, 12))
        ins = [modes] + [c + r for c, r in zip(modes[1:], ranks)]
        e = ",".join(ins) + "->" + modes[0] + ranks
    P = int(rng.choice([1, 2, 3, 4, 6, 8]))
    return e, ext, P


@pytest.mark.parametrize("fmt", ["npy", "jsonl"])
def test_run_json_tensor_files(eb, tmp_path, fmt):
    """einplan_run_json with input_paths / dump_output (tensor.cpp:76-103):
    the reference's jsonl format and the binary .npy side format (for GB-scale
    operands) give the oracle's result for the given inputs."""
    e, ext = "ijk,ja,ka->ia", dict(i=40, j=33, k=18, a=12)
    rng = np.random.default_rng(5)
    ops = [rng.uniform(-1, 1, oracle.shape_of(t, ext)) for t in e.split("->")[0].split(",")]
    paths = []
    for k, a in enumerate(ops):
        pth = str(tmp_path / f"in{k}.{fmt}")
        if fmt == "npy":
            np.save(pth, a)
        else:
            with open(pth, "w") as f:
                f.write(json.dumps({"shape": list(a.shape)}) + "\n")
                f.writelines(repr(float(v)) + "\n" for v in a.ravel())
        paths.append(pth)
    out = str(tmp_path / f"out.{fmt}")
    st, rep = eb.Session(e, ext).run_json(4, 1024.0, seed=0, verify=True,
                                          input_paths=",".join(paths), dump_output=out)
    assert st == 0 and json.loads(rep)["verification"]["pass"]
    got = np.load(out) if fmt == "npy" else np.loadtxt(out, skiprows=1)
    check(np.asarray(got).reshape(40, 12), oracle.naive_evaluate(e, ext, ops))


@pytest.mark.parametrize("seed", range(48))
def test_random_einsums_match_oracle(eb, seed):
    """Randomised parity: random MTTKRP / TTMc einsums, extents (odd and
    ragged) and P through the executor (fused kernels, TTM steps, padded odd
    extents, permuted TTM results, reductions and redistributions on virtual
    ranks) against the oracle's naive loop.  With every extent >= 2 no step
    may fall back to the generic (non-tensor-core) kernel."""
    rng = np.random.default_rng(1000 + seed)
    e, ext, P = _random_case(rng)
    ops = oracle.seeded_inputs(e, ext, seed)
    want = oracle.naive_evaluate(e, ext, ops)
    ex = eb.Executor(e, ext, P)
    ex.stage(ops)
    ex.run()
    check(ex.gather(), want)
    if min(ext.values()) >= 2:
        assert ex.stats()["generic_launches"] == 0, (e, ext, P, ex.stats())


@pytest.mark.parametrize("name,einsum,ext", DESK, ids=[d[0] for d in DESK])
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_comm_volumes_match_reference_accounting(eb, name, einsum, ext, P):
    """allreduce = elems x (group - 1); redistribute = plan transmitted volume
    (executor.cpp:103-105, 193-198; acceptance.cpp:377-426)."""
    ex = eb.Executor(einsum, ext, P)
    ex.stage(oracle.seeded_inputs(einsum, ext, 3))
    ex.run()
    out = ex.gather()
    st = ex.stats()
    plan = json.loads(eb.plan_json(einsum, ext, P))
    red = sum(r["plan"]["transmitted_volume"] for r in plan["schedule"]["redistributions"])
    assert st["redistribute_volume"] == red
    if oracle.ref_available():
        _, _, comm = oracle.ref_run(einsum, ext, P, oracle.seeded_inputs(einsum, ext, 3))
        assert (st["allreduce_volume"], st["redistribute_volume"], st["max_rank_sent"]) == comm
    want = oracle.naive_evaluate(einsum, ext, oracle.seeded_inputs(einsum, ext, 3))
    check(out, want)


def test_hot_path_kernels_are_the_ones_launched(eb):
    """MTTKRP terms go to the fused DMMA kernel, TTM steps to the batched
    kernel; nothing falls back to the generic path for the BASELINE shapes."""
    ex = eb.Executor("ijk,ja,ka->ia", dict(i=64, j=64, k=64, a=24), 8)
    ex.stage(oracle.seeded_inputs("ijk,ja,ka->ia", dict(i=64, j=64, k=64, a=24), 0))
    ex.run()
    st = ex.stats()
    assert st["fused_launches"] == 8 and st["generic_launches"] == 0
    ext = dict(i=64, j=64, k=64, b=16, c=16)
    ex = eb.Executor("ijk,jb,kc->ibc", ext, 4)
    ex.stage(oracle.seeded_inputs("ijk,jb,kc->ibc", ext, 0))
    ex.run()
    st = ex.stats()
    assert st["ttm_launches"] == 8 and st["generic_launches"] == 0


def test_run_is_bitwise_deterministic(eb):
    # acceptance.cpp:428-438: identically seeded runs give identical reports.
    s = eb.Session("ijk,ja,ka->ia", dict(i=10, j=10, k=10, a=6))
    a = s.run_json(8, 512.0, seed=4242, verify=True)
    b = s.run_json(8, 512.0, seed=4242, verify=True)
    assert a == b


def test_corrupt_output_negative_control(eb, monkeypatch):
    # executor.cpp:252-253 / capi.cpp:214: the hook must be caught.
    from paper_2206_08301_b200 import _capi
    monkeypatch.setenv("EINPLAN_TEST_CORRUPT", "1")
    s = eb.Session("ijk,ja,ka->ia", dict(i=10, j=10, k=10, a=6))
    st, rep = s.run_json(2, 1024.0, seed=1, verify=True)
    assert st == _capi.EINPLAN_E_VERIFY and json.loads(rep)["verification"]["pass"] is False


def test_bench_suite_small_scale(eb):
    st, rep = eb.bench_json(1 / 64, 8, 1024.0, 1)
    j = json.loads(rep)
    assert st == 0 and j["all_pass"], [k for k in j["kernels"] if not k["pass"]]


# ----------------------------------------------------- BASELINE full sizes --

def _golden(tag):
    p = os.path.join(GOLD, f"{tag}_summary.json")
    if not os.path.exists(p):
        pytest.skip(f"golden {tag} not generated")
    return json.load(open(p))


def _against_golden(tag, out):
    g = _golden(tag)
    out = np.asarray(out).ravel()
    npy = os.path.join(GOLD, f"{tag}_out.npy")
    if os.path.exists(npy):
        check(out, np.load(npy).ravel())
    idx = np.array(g["sample_index"])
    want = np.array(g["sample_value"])
    assert oracle.normwise_error(out[idx], want) <= TOL
    assert abs(out.sum() - g["sum"]) <= 1e-9 * max(1.0, abs(g["sum"]))
    norm = float(np.sqrt(np.sum(out.astype(np.longdouble) ** 2)))
    assert abs(norm - g["norm2"]) <= 1e-12 * g["norm2"]


@pytest.mark.parametrize("P", [1, 8])
def test_c1_full_size(eb, P):
    c = CONFIGS["C1"]
    e, ext = c["einsums"][0], c["extents"](P)
    ex = eb.Executor(e, ext, P)
    ex.stage(seeded(e, ext, 0))
    ex.run()
    _against_golden("C1", ex.gather())


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_c2_full_size(eb, mode):
    c = CONFIGS["C2"]
    e, ext = c["einsums"][mode], c["extents"](1)
    ex = eb.Executor(e, ext, 1)
    ex.stage(c2_inputs(mode, ext))
    ex.run()
    _against_golden(f"C2_m{mode}", ex.gather())


def test_c2_full_size_dimension_tree(eb):
    """The CP sweep with the dimension tree (bench.py --sweep dimtree): modes 0
    and 1 from one pass over the 8.6 GB X must still match the reference's
    own per-mode outputs (goldens)."""
    c = CONFIGS["C2"]
    ext = c["extents"](1)
    e0, e1 = c["einsums"][0], c["einsums"][1]
    ins0, ins1 = c2_inputs(0, ext), c2_inputs(1, ext)
    ex0 = eb.Executor(e0, ext, 1)
    ex0.stage(ins0)
    ex1 = eb.Executor(e1, ext, 1)
    ex1.share_input(0, ex0, 0)
    ex1.share_input(2, ex0, 2)
    ex1.stage([None, ins1[1], None])
    assert ex0.run_pair(ex1)
    _against_golden("C2_m0", ex0.gather())
    _against_golden("C2_m1", ex1.gather())


def test_c3_full_size(eb):
    c = CONFIGS["C3"]
    e, ext = c["einsums"][0], c["extents"](1)
    ex = eb.Executor(e, ext, 1)
    ex.stage(seeded(e, ext, 0))
    ex.run()
    _against_golden("C3", ex.gather())


def test_c4_full_size(eb):
    c = CONFIGS["C4"]
    e, ext = c["einsums"][0], c["extents"](1)
    ex = eb.Executor(e, ext, 1)
    ex.stage(seeded(e, ext, 0))
    ex.run()
    _against_golden("C4", ex.gather())


def test_c5_full_size(eb):
    c = CONFIGS["C5"]
    e, ext = c["einsums"][0], c["extents"](1)
    ex = eb.Executor(e, ext, 1)
    ex.stage(seeded(e, ext, 0))
    ex.run()
    _against_golden("C5", ex.gather())


def test_c4_two_ranks_redistribution_full_size(eb):
    """C4 at P=2 exchanges the 537 MB intermediate t0 between term grids
    (k2 -> b2); the output must equal the P=1 golden (no contracted dim is
    split: bit-identical across P in the reference)."""
    c = CONFIGS["C4"]
    e, ext = c["einsums"][0], c["extents"](2)
    ex = eb.Executor(e, ext, 2)
    ex.stage(seeded(e, ext, 0))
    ex.run()
    assert ex.stats()["redistribute_volume"] == 33554432
    _against_golden("C4", ex.gather())


def test_reference_c_smoke_runs_on_gpu(eb):
    """The reference's capi_smoke.c (compiled against include/einplan/einplan.h
    and libeinplan_b200.so by tests/test_capi_load.py) runs and passes."""
    import subprocess
    exe = os.path.join(os.path.dirname(__file__), "_bin", "capi_smoke")
    if not os.path.exists(exe):
        pytest.skip("capi_smoke not built (needs the reference sources at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr


def test_share_input_across_modes(eb):
    """One X staged once and aliased by the three MTTKRP executors of a sweep
    (eb_exec_share_input); each mode must still match the oracle."""
    ext = dict(i=48, j=40, k=36, a=16)
    es = ["ijk,ja,ka->ia", "ijk,ia,ka->ja", "ijk,ia,ja->ka"]
    X = oracle.random_tensor((48, 40, 36), 0)
    F = {c: oracle.random_tensor((ext[c], 16), s) for c, s in (("i", 1), ("j", 2), ("k", 3))}
    ex0 = None
    for m, e in enumerate(es):
        ins, _ = oracle.parse(e)
        ops = [X] + [F[t[0]] for t in ins[1:]]
        for P in (1, 4):
            ex = eb.Executor(e, ext, P)
            if m == 0:
                ex.stage(ops)
                if P == 4:
                    ex0 = ex
            else:
                if P == 4:
                    ex = eb.Executor(e, ext, like=ex0)  # same ranks / transport as mode 0
                    ex.share_input(0, ex0, 0)
                    ex.stage([None] + ops[1:])
                else:
                    ex.stage(ops)
            ex.run()
            check(ex.gather(), oracle.naive_evaluate(e, ext, ops))


def test_stage_block_one_rank_process(eb):
    """eb_exec_block / eb_exec_stage_block on a one-rank NCCL executor: the
    rank's boxes generated with eb_random_fill_block (no global tensor) give
    the same output as staging the global tensors."""
    e, ext = "ijk,jb,kc->ibc", dict(i=24, j=40, k=32, b=8, c=6)
    nid = eb.Executor.nccl_unique_id()
    ex = eb.Executor(e, ext, 1, rank=0, nccl_id=nid)
    ins = e.split("->")[0].split(",")
    for k, t in enumerate(ins):
        base, shape = ex.block(k)
        gshape = [ext[c] for c in t]
        assert base == [0] * len(t) and shape == gshape
        ex.stage_block(k, eb.random_block(k, gshape, base, shape))
    ex.run()
    got = ex.gather()
    want = oracle.naive_evaluate(e, ext, oracle.seeded_inputs(e, ext, 0))
    check(got, want)


def test_nccl_transport_single_rank(eb):
    """The one-process-per-GPU transport (NCCL communicator from a unique id,
    rank 0 of 1) runs the schedule and gathers on rank 0.  Multi-rank NCCL
    needs several GPUs; the exchange logic is covered by the gloo tests."""
    ext = dict(i=32, j=24, k=20, a=8)
    e = "ijk,ja,ka->ia"
    ops = oracle.seeded_inputs(e, ext, 4)
    nid = eb.Executor.nccl_unique_id()
    assert len(nid) == 128
    ex = eb.Executor(e, ext, 1, 1024.0, rank=0, nccl_id=nid)
    ex2 = eb.Executor("ijk,ia,ka->ja", ext, like=ex)
    ex.stage(ops)
    ex.run()
    check(ex.gather(), oracle.naive_evaluate(e, ext, ops))
    ops2 = oracle.seeded_inputs("ijk,ia,ka->ja", ext, 4)
    ex2.stage(ops2)
    ex2.run()
    check(ex2.gather(), oracle.naive_evaluate("ijk,ia,ka->ja", ext, ops2))


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name,einsum,ext", DESK, ids=[d[0] for d in DESK])
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_run_report_matches_reference_report(eb, name, einsum, ext, P):
    """our einplan_run_json report (GPU execution) against the
    reference's own einplan_run_json on the same session: every field is
    identical (tree, partition, schedule, comm volumes, verification verdict,
    output shape) except the floating-point ones, which agree to tolerance."""
    st, mine = eb.Session(einsum, ext).run_json(P, 1024.0, seed=7, verify=True)
    rst, theirs = oracle.ref_run_json(einsum, ext, P, 1024.0, seed=7, verify=True)
    assert st == rst == 0
    a, b = json.loads(mine), json.loads(theirs)
    # the B200 extension field (how the ranks ran) comes after every reference field
    assert list(a.keys())[-1] == "execution" and "execution" not in b
    assert a.pop("execution")["mode"] in ("devices", "virtual")
    sa, sb = a["output"].pop("sum"), b["output"].pop("sum")
    assert abs(sa - sb) <= 1e-11 * max(1.0, abs(sb))
    ea = a["verification"].pop("max_rel_error")
    eb_ = b["verification"].pop("max_rel_error")
    assert ea <= 1e-10 and eb_ <= 1e-10
    assert list(a.keys()) == list(b.keys())
    assert a == b


@pytest.mark.parametrize("M,L,R", [(128, 16, 65), (300, 96, 200), (257, 64, 130),
                                   (1000, 512, 1024), (4096, 4096, 72)])
@pytest.mark.parametrize("gemm_mode", [True, False])
def test_contract_gemm_wide(eb, M, L, R, gemm_mode, opts):
    """GEMM steps with N = R > 64 (the 1MM/2MM/3MM chains):
    the GEMM mode of the contraction kernel (items = row tile x 64-column
    block, whole K loop per item, Uᵀ staged once, direct stores) and, forced
    off, the per-64-column split-K path — both against numpy FP64."""
    from paper_2206_08301_b200 import _capi as C
    torch = _torch()
    opts("gemm", 1 if gemm_mode else 2)
    A = oracle.random_tensor((M, L), 41)
    B = oracle.random_tensor((L, R), 42)
    want = A @ B
    out = torch.full((M, R), float("nan"), dtype=torch.float64, device="cuda")
    got = _contract(eb, C.EB_ROW, C.EB_REDUCE, 1, M, 1, L, R, torch.from_numpy(A).cuda(),
                    torch.from_numpy(B).cuda(), [], [], out)
    check(got, want)


def test_executor_gemm_chain_uses_the_gemm_mode(eb):
    """2MM through the executor at P = 1 and 4: every step on the DMMA
    contraction kernel (no generic launches), equal to the oracle chain."""
    e, ext = "ij,jk,kl->il", dict(i=256, j=192, k=160, l=320)
    ops = oracle.seeded_inputs(e, ext, 9)
    want = oracle.naive_evaluate(e, ext, ops)
    for P in (1, 4):
        ex = eb.Executor(e, ext, P)
        ex.stage(ops)
        ex.run()
        st = ex.stats()
        assert st["generic_launches"] == 0, st
        check(ex.gather(), want)


@pytest.mark.parametrize("e,ext", [
    ("ijk,ja,ka->ia", dict(i=40, j=36, k=35, a=24)),      # ROW, odd contracted extent
    ("ijk,ia,ka->ja", dict(i=30, j=130, k=17, a=8)),      # ROW mode 1, odd L
    ("ijk,ia,ja->ka", dict(i=12, j=10, k=137, a=24)),     # COL, odd output extent
    ("ijk,jb,kc->ibc", dict(i=20, j=31, k=33, b=8, c=5)),  # TTMs with odd extents
    ("ijkl,jb,kc,ld->ibcd", dict(i=8, j=11, k=2, l=7, b=2, c=3, d=5)),  # permuted results
    ("ij,jk,kl->il", dict(i=33, j=35, k=37, l=39)),       # GEMM chain, odd everything
])
@pytest.mark.parametrize("P", [1, 4])
def test_odd_extents_stay_on_the_dmma_path(eb, e, ext, P):
    """Odd contiguous extents are zero-padded (TMA needs 16-byte pitches) and
    TTM results in another index order are permuted after the kernel: no step
    falls back to the generic kernel, and the result equals the oracle's."""
    ops = oracle.seeded_inputs(e, ext, 51)
    want = oracle.naive_evaluate(e, ext, ops)
    ex = eb.Executor(e, ext, P)
    ex.stage(ops)
    ex.run()
    st = ex.stats()
    assert st["generic_launches"] == 0, st
    assert st["fused_launches"] + st["ttm_launches"] > 0, st
    check(ex.gather(), want)


@pytest.mark.parametrize("e,ext,P", [
    ("ijk,jb,kc->ibc", dict(i=96, j=96, k=96, b=24, c=24), 2),    # C4-like: k2 -> i2
    ("ijk,jb,kc->ibc", dict(i=96, j=96, k=96, b=24, c=24), 4),    # k4 -> i2 b2
    ("ijk,jb,kc->ibc", dict(i=128, j=128, k=128, b=32, c=32), 8),
    ("ijklm,jb,kc,ld,me->ibcde", dict(i=32, j=16, k=16, l=16, m=16, b=12, c=12, d=12, e=12),
     4),                                                            # eb_ttm2 epilogue: i2m2 -> i2c2
])
def test_fused_redistribution_push(eb, e, ext, P, opts):
    """The redistribution of a TTMc intermediate fused into its producer: the
    TTM (COL BATCHED) / TTM-pair (eb_ttm2) epilogue stores every element
    straight into the next term's destination blocks (eb_scatter).  Bitwise
    equal to the separate apply_plan copy, same comm accounting, and equal to
    the oracle chain."""
    ops = oracle.seeded_inputs(e, ext, 61)
    if e.startswith("ijklm"):
        want = _ttmc_o5_chain(ext, ops)
    else:
        want = oracle.naive_evaluate(e, ext, ops)
    outs, stats = [], []
    for fuse in (1, 0):
        opts("fuse_redistribution", fuse)
        ex = eb.Executor(e, ext, P)
        ex.stage(ops)
        ex.run()
        outs.append(ex.gather())
        stats.append(ex.stats())
        ex.close()
    assert stats[0]["fused_redistributions"] == 1, stats[0]
    assert stats[1]["fused_redistributions"] == 0
    assert stats[0]["redistribute_volume"] == stats[1]["redistribute_volume"] > 0
    assert stats[0]["max_rank_sent"] == stats[1]["max_rank_sent"]
    assert np.array_equal(outs[0], outs[1])
    check(outs[0], want)


def test_scatter_rejects_bad_descriptors(eb):
    from paper_2206_08301_b200 import _capi as C
    L = C.lib()
    d = C.Ttm2Desc(1, 4, 4, 16, 4, 4, 8, 8, 4, 8, 4, 8)
    assert L.eb_ttm2_scatter(ctypes.byref(d), None, None) == 1  # EB_E_INVALID


@pytest.mark.parametrize("P,ext", [
    (1, dict(i=32, j=16, k=16, l=16, m=16, b=12, c=12, d=12, e=12)),
    (2, dict(i=64, j=16, k=16, l=16, m=16, b=12, c=12, d=12, e=12)),
    (1, dict(i=20, j=24, k=20, l=18, m=14, b=16, c=16, d=16, e=16)),   # ragged row tiles
    (2, dict(i=128, j=32, k=32, l=32, m=32, b=16, c=16, d=16, e=16)),
])
def test_ttm2_chain_both_terms_one_launch(eb, P, ext, opts):
    """TTMc-O5 with both terms in one persistent eb_ttm2_chain launch per rank
    (t1 handed over through L2, slab dependencies inside the grid): equal to
    the oracle chain and to the two-launch path, repeatedly (the in-kernel
    counters are re-zeroed per launch)."""
    e = "ijklm,jb,kc,ld,me->ibcde"
    ops = oracle.seeded_inputs(e, ext, 71)
    want = _ttmc_o5_chain(ext, ops)
    opts("chain_terms", 1)
    ex = eb.Executor(e, ext, P)
    ex.stage(ops)
    for _ in range(3):
        ex.run()
        assert ex.stats()["fused_launches"] == P
        check(ex.gather(), want)
    opts("chain_terms", 0)
    ex2 = eb.Executor(e, ext, P)
    ex2.stage(ops)
    ex2.run()
    assert ex2.stats()["fused_launches"] == 2 * P
    check(ex2.gather(), want)


@pytest.mark.parametrize("e,ext,P", [
    ("ijklm,jb,kc,ld,me->ibcde", dict(i=128, j=32, k=32, l=32, m=32, b=16, c=16, d=16, e=16), 4),
    ("ijklm,jb,kc,ld,me->ibcde", dict(i=256, j=32, k=32, l=32, m=32, b=16, c=16, d=16, e=16), 4),
    ("ijk,jb,kc->ibc", dict(i=256, j=256, k=256, b=64, c=64), 8),
])
@pytest.mark.parametrize("variant", [1, 2])
def test_back_to_back_runs_are_bitwise_stable(eb, e, ext, P, variant, opts):
    """Batches of back-to-back runs with no host sync in between (the bench
    pattern: launches overlap under programmatic dependent launch, blocks are
    recycled by the stream-ordered pool) give bitwise the output of a single
    synchronised run, with the pushed destination blocks zeroed before every
    run (so a store the scatter epilogue misses cannot hide behind the
    previous run's identical data), for both ttm2 step-0 splits."""
    import torch
    ops = oracle.seeded_inputs(e, ext, 81)
    # the separate-copy path (every kernel of it is pinned to the oracle in
    # the tests above) is the want: the fused path must equal it bitwise
    opts("fuse_redistribution", 0)
    sep = eb.Executor(e, ext, P)
    sep.stage(ops)
    sep.run()
    want = sep.gather().copy()
    sep.close()
    opts("fuse_redistribution", 1)
    opts("zero_push", 1)
    opts("ttm2_variant", variant)
    ex = eb.Executor(e, ext, P)
    ex.stage(ops)
    ex.run()
    torch.cuda.synchronize()
    ref = ex.gather().copy()
    assert np.array_equal(ref, want)
    assert ex.stats()["fused_redistributions"] == 1
    for _ in range(6):
        for _ in range(5):
            ex.run()
        assert np.array_equal(ex.gather(), ref)


# ---------------------------------------------------- TTMc-O5 fold (m in A) --

def _fold_descs(C, ext, X, U1, U2, U3, U4, out):
    i, j, k, l, m = (ext[c] for c in "ijklm")
    b, c, d, e = (ext[s] for s in "bcde")
    da = C.Ttm2Desc(i, j, k, l * m, b, c, X.data_ptr(), U1.data_ptr(), b, U2.data_ptr(), c, None)
    db = C.Ttm2Desc(i, l, m, b * c, d, e, None, U3.data_ptr(), d, U4.data_ptr(), e,
                    out.data_ptr())
    return da, db


@pytest.mark.parametrize("ext", [
    dict(i=3, j=16, k=16, l=4, m=16, b=16, c=16, d=16, e=16),
    dict(i=2, j=20, k=13, l=3, m=32, b=12, c=11, d=9, e=13),     # ragged j, k, odd c
    dict(i=5, j=64, k=64, l=2, m=64, b=16, c=16, d=16, e=16),    # C5 tile shape, l small
    dict(i=1, j=7, k=5, l=9, m=48, b=5, c=16, d=16, e=1),
    dict(i=300, j=8, k=4, l=2, m=16, b=4, c=4, d=3, e=2),        # more fold groups than SMs
])
def test_ttmc_fold_kernel(eb, ext):
    """eb_ttmc_fold = both TTMc-O5 terms with term B's m contraction folded
    into term A's epilogue (t1 never stored), against the oracle's step-by-step
    reference chain (ijklm -> iklmb -> ilmbc -> imbcd -> ibcde), ragged in
    every extent the kernel allows; the result must not depend on workspace
    contents (filled with NaN first)."""
    from paper_2206_08301_b200 import _capi as C
    torch = _torch()
    e = "ijklm,jb,kc,ld,me->ibcde"
    ops = oracle.seeded_inputs(e, ext, 97)
    want = _ttmc_o5_chain(ext, ops)
    X, U1, U2, U3, U4 = [torch.from_numpy(o).cuda() for o in ops]
    out = torch.full(want.shape, float("nan"), dtype=torch.float64, device="cuda")
    da, db = _fold_descs(C, ext, X, U1, U2, U3, U4, out)
    L = C.lib()
    wb = L.eb_ttmc_fold_workspace(ctypes.byref(da), ctypes.byref(db))
    assert wb == 8 * ext["i"] * ext["l"] * ext["e"] * ext["b"] * ext["c"]
    ws = torch.full((wb // 8,), float("nan"), dtype=torch.float64, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for _ in range(2):
        C.check(L.eb_ttmc_fold(ctypes.byref(da), ctypes.byref(db), ctypes.c_void_p(ws.data_ptr()),
                               wb, st))
        torch.cuda.synchronize()
        check(out.cpu().numpy(), want)


def test_ttmc_fold_rejects_unsupported_shapes(eb):
    from paper_2206_08301_b200 import _capi as C
    torch = _torch()
    L = C.lib()
    buf = torch.zeros(1 << 16, dtype=torch.float64, device="cuda")
    p = buf.data_ptr()
    for m, e, d in ((14, 4, 4), (80, 4, 4), (16, 17, 4), (16, 4, 17)):
        da = C.Ttm2Desc(1, 4, 4, 2 * m, 4, 4, p, p, 4, p, 4, None)
        db = C.Ttm2Desc(1, 2, m, 16, d, e, None, p, d, p, e, p)
        assert L.eb_ttmc_fold(ctypes.byref(da), ctypes.byref(db), ctypes.c_void_p(p),
                              buf.numel() * 8, None) == 1  # EB_E_INVALID
    da = C.Ttm2Desc(1, 4, 4, 32, 4, 4, p, p, 4, p, 4, None)
    db = C.Ttm2Desc(1, 2, 16, 16, 4, 4, None, p, 4, p, 4, p)
    assert L.eb_ttmc_fold(ctypes.byref(da), ctypes.byref(db), ctypes.c_void_p(p), 8, None) == 1


@pytest.mark.parametrize("P,ext", [
    (1, dict(i=16, j=32, k=32, l=32, m=32, b=16, c=16, d=16, e=16)),
    (2, dict(i=16, j=16, k=16, l=16, m=16, b=12, c=12, d=12, e=12)),
])
def test_executor_folds_ttmc_o5_terms(eb, P, ext, opts):
    """Executor with fold_terms: where the t1 hand-over is a whole-block self
    message on every rank, the TTMc-O5 terms run as eb_ttmc_fold (2 launches
    per rank, t1 not stored); same output as the two-launch path (fold_terms 0)
    and the oracle chain, repeatedly."""
    e = "ijklm,jb,kc,ld,me->ibcde"
    plan_r = json.loads(eb.plan_json(e, ext, P, include_messages=True))
    assert [t["output"] for t in plan_r["schedule"]["terms"]] == ["t1", "out"]
    assert all(m["self"] for r in plan_r["schedule"]["redistributions"]
               for m in r["plan"]["messages"])
    ops = oracle.seeded_inputs(e, ext, 13)
    want = _ttmc_o5_chain(ext, ops)
    opts("fold_terms", 0)
    ref = eb.Executor(e, ext, P)
    ref.stage(ops)
    ref.run()
    two = ref.gather().copy()
    st0 = ref.stats()
    ref.close()
    check(two, want)
    opts("fold_terms", 1)
    ex = eb.Executor(e, ext, P)
    ex.stage(ops)
    n0 = eb.launch_count()
    ex.run()
    st = ex.stats()
    assert st["fused_launches"] == 2 * P and st["generic_launches"] == 0, st
    assert st["redistribute_volume"] == st0["redistribute_volume"]
    assert eb.launch_count() - n0 >= 2 * P
    for _ in range(3):
        ex.run()
        got = ex.gather()
        check(got, want)
        check(got, two)
