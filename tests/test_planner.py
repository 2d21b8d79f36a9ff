"""Host planner parity: the B200 build's restated planner (optimal_path,
SOAP tile solver, choose_grid, placements, redistribution plans) must give
the reference's plan report byte for byte — grids, blocks, replicas,
reduction groups, message lists and the solver's doubles."""
import json
import os
import random

import pytest

import oracle
from tests.configs import CONFIGS

GOLD = os.path.join(os.path.dirname(__file__), "golden", "plans")
needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def _cases():
    for name, c in CONFIGS.items():
        for P in c["procs"]:
            for mode, e in enumerate(c["einsums"]):
                tag = f"{name}_m{mode}" if len(c["einsums"]) > 1 else name
                yield tag, e, c["extents"](P), P


CASES = list(_cases())


@pytest.mark.parametrize("tag,einsum,ext,P", CASES, ids=[f"{c[0]}_P{c[3]}" for c in CASES])
def test_plan_matches_reference_golden(eb, tag, einsum, ext, P):
    want = open(os.path.join(GOLD, f"{tag}_P{P}.json")).read()
    got = eb.plan_json(einsum, ext, P, 1024.0, include_messages=True)
    assert got == want


def test_appendix_a_grids(eb):
    # the processor grids themselves.
    def grids(e, ext, P):
        j = json.loads(eb.plan_json(e, ext, P))
        return [{k: v for k, v in t["grid"].items() if v > 1} for t in j["schedule"]["terms"]]
    c1 = CONFIGS["C1"]["extents"](1)
    assert grids("ijk,ja,ka->ia", c1, 2) == [{"j": 2}]
    assert grids("ijk,ja,ka->ia", c1, 8) == [{"i": 2, "j": 2, "k": 2}]
    c2 = CONFIGS["C2"]["extents"](1)
    for e in CONFIGS["C2"]["einsums"]:
        assert grids(e, c2, 2) == [{"k": 2}]      # exact tie -> lexicographic
        assert grids(e, c2, 4) == [{"j": 2, "k": 2}]
    c4 = CONFIGS["C4"]["extents"](1)
    assert grids("ijk,jb,kc->ibc", c4, 8) == [{"k": 8}, {"i": 2, "b": 4}]
    c5 = CONFIGS["C5"]["extents"](4)
    assert grids("ijklm,jb,kc,ld,me->ibcde", c5, 4) == [{"i": 2, "m": 2}, {"i": 4}]


def test_worked_example(eb):
    # acceptance.cpp:262-345 (SPEC worked example at P = 8).
    ext = dict(i=10, j=10, k=10, a=10, l=10)
    j = json.loads(eb.plan_json("ijk,ja,ka,al->il", ext, 8))
    t0, t1 = j["schedule"]["terms"]
    assert t0["grid"] == {"i": 2, "j": 2, "k": 2, "a": 1}
    assert t1["grid"] == {"i": 2, "a": 2, "l": 2}
    assert t0["blocks"] == {"i": 5, "j": 5, "k": 5, "a": 10}
    assert t0["reduction"] == {"dims": "jk", "depth": 4}
    reds = j["schedule"]["redistributions"]
    assert [r["tensor"] for r in reds] == ["t1"]
    steps = j["tree"]["steps"]
    assert [s["op_class"] for s in steps] == ["KRP", "TDOT", "GEMM"]
    assert steps[0]["expr"] == "ja,ka->jka" and steps[1]["expr"] == "ijk,jka->ia"


def test_mttkrp_closed_forms(eb):
    # acceptance.cpp:227-247: rho = S^(2/3)/3, x0 = 5S/2, tiles S^(1/3), S^(2/3)/2.
    n = 1 << 17
    s = eb.Session("ijk,ja,ka->ia", dict(i=n, j=n, k=n, a=n))
    for S in (512.0, 1024.0, 8192.0):
        b = json.loads(s.bound_json(S))["partition"]["terms"][0]["bound"]
        assert abs(b["rho"] / (S ** (2 / 3) / 3) - 1) < 0.01
        assert abs(b["x0"] / (2.5 * S) - 1) < 0.01
        for c in "ijk":
            assert abs(b["tiles"][c] / S ** (1 / 3) - 1) < 0.01
        assert abs(b["tiles"]["a"] / (S ** (2 / 3) / 2) - 1) < 0.01


def test_gemm_intensity(eb):
    # acceptance.cpp:215-225: GEMM rho = sqrt(S)/2.
    n = 1 << 20
    s = eb.Session("ij,jk->ik", dict(i=n, j=n, k=n))
    for S in (256.0, 1024.0, 4096.0):
        b = json.loads(s.bound_json(S))["partition"]["terms"][0]["bound"]
        assert abs(b["rho"] / (S ** 0.5 / 2) - 1) < 0.005


def test_error_statuses(eb):
    from paper_2206_08301_b200 import _capi
    with pytest.raises(eb.EinplanError) as e:
        eb.Session("ii,j->j", "i=3,j=4")
    assert e.value.status == _capi.EINPLAN_E_PARSE
    with pytest.raises(eb.EinplanError) as e:
        eb.Session("ij,jk->ik", "i=3,j=4")          # k has no extent
    assert e.value.status == _capi.EINPLAN_E_PARSE
    s = eb.Session("ij,jk->ik", dict(i=2, j=2, k=2))
    with pytest.raises(eb.EinplanError) as e:
        s.plan_json(64, 64.0)                          # too many processes
    assert e.value.status == _capi.EINPLAN_E_GRID
    with pytest.raises(eb.EinplanError) as e:
        s.plan_json(1, 2.0)                            # fast memory below #arrays + 1
    assert e.value.status == _capi.EINPLAN_E_INFEASIBLE


def test_resource_cap_before_any_device_work(eb, monkeypatch):
    from paper_2206_08301_b200 import _capi
    monkeypatch.setenv("EINPLAN_MAX_POINTS", "100")
    s = eb.Session("ij,jk->ik", dict(i=8, j=8, k=8))
    with pytest.raises(eb.EinplanError) as e:
        s.run_json(1)
    assert e.value.status == _capi.EINPLAN_E_RESOURCE


def _random_einsum(rng):
    letters = "ijklmnab"
    nops = rng.randint(1, 4)
    ops = []
    for _ in range(nops):
        k = rng.randint(1, 3)
        ops.append("".join(rng.sample(letters[:6], k)))
    used = sorted(set("".join(ops)))
    out = "".join(rng.sample(used, rng.randint(1, min(3, len(used)))))
    ext = {c: rng.randint(2, 12) for c in used}
    return ",".join(ops) + "->" + out, ext


@needs_ref
@pytest.mark.parametrize("seed", range(60))
def test_random_plans_match_reference(eb, seed):
    rng = random.Random(seed)
    e, ext = _random_einsum(rng)
    P = rng.choice([1, 2, 3, 4, 6, 8])
    S = rng.choice([16.0, 64.0, 256.0, 1024.0])
    try:
        want = oracle.ref_plan_json(e, ext, P, S, include_messages=True)
    except RuntimeError:
        want = None
    try:
        got = eb.plan_json(e, ext, P, S, include_messages=True)
    except eb.EinplanError:
        got = None
    assert got == want, (e, ext, P, S)


@needs_ref
@pytest.mark.parametrize("P", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("S", [256.0, 1024.0, 4096.0])
def test_desk_kernels_match_reference(eb, P, S):
    from tests.test_oracle import DESK
    for name, e, ext in DESK:
        try:
            want = oracle.ref_plan_json(e, ext, P, S, include_messages=True)
        except RuntimeError:
            want = None
        try:
            got = eb.plan_json(e, ext, P, S, include_messages=True)
        except eb.EinplanError:
            got = None
        assert got == want, (name, P, S)
