"""The C-ABI library loads without a GPU and exports every symbol the
headers in include/ declare; the reference's own C smoke test compiles
against our header (the drop-in claim at the source level)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in ("include/einplan/einplan.h", "include/einplan_b200.h"):
        txt = open(os.path.join(ROOT, h)).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        for m in re.finditer(r"\b((?:einplan|eb)_[a-z0-9_]+)\s*\(", txt):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol(eb):
    from paper_2206_08301_b200 import _capi
    lib = ctypes.CDLL(_capi.LIB_PATH)
    declared = _declared()
    assert len(declared) >= 30
    missing = [n for n in sorted(declared) if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_capi.EXPORTS) == declared


def test_no_cuda_call_at_load_and_planning_works_without_gpu(eb):
    # planning is host code: usable on a CPU-only machine
    import json
    j = json.loads(eb.plan_json("ijk,ja,ka->ia", dict(i=8, j=8, k=8, a=4), 8))
    assert j["schedule"]["procs"] == 8
    assert eb.version().endswith("b200")


def test_status_names_match_reference():
    from paper_2206_08301_b200 import _capi
    L = _capi.lib()
    names = [L.einplan_status_name(s).decode() for s in range(8)]
    assert names == ["ok", "verification failed", "parse error", "infeasible fast memory",
                     "invalid process grid", "resource cap exceeded", "invalid argument",
                     "internal error"]


REF_SMOKE = "/root/reference/proj/tests/capi_smoke.c"


@pytest.mark.skipif(not os.path.exists(REF_SMOKE), reason="reference sources not mounted")
def test_reference_c_smoke_compiles_against_our_header(eb, tmp_path):
    exe = os.path.join(ROOT, "tests", "_bin", "capi_smoke")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    libdir = os.path.join(ROOT, "paper_2206_08301_b200", "lib")
    subprocess.run(["gcc", "-std=c11", "-Wall", "-I", os.path.join(ROOT, "include"), REF_SMOKE,
                    "-L", libdir, "-leinplan_b200", f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    assert os.path.exists(exe)


def test_random_block_is_the_box_of_random_tensor(eb):
    """eb_random_fill_block: any box of random_tensor(shape, seed) without the
    global tensor (multi-process staging of GB-scale inputs)."""
    import numpy as np
    import oracle
    g = (6, 7, 9, 5)
    full = oracle.random_tensor(g, 11)
    for base, shape in [((0, 0, 0, 0), g), ((2, 3, 1, 0), (3, 4, 8, 5)), ((5, 6, 8, 4), (1, 1, 1, 1)),
                        ((1, 0, 2, 1), (4, 7, 3, 2))]:
        got = eb.random_block(11, g, base, shape)
        want = full[tuple(slice(a, a + n) for a, n in zip(base, shape))]
        assert np.array_equal(got, want)


def test_path_options_set_and_validated_without_gpu(eb):
    """eb_set_option: the path options are plain host state (read once from
    EB_* at load); unknown names and out-of-range values are rejected."""
    from paper_2206_08301_b200 import EinplanError
    for name, good in (("no_fused_tma", 1), ("no_rf", 1), ("rf_cfg", "64x1"),
                       ("ttm2_variant", 2), ("fuse_ttm2", 0), ("gemm", 1),
                       ("fuse_redistribution", 0), ("chain_terms", 1), ("fold_terms", 1)):
        eb.set_option(name, good)
    for name, value in (("no_fused_tma", 0), ("no_rf", 0), ("rf_cfg", "auto"),
                        ("ttm2_variant", 0), ("fuse_ttm2", 1), ("gemm", 0),
                        ("fuse_redistribution", 1), ("chain_terms", 0), ("fold_terms", 0)):
        eb.set_option(name, value)
    for name, bad in (("no_such_option", 1), ("ttm2_variant", 7), ("gemm", 3),
                      ("rf_cfg", "sixteen")):
        with pytest.raises(EinplanError):
            eb.set_option(name, bad)


def test_random_stream_continues_the_reference_stream(eb):
    """RandomStream (eb_rng_*): consecutive fills are consecutive slices of
    random_tensor's mt19937_64 stream (tensor.cpp:55-63), also from a skip."""
    import numpy as np
    import oracle
    want = oracle.random_tensor((3000,), 5)
    rs = eb.RandomStream(5)
    a = rs.fill(np.empty(1234))
    b = rs.fill(np.empty(1766))
    assert np.array_equal(np.concatenate([a, b]), want)
    c = eb.RandomStream(5, skip=1000).fill(np.empty(500))
    assert np.array_equal(c, want[1000:1500])


def test_python_mirror_rejects_bad_shapes_before_the_abi(eb):
    """Executor.stage / gather check operand counts, shapes and output buffers
    in Python (no host pointer with the wrong size crosses the C ABI)."""
    import numpy as np
    ex = eb.Executor.__new__(eb.Executor)  # no device: exercise the checks only
    ex._shapes = [(4, 5, 6), (5, 3), (6, 3)]
    ex._h = None
    ex.rank = -1
    with pytest.raises(ValueError):
        ex.stage([np.zeros((4, 5, 6))])  # operand count
    with pytest.raises(ValueError):
        ex.stage([np.zeros((4, 5, 7)), np.zeros((5, 3)), np.zeros((6, 3))])  # shape
