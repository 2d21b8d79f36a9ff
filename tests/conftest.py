import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no GPU in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def eb():
    """The product package with its CUDA library built in-tree."""
    from paper_2206_08301_b200 import build as _b
    _b.build()
    import paper_2206_08301_b200 as pkg
    return pkg


@pytest.fixture(scope="session")
def ora():
    import oracle
    oracle.build(ref=True)
    return oracle


_OPTION_DEFAULTS = {"no_fused_tma": 0, "no_rf": 0, "rf_cfg": "auto", "ttm2_variant": 0,
                    "fuse_ttm2": 1, "gemm": 0, "fuse_redistribution": 1, "chain_terms": 0, "fold_terms": 0, "zero_push": 0,
                    "scatter_fast": 1, "pdl": 1}


@pytest.fixture
def opts(eb):
    """Set kernel-path options (eb_set_option) for one test; restored after."""
    touched = []

    def set_(name, value):
        touched.append(name)
        eb.set_option(name, value)

    yield set_
    for n in touched:
        eb.set_option(n, _OPTION_DEFAULTS[n])
