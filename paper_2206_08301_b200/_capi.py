"""ctypes bindings of the in-tree libeinplan_b200.so (C ABIs in include/).

This is the product path: every compute call goes to the CUDA library.  If
the library cannot be loaded the import of the call site fails loudly —
there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# EB_LIB_PATH: load another build of the library (A/B timing of two builds)
LIB_PATH = os.environ.get("EB_LIB_PATH") or os.path.join(_HERE, "lib", "libeinplan_b200.so")

_dp = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64


class Factor(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("extent", ctypes.c_int64), ("ld", ctypes.c_int64)]


class ContractDesc(ctypes.Structure):
    _fields_ = [
        ("variant", ctypes.c_int), ("mode", ctypes.c_int),
        ("P", ctypes.c_int64), ("M", ctypes.c_int64), ("Q", ctypes.c_int64), ("L", ctypes.c_int64),
        ("R", ctypes.c_int64),
        ("X", ctypes.c_void_p), ("U", ctypes.c_void_p), ("ldu", ctypes.c_int64),
        ("n_pre", ctypes.c_int), ("pre", Factor * 8),
        ("n_mid", ctypes.c_int), ("mid", Factor * 8),
        ("out", ctypes.c_void_p),
    ]


class Ttm2Desc(ctypes.Structure):
    _fields_ = [
        ("P", ctypes.c_int64), ("Q1", ctypes.c_int64), ("Q2", ctypes.c_int64),
        ("M", ctypes.c_int64), ("N1", ctypes.c_int64), ("N2", ctypes.c_int64),
        ("X", ctypes.c_void_p), ("U1", ctypes.c_void_p), ("ldu1", ctypes.c_int64),
        ("U2", ctypes.c_void_p), ("ldu2", ctypes.c_int64), ("out", ctypes.c_void_p),
    ]


EB_ROW, EB_COL = 0, 1
EB_REDUCE, EB_BATCHED = 0, 1

# einplan_status (include/einplan/einplan.h)
EINPLAN_OK, EINPLAN_E_VERIFY, EINPLAN_E_PARSE, EINPLAN_E_INFEASIBLE = 0, 1, 2, 3
EINPLAN_E_GRID, EINPLAN_E_RESOURCE, EINPLAN_E_INVALID, EINPLAN_E_INTERNAL = 4, 5, 6, 7

# Every symbol include/*.h declares (checked by tests/test_capi_load.py).
EXPORTS = [
    "einplan_version", "einplan_status_name", "einplan_last_error", "einplan_free",
    "einplan_session_create", "einplan_session_destroy", "einplan_bound_json",
    "einplan_plan_json", "einplan_run_json", "einplan_bench_json",
    "eb_last_error", "eb_build_info", "eb_contract_workspace", "eb_contract", "eb_mttkrp2_workspace", "eb_mttkrp2", "eb_ttm2",
    "eb_cp3_als_workspace", "eb_cp3_als_sweep",
    "eb_step_generic",
    "eb_group_sum", "eb_group_sum_into", "eb_copy_box", "eb_set_option", "eb_exec_create_peer",
    "eb_exec_stage_region", "eb_rng_create", "eb_rng_fill", "eb_rng_destroy", "eb_mem_in_use", "eb_pad_rows", "eb_permute",
    "eb_contract_scatter", "eb_ttm2_scatter", "eb_exec_fused_redistributions",
    "eb_ttm2_chain", "eb_ttm2_chain_workspace", "eb_ttmc_fold", "eb_ttmc_fold_workspace", "eb_exec_create_hybrid", "eb_einsum_generic", "eb_random_fill_host",
    "eb_random_fill_block", "eb_exec_block", "eb_exec_stage_block", "eb_free",
    "eb_plan_json", "eb_nccl_unique_id", "eb_exec_create", "eb_exec_create_like", "eb_exec_destroy", "eb_exec_stage",
    "eb_exec_share_input", "eb_exec_run", "eb_exec_run_pair", "eb_exec_set_async_reduce",
    "eb_exec_join", "eb_exec_capture", "eb_exec_replay", "eb_exec_gather", "eb_exec_output_elems", "eb_exec_stats",
    "eb_exec_report_json", "eb_launch_count", "eb_timer_enable", "eb_timer_collect",
]

_lib = None


class EinplanError(RuntimeError):
    """A nonzero status from the C ABI (status carries the code)."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status


def _sig(L, name, res, args):
    try:
        f = getattr(L, name)
    except AttributeError:
        # an older build loaded through EB_LIB_PATH (A/B timing); the export
        # test checks that the shipped library has every symbol
        if os.environ.get("EB_LIB_PATH"):
            return
        raise
    f.restype = res
    f.argtypes = args


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: build it with "
                              "`python -m paper_2206_08301_b200.build` (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        c = ctypes.c_char_p
        _sig(L, "einplan_version", c, [])
        _sig(L, "einplan_status_name", c, [ctypes.c_int])
        _sig(L, "einplan_last_error", c, [])
        _sig(L, "einplan_free", None, [_vp])
        _sig(L, "einplan_session_create", ctypes.c_int, [c, c, ctypes.POINTER(_vp)])
        _sig(L, "einplan_session_destroy", None, [_vp])
        _sig(L, "einplan_bound_json", ctypes.c_int, [_vp, ctypes.c_double, ctypes.POINTER(_vp)])
        _sig(L, "einplan_plan_json", ctypes.c_int,
             [_vp, _i64, ctypes.c_double, ctypes.c_int, ctypes.POINTER(_vp)])
        _sig(L, "einplan_run_json", ctypes.c_int,
             [_vp, _i64, ctypes.c_double, ctypes.c_uint64, ctypes.c_int, c, c, ctypes.POINTER(_vp)])
        _sig(L, "einplan_bench_json", ctypes.c_int,
             [ctypes.c_double, _i64, ctypes.c_double, ctypes.c_uint64, ctypes.POINTER(_vp)])
        _sig(L, "eb_last_error", c, [])
        _sig(L, "eb_build_info", c, [])
        _sig(L, "eb_contract_workspace", ctypes.c_size_t, [ctypes.POINTER(ContractDesc)])
        _sig(L, "eb_contract", ctypes.c_int,
             [ctypes.POINTER(ContractDesc), _vp, ctypes.c_size_t, _vp])
        _sig(L, "eb_ttm2", ctypes.c_int, [ctypes.POINTER(Ttm2Desc), _vp])
        _sig(L, "eb_cp3_als_workspace", ctypes.c_size_t, [_i64, _i64, _i64, _i64])
        _sig(L, "eb_cp3_als_sweep", ctypes.c_int,
             [_vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp])
        _sig(L, "eb_mttkrp2_workspace", ctypes.c_size_t, [ctypes.POINTER(ContractDesc)])
        _sig(L, "eb_mttkrp2", ctypes.c_int,
             [ctypes.POINTER(ContractDesc), _vp, _i64, _vp, _vp, ctypes.c_size_t, _vp])
        _sig(L, "eb_exec_run_pair", ctypes.c_int, [_vp, _vp, ctypes.POINTER(ctypes.c_int)])
        _sig(L, "eb_exec_set_async_reduce", ctypes.c_int, [_vp, ctypes.c_int])
        _sig(L, "eb_exec_join", ctypes.c_int, [_vp])
        _sig(L, "eb_exec_capture", ctypes.c_int, [_vp])
        _sig(L, "eb_exec_replay", ctypes.c_int, [_vp])
        _sig(L, "eb_random_fill_host", None, [_dp, _i64, ctypes.c_uint64, _i64])
        _sig(L, "eb_random_fill_block", ctypes.c_int,
             [_dp, ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
              ctypes.POINTER(_i64)])
        _sig(L, "eb_exec_block", ctypes.c_int,
             [_vp, ctypes.c_int, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
              ctypes.POINTER(ctypes.c_int)])
        _sig(L, "eb_exec_stage_block", ctypes.c_int, [_vp, ctypes.c_int, _dp])
        _sig(L, "eb_exec_stage_region", ctypes.c_int,
             [_vp, ctypes.c_int, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.c_int, _dp,
              ctypes.POINTER(ctypes.c_int)])
        _sig(L, "eb_exec_create_peer", ctypes.c_int,
             [c, c, _i64, ctypes.c_double, _i64, c, _vp, ctypes.POINTER(_vp)])
        _sig(L, "eb_set_option", ctypes.c_int, [c, c])
        _sig(L, "eb_exec_create_hybrid", ctypes.c_int,
             [c, c, _i64, ctypes.c_double, _i64, c, _vp, _vp, ctypes.POINTER(_vp)])
        _sig(L, "eb_group_sum", ctypes.c_int, [ctypes.POINTER(_dp), ctypes.c_int, _i64, _vp])
        _sig(L, "eb_group_sum_into", ctypes.c_int,
             [ctypes.POINTER(_dp), ctypes.c_int, _i64, _dp, _vp])
        _sig(L, "eb_copy_box", ctypes.c_int,
             [ctypes.c_int, _vp, ctypes.POINTER(_i64), _vp, ctypes.POINTER(_i64),
              ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i64), _vp])
        _sig(L, "eb_rng_create", ctypes.c_int, [ctypes.c_uint64, _i64, ctypes.POINTER(_vp)])
        _sig(L, "eb_rng_fill", None, [_vp, _dp, _i64])
        _sig(L, "eb_rng_destroy", None, [_vp])
        _sig(L, "eb_mem_in_use", ctypes.c_int, [ctypes.POINTER(_i64)])
        _sig(L, "eb_exec_fused_redistributions", ctypes.c_int, [_vp])
        _sig(L, "eb_ttm2_scatter", ctypes.c_int, [ctypes.POINTER(Ttm2Desc), _vp, _vp])
        _sig(L, "eb_ttm2_chain_workspace", ctypes.c_size_t, [ctypes.POINTER(Ttm2Desc)])
        _sig(L, "eb_ttm2_chain", ctypes.c_int,
             [ctypes.POINTER(Ttm2Desc), ctypes.POINTER(Ttm2Desc), _vp, ctypes.c_size_t, _vp])
        _sig(L, "eb_ttmc_fold_workspace", ctypes.c_size_t,
             [ctypes.POINTER(Ttm2Desc), ctypes.POINTER(Ttm2Desc)])
        _sig(L, "eb_ttmc_fold", ctypes.c_int,
             [ctypes.POINTER(Ttm2Desc), ctypes.POINTER(Ttm2Desc), _vp, ctypes.c_size_t, _vp])
        _sig(L, "eb_free", None, [_vp])
        _sig(L, "eb_plan_json", ctypes.c_int,
             [c, c, _i64, ctypes.c_double, ctypes.c_int, ctypes.POINTER(_vp)])
        _sig(L, "eb_nccl_unique_id", ctypes.c_int, [_vp])
        _sig(L, "eb_exec_create", ctypes.c_int,
             [c, c, _i64, ctypes.c_double, _i64, _vp, _vp, ctypes.POINTER(_vp)])
        _sig(L, "eb_exec_destroy", None, [_vp])
        _sig(L, "eb_exec_create_like", ctypes.c_int,
             [c, c, ctypes.c_double, _vp, _vp, ctypes.POINTER(_vp)])
        _sig(L, "eb_exec_stage", ctypes.c_int, [_vp, ctypes.POINTER(_dp)])
        _sig(L, "eb_exec_run", ctypes.c_int, [_vp])
        _sig(L, "eb_exec_share_input", ctypes.c_int, [_vp, ctypes.c_int, _vp, ctypes.c_int])
        _sig(L, "eb_exec_gather", ctypes.c_int, [_vp, _dp])
        _sig(L, "eb_exec_output_elems", _i64, [_vp])
        _sig(L, "eb_exec_stats", ctypes.c_int, [_vp, ctypes.POINTER(_i64)])
        _sig(L, "eb_exec_report_json", ctypes.c_int, [_vp, _dp, ctypes.POINTER(_vp)])
        _sig(L, "eb_launch_count", ctypes.c_longlong, [])
        _sig(L, "eb_timer_enable", None, [ctypes.c_int])
        _sig(L, "eb_timer_collect", ctypes.c_int,
             [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_longlong)])
        _lib = L
    return _lib


def check(status: int):
    """Raise EinplanError for a nonzero eb_status."""
    if status != 0:
        raise EinplanError(status, lib().eb_last_error().decode())


def take_string(p: ctypes.c_void_p, free=None) -> str:
    s = ctypes.string_at(p).decode()
    (free or lib().einplan_free)(p)
    return s
