"""ctypes bindings of the in-tree libeinplan_b200.so (C ABI in include/).

The product path: every compute call goes to the CUDA library; if it cannot
be loaded the import fails loudly (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libeinplan_b200.so")

_dp = ctypes.POINTER(ctypes.c_double)


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


EB_ROW, EB_COL = 0, 1
EB_REDUCE, EB_BATCHED = 0, 1

_lib = None


class EinplanError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: build it with "
                              "`python -m paper_2206_08301_b200.build` (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        L.eb_last_error.restype = ctypes.c_char_p
        L.eb_contract_workspace.argtypes = [ctypes.POINTER(ContractDesc)]
        L.eb_contract_workspace.restype = ctypes.c_size_t
        L.eb_contract.argtypes = [ctypes.POINTER(ContractDesc), ctypes.c_void_p, ctypes.c_size_t,
                                  ctypes.c_void_p]
        L.eb_contract.restype = ctypes.c_int
        _lib = L
    return _lib


def check(status: int):
    if status != 0:
        raise EinplanError(status, lib().eb_last_error().decode())
