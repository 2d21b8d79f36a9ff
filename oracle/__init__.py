"""CPU oracle for the Deinsum hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and only
as the checker or the timed CPU baseline — never as the thing measured or
shipped.  The product package (``paper_2206_08301_b200``) never imports it.

Two back ends:

* ``liboracle.so`` — ``oracle.c``, a plain-C restatement of the reference's
  ``random_tensor`` (tensor.cpp:55-63), ``naive_evaluate`` (evaluate.cpp:7-63),
  ``max_rel_error`` (tensor.cpp:65-74), the allreduce group sum
  (executor.cpp:80-108) and the redistribution box copy
  (redistribute.cpp:152-183).
* ``_ref/libeinplan_ref.so`` — the reference einplan itself, compiled from
  ``/root/reference/proj/src`` by ``oracle/Makefile`` (git-ignored; travels to
  the GPU box as a prebuilt file).  Used to pin the restatement, to produce
  golden fixtures and schedule JSON, and as the CPU baseline
  (``cpu_baseline.kind == "reference"``).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None
_ref = None
_dp = ctypes.POINTER(ctypes.c_double)


def build(ref: bool = True) -> None:
    """Compile the C oracle and, when /root/reference is present, oracle/_ref."""
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    if ref and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build(ref=False)
        L = ctypes.CDLL(path)
        L.oracle_random_fill.argtypes = [_dp, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int64]
        L.oracle_naive_evaluate.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64),
                                            ctypes.POINTER(_dp), _dp]
        L.oracle_naive_evaluate.restype = ctypes.c_int
        L.oracle_max_rel_error.argtypes = [_dp, _dp, ctypes.c_int64]
        L.oracle_max_rel_error.restype = ctypes.c_double
        L.oracle_normwise_error.argtypes = [_dp, _dp, ctypes.c_int64]
        L.oracle_normwise_error.restype = ctypes.c_double
        L.oracle_group_sum.argtypes = [ctypes.POINTER(_dp), ctypes.c_int, ctypes.c_int64, _dp]
        I64 = ctypes.POINTER(ctypes.c_int64)
        L.oracle_copy_box.argtypes = [ctypes.c_int, _dp, I64, _dp, I64, I64, I64, I64]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libeinplan_ref.so"))


def ref():
    """The reference einplan library (oracle/_ref), or raise if not built."""
    global _ref
    if _ref is None:
        path = os.path.join(HERE, "_ref", "libeinplan_ref.so")
        if not os.path.exists(path):
            raise FileNotFoundError(path + " (run oracle.build() where /root/reference exists)")
        R = ctypes.CDLL(path)
        R.ref_random_fill.argtypes = [_dp, ctypes.c_int64, ctypes.c_uint64]
        R.ref_plan_json.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int64,
                                    ctypes.c_double, ctypes.c_int]
        R.ref_plan_json.restype = ctypes.c_void_p
        R.ref_free.argtypes = [ctypes.c_void_p]
        R.ref_last_error.restype = ctypes.c_char_p
        R.ref_naive_evaluate.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(_dp), _dp]
        R.ref_run.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int64, ctypes.c_double,
                              ctypes.POINTER(_dp), _dp, ctypes.POINTER(ctypes.c_double),
                              ctypes.POINTER(ctypes.c_int64)]
        _ref = R
    return _ref


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


# ---------------------------------------------------------------- einsum ----
def parse(einsum: str):
    s = einsum.replace(" ", "")
    lhs, out = s.split("->")
    return lhs.split(","), out


def symbols(einsum: str):
    ins, out = parse(einsum)
    seen = []
    for t in ins + [out]:
        for c in t:
            if c not in seen:
                seen.append(c)
    return seen


def dims_string(extents: dict) -> str:
    return ",".join(f"{k}={v}" for k, v in extents.items())


def shape_of(indices: str, extents: dict):
    return tuple(int(extents[c]) for c in indices)


def random_tensor(shape, seed: int, skip: int = 0) -> np.ndarray:
    """Reference random_tensor(shape, seed) (tensor.cpp:55-63)."""
    n = int(np.prod(shape)) if len(shape) else 1
    out = np.empty(n, dtype=np.float64)
    lib().oracle_random_fill(_ptr(out), n, seed, skip)
    return out.reshape(shape)


def seeded_inputs(einsum: str, extents: dict, seed: int):
    """Operands as einplan_run_json makes them: seed + operand index
    (capi.cpp:206-208)."""
    ins, _ = parse(einsum)
    return [random_tensor(shape_of(t, extents), seed + k) for k, t in enumerate(ins)]


def naive_evaluate(einsum: str, extents: dict, operands) -> np.ndarray:
    """Restated naive_evaluate (evaluate.cpp:7-63)."""
    ins, out = parse(einsum)
    ext = (ctypes.c_int64 * 256)()
    for k, v in extents.items():
        ext[ord(k)] = int(v)
    ops = [np.ascontiguousarray(o, dtype=np.float64) for o in operands]
    for t, o in zip(ins, ops):
        assert o.shape == shape_of(t, extents), (t, o.shape)
    arr = (_dp * len(ops))(*[_ptr(o) for o in ops])
    res = np.empty(shape_of(out, extents), dtype=np.float64)
    rc = lib().oracle_naive_evaluate(einsum.replace(" ", "").encode(), ext, arr, _ptr(res))
    if rc:
        raise ValueError("oracle_naive_evaluate rejected " + einsum)
    return res


def max_rel_error(got, want) -> float:
    g = np.ascontiguousarray(got, dtype=np.float64).ravel()
    w = np.ascontiguousarray(want, dtype=np.float64).ravel()
    assert g.size == w.size
    return lib().oracle_max_rel_error(_ptr(g), _ptr(w), g.size)


def normwise_error(got, want) -> float:
    g = np.ascontiguousarray(got, dtype=np.float64).ravel()
    w = np.ascontiguousarray(want, dtype=np.float64).ravel()
    assert g.size == w.size
    return lib().oracle_normwise_error(_ptr(g), _ptr(w), g.size)


def group_sum(members) -> np.ndarray:
    ms = [np.ascontiguousarray(m, dtype=np.float64).ravel() for m in members]
    acc = np.empty_like(ms[0])
    arr = (_dp * len(ms))(*[_ptr(m) for m in ms])
    lib().oracle_group_sum(arr, len(ms), acc.size, _ptr(acc))
    return acc.reshape(np.shape(members[0]))


# ------------------------------------------------------------- reference ----
def ref_plan_json(einsum: str, extents: dict, procs: int, fast_mem: float = 1024.0,
                  include_messages: bool = False) -> str:
    R = ref()
    p = R.ref_plan_json(einsum.encode(), dims_string(extents).encode(), procs, fast_mem,
                        int(include_messages))
    if not p:
        raise RuntimeError(R.ref_last_error().decode())
    try:
        return ctypes.string_at(p).decode()
    finally:
        R.ref_free(p)


def ref_naive_evaluate(einsum: str, extents: dict, operands) -> np.ndarray:
    R = ref()
    ins, out = parse(einsum)
    ops = [np.ascontiguousarray(o, dtype=np.float64) for o in operands]
    arr = (_dp * len(ops))(*[_ptr(o) for o in ops])
    res = np.empty(shape_of(out, extents), dtype=np.float64)
    if R.ref_naive_evaluate(einsum.encode(), dims_string(extents).encode(), arr, _ptr(res)):
        raise RuntimeError(R.ref_last_error().decode())
    return res


def ref_run(einsum: str, extents: dict, procs: int, operands, fast_mem: float = 1024.0):
    """Reference make_pipeline + run() (executor.cpp:156-263), verify off.
    Returns (output, run_seconds, (allreduce_vol, redistribute_vol, max_rank_sent))."""
    R = ref()
    ins, out = parse(einsum)
    ops = [np.ascontiguousarray(o, dtype=np.float64) for o in operands]
    arr = (_dp * len(ops))(*[_ptr(o) for o in ops])
    res = np.empty(shape_of(out, extents), dtype=np.float64)
    secs = ctypes.c_double(0.0)
    comm = (ctypes.c_int64 * 3)()
    if R.ref_run(einsum.encode(), dims_string(extents).encode(), procs, fast_mem, arr,
                 _ptr(res), ctypes.byref(secs), comm):
        raise RuntimeError(R.ref_last_error().decode())
    return res, secs.value, (comm[0], comm[1], comm[2])


def ref_run_json(einsum: str, extents: dict, procs: int, fast_mem: float = 1024.0,
                 seed: int = 0, verify: bool = True):
    """The reference's own C ABI einplan_run_json (capi.cpp:169-226)."""
    R = ref()
    R.einplan_session_create.argtypes = [ctypes.c_char_p, ctypes.c_char_p,
                                         ctypes.POINTER(ctypes.c_void_p)]
    R.einplan_run_json.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_double,
                                   ctypes.c_uint64, ctypes.c_int, ctypes.c_char_p,
                                   ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
    R.einplan_free.argtypes = [ctypes.c_void_p]
    R.einplan_session_destroy.argtypes = [ctypes.c_void_p]
    R.einplan_last_error.restype = ctypes.c_char_p
    s = ctypes.c_void_p()
    if R.einplan_session_create(einsum.encode(), dims_string(extents).encode(), ctypes.byref(s)):
        raise RuntimeError(R.einplan_last_error().decode())
    p = ctypes.c_void_p()
    st = R.einplan_run_json(s, procs, fast_mem, seed, int(verify), None, None, ctypes.byref(p))
    try:
        if not p:
            raise RuntimeError(R.einplan_last_error().decode())
        return st, ctypes.string_at(p).decode()
    finally:
        if p:
            R.einplan_free(p)
        R.einplan_session_destroy(s)
