"""B200-native Deinsum hot path (einplan interface).

The reference ("einplan", a C++ planner + virtual executor) is reached
through its C ABI (``einplan.h``) and its C++ host API.  This package mirrors
that interface for Python callers:

* :class:`Session` — ``einplan_session_*`` / ``einplan_{bound,plan,run}_json``
  (reference proj/src/capi.cpp:111-226) with ``run_json`` executing on the GPU;
* :func:`bench_json` — ``einplan_bench_json`` (capi.cpp:228-254);
* :class:`Executor` — the rank-local GPU executor (``eb_exec_*``): stage
  inputs once, run the schedule repeatedly with data resident in HBM, gather;
  one process per GPU over NCCL when ``rank >= 0``, or over peer memory
  (CUDA IPC, ``transport="peer"``);
* :func:`set_option` — the path options (``eb_set_option``);
* :class:`RandomStream` — the reference input stream, consumed in order;
* :func:`plan_json`, :func:`random_tensor` — host-only helpers.

Compute happens only in ``lib/libeinplan_b200.so`` (sm_100a kernels).  There
is no CPU fallback: without the library every call raises.
"""
from __future__ import annotations

import ctypes
from typing import Mapping, Sequence

import numpy as np

from . import _capi
from ._capi import EinplanError

__all__ = ["Session", "Executor", "EinplanError", "RandomStream", "bench_json", "plan_json",
           "launch_count",
           "random_tensor", "set_option", "version", "dims_string"]


def version() -> str:
    return _capi.lib().einplan_version().decode()


def dims_string(dims) -> str:
    if isinstance(dims, str):
        return dims
    return ",".join(f"{k}={int(v)}" for k, v in dims.items())


def _outer(status: int):
    if status != 0:
        raise EinplanError(status, _capi.lib().einplan_last_error().decode())


class Session:
    """einplan_session: an einsum with bound extents (capi.cpp:111-133)."""

    def __init__(self, einsum: str, dims):
        L = _capi.lib()
        self._h = ctypes.c_void_p()
        _outer(L.einplan_session_create(einsum.encode(), dims_string(dims).encode(),
                                        ctypes.byref(self._h)))
        self.einsum = einsum

    def close(self):
        if self._h:
            _capi.lib().einplan_session_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def bound_json(self, fast_mem: float = 1024.0) -> str:
        p = ctypes.c_void_p()
        _outer(_capi.lib().einplan_bound_json(self._h, fast_mem, ctypes.byref(p)))
        return _capi.take_string(p)

    def plan_json(self, procs: int, fast_mem: float = 1024.0, include_messages=False) -> str:
        p = ctypes.c_void_p()
        _outer(_capi.lib().einplan_plan_json(self._h, procs, fast_mem, int(include_messages),
                                             ctypes.byref(p)))
        return _capi.take_string(p)

    def run_json(self, procs: int, fast_mem: float = 1024.0, seed: int = 0, verify=True,
                 input_paths: str | None = None, dump_output: str | None = None):
        """Returns (status, report); status EINPLAN_E_VERIFY still carries a report."""
        p = ctypes.c_void_p()
        st = _capi.lib().einplan_run_json(
            self._h, procs, fast_mem, seed, int(verify),
            input_paths.encode() if input_paths else None,
            dump_output.encode() if dump_output else None, ctypes.byref(p))
        if st not in (0, _capi.EINPLAN_E_VERIFY):
            _outer(st)
        return st, _capi.take_string(p)


def cp3_als_sweep(X, A, B, C, stream=None, workspace=None):
    """One CP-ALS sweep (eb_cp3_als_sweep) on torch CUDA tensors: X [I][J][K],
    factors [n][R], float64, contiguous; A, B, C are updated in place.
    Returns the workspace tensor (reuse it across sweeps)."""
    import torch
    I, J, K = X.shape
    R = A.shape[1]
    L = _capi.lib()
    nb = L.eb_cp3_als_workspace(I, J, K, R)
    if nb == 0:
        raise EinplanError(_capi.EINPLAN_E_INVALID, L.eb_last_error().decode())
    if workspace is None or workspace.numel() < nb:
        workspace = torch.empty(nb, dtype=torch.uint8, device=X.device)
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    _capi.check(L.eb_cp3_als_sweep(X.data_ptr(), I, J, K, R, A.data_ptr(), B.data_ptr(),
                                   C.data_ptr(), workspace.data_ptr(), nb, s))
    return workspace


def set_option(name: str, value) -> None:
    """Path options of the kernel layer (eb_set_option): "no_fused_tma",
    "no_rf", "rf_cfg" ("RTxOS" / "auto"), "ttm2_variant" (0/1/2), "fuse_ttm2".
    Read once from the EB_* environment at load; change them between runs."""
    _capi.check(_capi.lib().eb_set_option(name.encode(), str(value).encode()))


class RandomStream:
    """random_tensor's mt19937_64 stream (tensor.cpp:55-63) consumed in order:
    successive :meth:`fill` calls continue where the last one stopped."""

    def __init__(self, seed: int, skip: int = 0):
        self._h = ctypes.c_void_p()
        _capi.check(_capi.lib().eb_rng_create(seed, skip, ctypes.byref(self._h)))

    def fill(self, out: np.ndarray) -> np.ndarray:
        if out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ValueError("RandomStream.fill: out must be a contiguous float64 array")
        _capi.lib().eb_rng_fill(self._h, out.ctypes.data_as(_capi._dp), out.size)
        return out

    def close(self):
        if self._h:
            _capi.lib().eb_rng_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def launch_count() -> int:
    """Kernel launches issued by the library so far (graph replays add the
    launches of their captured run)."""
    return int(_capi.lib().eb_launch_count())


def mem_in_use() -> int:
    """Bytes in use in the current device's stream-ordered pool (eb_mem_in_use)."""
    v = ctypes.c_int64(0)
    _capi.check(_capi.lib().eb_mem_in_use(ctypes.byref(v)))
    return v.value


def _operand_shapes(einsum: str, dims) -> list:
    ins = einsum.replace(" ", "").split("->")[0].split(",")
    d = dict(dims) if not isinstance(dims, str) else {
        kv.split("=")[0]: int(kv.split("=")[1]) for kv in dims.split(",") if kv}
    return [tuple(int(d[c]) for c in t) for t in ins]


def random_block(seed: int, gshape, base, shape, out: np.ndarray | None = None) -> np.ndarray:
    """The box [base, base+shape) of random_tensor(gshape, seed), generated
    without materialising the global tensor (into `out` when given, e.g. a
    pinned buffer)."""
    nd = len(gshape)
    n = int(np.prod(shape))
    if out is None:
        out = np.empty(n, dtype=np.float64)
    out = out.reshape(-1)
    if out.size != n or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError("random_block: out must be a contiguous float64 array of the box size")
    arr = lambda v: (ctypes.c_int64 * nd)(*[int(x) for x in v])
    _capi.check(_capi.lib().eb_random_fill_block(out.ctypes.data_as(_capi._dp), seed, nd,
                                                 arr(gshape), arr(base), arr(shape)))
    return out.reshape([int(x) for x in shape])


def bench_json(scale: float, procs: int, fast_mem: float = 1024.0, seed: int = 1):
    p = ctypes.c_void_p()
    st = _capi.lib().einplan_bench_json(scale, procs, fast_mem, seed, ctypes.byref(p))
    if st not in (0, _capi.EINPLAN_E_VERIFY):
        _outer(st)
    return st, _capi.take_string(p)


def plan_json(einsum: str, dims, procs: int, fast_mem: float = 1024.0,
              include_messages=False) -> str:
    """Host-only make_pipeline + plan_report (no GPU needed)."""
    L = _capi.lib()
    p = ctypes.c_void_p()
    _capi.check(L.eb_plan_json(einsum.encode(), dims_string(dims).encode(), procs, fast_mem,
                               int(include_messages), ctypes.byref(p)))
    return _capi.take_string(p, L.eb_free)


def random_tensor(shape: Sequence[int], seed: int) -> np.ndarray:
    """random_tensor(shape, seed) (tensor.cpp:55-63), generated by the library."""
    n = int(np.prod(shape)) if len(shape) else 1
    out = np.empty(n, dtype=np.float64)
    _capi.lib().eb_random_fill_host(out.ctypes.data_as(_capi._dp), n, seed, 0)
    return out.reshape(tuple(shape))


class Executor:
    """Rank-local GPU executor of an einplan schedule (eb_exec_*).

    ``rank=-1``: all ``procs`` ranks virtual on the current device.
    ``rank>=0``: this process is one rank; ``transport="nccl"`` (default)
    takes ``nccl_id`` (128 bytes) from :meth:`nccl_unique_id` on rank 0;
    ``transport="peer"`` meets the other ranks' processes in the POSIX
    shared-memory segment ``group`` (e.g. "/eb_job42") and exchanges over
    CUDA IPC peer memory — several processes may share one GPU;
    ``transport="hybrid"`` (one GPU per process) is the peer transport with
    its allreduces on NCCL (needs both ``group`` and ``nccl_id``).
    """

    def __init__(self, einsum: str, dims, procs: int = 1, fast_mem: float = 1024.0,
                 rank: int = -1, nccl_id: bytes | None = None, stream: int | None = None,
                 like: "Executor | None" = None, transport: str = "nccl",
                 group: str | None = None):
        """``like=other``: same ranks and the same transport (communicator,
        communication stream) as ``other``."""
        L = _capi.lib()
        self._h = ctypes.c_void_p()
        if like is not None:
            _capi.check(L.eb_exec_create_like(einsum.encode(), dims_string(dims).encode(),
                                              fast_mem, like._h, ctypes.c_void_p(stream or 0),
                                              ctypes.byref(self._h)))
            procs, rank = like.procs, like.rank
            self._peer = like
        elif rank >= 0 and transport == "peer":
            if not group:
                raise ValueError("Executor(transport='peer') needs a group name")
            _capi.check(L.eb_exec_create_peer(einsum.encode(), dims_string(dims).encode(), procs,
                                              fast_mem, rank, group.encode(),
                                              ctypes.c_void_p(stream or 0), ctypes.byref(self._h)))
        elif rank >= 0 and transport == "hybrid":
            if not group or nccl_id is None:
                raise ValueError("Executor(transport='hybrid') needs a group name and an nccl_id")
            idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            _capi.check(L.eb_exec_create_hybrid(einsum.encode(), dims_string(dims).encode(),
                                                procs, fast_mem, rank, group.encode(), idbuf,
                                                ctypes.c_void_p(stream or 0),
                                                ctypes.byref(self._h)))
        else:
            if transport not in ("nccl", "peer", "hybrid"):
                raise ValueError(f"unknown transport {transport!r}")
            idbuf = (ctypes.create_string_buffer(bytes(nccl_id), 128)
                     if nccl_id is not None else None)
            _capi.check(L.eb_exec_create(einsum.encode(), dims_string(dims).encode(), procs,
                                         fast_mem, rank, idbuf, ctypes.c_void_p(stream or 0),
                                         ctypes.byref(self._h)))
        self.einsum, self.procs, self.rank = einsum, procs, rank
        self.extents = dict(dims) if not isinstance(dims, str) else dims
        self._shapes = _operand_shapes(einsum, dims)
        self._keep = None

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _capi.check(_capi.lib().eb_nccl_unique_id(buf))
        return buf.raw

    def close(self):
        if self._h:
            _capi.lib().eb_exec_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stage(self, inputs: Sequence[np.ndarray | None]):
        """Copy host operands to this process's device blocks; ``None`` keeps an
        operand's device contents (e.g. one shared with :meth:`share_input`)."""
        if len(inputs) != len(self._shapes):
            raise ValueError(f"stage: {len(self._shapes)} operands expected, got {len(inputs)}")
        arrs = []
        for k, a in enumerate(inputs):
            if a is None:
                arrs.append(None)
                continue
            a = np.ascontiguousarray(a, dtype=np.float64)
            if a.size != int(np.prod(self._shapes[k])) or (
                    a.ndim > 1 and tuple(a.shape) != self._shapes[k]):
                raise ValueError(f"stage: operand {k} has shape {a.shape}, "
                                 f"expected {self._shapes[k]}")
            arrs.append(a)
        ptrs = (_capi._dp * len(arrs))(*[None if a is None else a.ctypes.data_as(_capi._dp)
                                          for a in arrs])
        _capi.check(_capi.lib().eb_exec_stage(self._h, ptrs))
        self._keep = arrs  # the copies are asynchronous: keep the sources alive

    def block(self, k: int):
        """(base, shape) of operand k's box on this process's rank."""
        base, shape = (ctypes.c_int64 * 16)(), (ctypes.c_int64 * 16)()
        nd = ctypes.c_int(0)
        _capi.check(_capi.lib().eb_exec_block(self._h, k, base, shape, ctypes.byref(nd)))
        return list(base[:nd.value]), list(shape[:nd.value])

    def stage_block(self, k: int, block: np.ndarray):
        """Stage operand k from a host array holding just this rank's box."""
        _, shape = self.block(k)
        a = np.ascontiguousarray(block, dtype=np.float64)
        if a.size != int(np.prod(shape)):
            raise ValueError(f"stage_block: operand {k} box has {int(np.prod(shape))} elements, "
                             f"got {a.size}")
        _capi.check(_capi.lib().eb_exec_stage_block(self._h, k, a.ctypes.data_as(_capi._dp)))
        self._keep_blocks = getattr(self, "_keep_blocks", {})
        self._keep_blocks[k] = a  # asynchronous copy: keep the source alive

    def stage_region(self, k: int, base, region: np.ndarray) -> int:
        """Virtual ranks: stage operand k's blocks that lie inside the global
        sub-box [base, base + region.shape) from ``region`` (no global tensor
        on the host).  Returns how many blocks were staged.  Synchronous."""
        a = np.ascontiguousarray(region, dtype=np.float64)
        nd = a.ndim
        if nd != len(self._shapes[k]) or len(base) != nd:
            raise ValueError("stage_region: region rank differs from the operand's")
        arr = lambda v: (ctypes.c_int64 * nd)(*[int(x) for x in v])
        n = ctypes.c_int(0)
        _capi.check(_capi.lib().eb_exec_stage_region(self._h, k, arr(base), arr(a.shape), nd,
                                                     a.ctypes.data_as(_capi._dp),
                                                     ctypes.byref(n)))
        import torch  # the copies read `a`: finish them before it may go away
        torch.cuda.synchronize()
        return n.value

    def share_input(self, k: int, src: "Executor", k_src: int):
        """Use ``src``'s staged device blocks for operand ``k`` (no copy)."""
        _capi.check(_capi.lib().eb_exec_share_input(self._h, k, src._h, k_src))
        self._shared_from = getattr(self, "_shared_from", []) + [src]

    def run(self):
        _capi.check(_capi.lib().eb_exec_run(self._h))

    def set_async_reduce(self, on: bool = True):
        """Issue this executor's allreduces on a side stream (see join)."""
        _capi.check(_capi.lib().eb_exec_set_async_reduce(self._h, int(on)))

    def join(self):
        """Order the compute stream after this executor's pending reduction."""
        _capi.check(_capi.lib().eb_exec_join(self._h))

    def capture(self):
        """Capture one run as a CUDA graph (after a warm eager run); then
        :meth:`replay` launches it.  Virtual / NCCL transports only."""
        _capi.check(_capi.lib().eb_exec_capture(self._h))

    def replay(self):
        """Launch the captured run (same kernels and collectives, one host call)."""
        _capi.check(_capi.lib().eb_exec_replay(self._h))

    def run_pair(self, mode1: "Executor") -> bool:
        """CP-sweep dimension tree: this executor (order-3 mode 0) and ``mode1``
        (mode 1 over the same shared X and k factor) in one pass over X.
        Returns whether the fused path ran (else both ran separately)."""
        fused = ctypes.c_int(0)
        _capi.check(_capi.lib().eb_exec_run_pair(self._h, mode1._h, ctypes.byref(fused)))
        return bool(fused.value)

    def output_elems(self) -> int:
        return int(_capi.lib().eb_exec_output_elems(self._h))

    def gather(self, out: np.ndarray | None = None) -> np.ndarray | None:
        """The output on rank 0 (or in virtual mode); other ranks of a process
        group take part (the call is collective) and get None."""
        n = self.output_elems()
        if self.rank > 0:
            _capi.check(_capi.lib().eb_exec_gather(self._h, None))
            return None
        if out is None:
            out = np.empty(n, dtype=np.float64)
        if out.dtype != np.float64 or not out.flags.c_contiguous or out.size != n:
            raise ValueError(f"gather: out must be a C-contiguous float64 array of {n} elements")
        _capi.check(_capi.lib().eb_exec_gather(self._h, out.ctypes.data_as(_capi._dp)))
        return out

    def stats(self) -> dict:
        v = (ctypes.c_int64 * 8)()
        _capi.check(_capi.lib().eb_exec_stats(self._h, v))
        keys = ["allreduce_volume", "redistribute_volume", "max_rank_sent", "fused_launches",
                "ttm_launches", "generic_launches", "tree_flops", "terms"]
        d = dict(zip(keys, list(v)))
        d["fused_redistributions"] = int(_capi.lib().eb_exec_fused_redistributions(self._h))
        return d

    def report_json(self, out: np.ndarray | None = None) -> str:
        p = ctypes.c_void_p()
        ptr = out.ctypes.data_as(_capi._dp) if out is not None else None
        _capi.check(_capi.lib().eb_exec_report_json(self._h, ptr, ctypes.byref(p)))
        return _capi.take_string(p, _capi.lib().eb_free)
