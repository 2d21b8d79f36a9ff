#!/usr/bin/env python
"""Benchmark of the B200 Deinsum hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl b200|reference]

Workload (default C2 = BASELINE configs[1], the config the metric is quoted
on that fits one GPU): the order-3 CP-ALS MTTKRP sweep — mode-0, mode-1 and
mode-2 MTTKRP of a dense fp64 1024^3 tensor with 1024x32 factors — each mode
planned by the reference's pipeline (make_pipeline, S = 1024) on the
processor grid for N ranks and executed by the GPU executor.  One step = the
three modes.  N > 1 runs one process per GPU (torchrun), each rank the
reference grid's rank r, partial outputs summed by NCCL allreduce on
ncclCommSplit sub-communicators; the JSON line is printed by rank 0 with the
max-over-ranks device time.

`value` (device-timed, inputs resident in HBM) = reference tree flops of the
step / time.  `e2e` = the same metric through the C ABI with host buffers
(pinned at N = 1): per mode eb_exec_stage (H2D) + eb_exec_run + eb_exec_gather
(D2H), wall clock with device syncs on both sides.  `--impl reference` times
the reference implementation itself (oracle/_ref, compiled from the
reference's sources) on the host cores.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASELINE["metric"]
FP64_PEAK_TFLOPS = 37.05   # measured DMMA.8x8x4 peak on this pool's B200 (profiles/fp64_peak_r01.jsonl)
FP64_PEAK_CLOCK_MHZ = 1965  # the SM clock that peak was measured at (same file, first line)
HBM_READ_GBS = 7182.5      # measured read-only stream (same file)


def _load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))
    except Exception:
        return {"hbm_gbs": 6650.0, "_source": "fallback (B200_PROFILING.md)"}


# --------------------------------------------------------------- configs --

def workload(name: str, P: int):
    """(label, [(einsum, extents, input-builder)], scaling, l2_note)."""
    from tests.configs import CONFIGS, C2_FACTOR_SEED
    import paper_2206_08301_b200 as eb
    c = CONFIGS[name]
    ext = c["extents"](P)

    def seeded_builder(e, shared_seed=None):
        ins, _ = e.split("->")[0].split(","), None

        def build(pinned, skip_x=False, ex=None):
            """Host operands: global tensors, or (ex given: one process per
            GPU) just the boxes this rank holds — no rank materialises the
            global X (C5 at P = 8: 69 GB)."""
            out = []
            for k, t in enumerate(ins):
                if k == 0 and skip_x:
                    out.append(None)
                    continue
                shape = tuple(ext[s] for s in t)
                seed = k if shared_seed is None else (0 if k == 0 else C2_FACTOR_SEED[t[0]])
                if ex is not None:
                    base, bshape = ex.block(k)
                    buf = _host_buffer(int(np.prod(bshape)), pinned and k == 0)
                    out.append(eb.random_block(seed, shape, base, bshape, out=buf))
                else:
                    out.append(_fill(shape, seed, pinned and k == 0))
            return out
        return build

    modes = []
    for e in c["einsums"]:
        modes.append((e, ext, seeded_builder(e, shared_seed=(True if name == "C2" else None))))
    label = {
        "C1": "C1: order-3 MTTKRP mode-0, X 512^3, R=24",
        "C2": "C2: order-3 CP-ALS MTTKRP sweep (modes 0,1,2), X 1024^3 fp64, factors 1024x32",
        "C3": "C3: order-5 MTTKRP mode-0, X 64^5, R=24",
        "C4": "C4: order-3 TTMc mode-0, X 1024^3, U1/U2 1024x64 (binary chain)",
        "C5": "C5: order-5 TTMc mode-0, X (64P)x64^4, factors 64x16 (weak scaling)",
    }[name]
    scaling = "weak" if name == "C5" else "strong"
    return label, modes, scaling


_pinned_keep = []


def _host_buffer(n, pinned):
    if pinned:
        import torch
        t = torch.empty(n, dtype=torch.float64, pin_memory=True)
        _pinned_keep.append(t)
        return t.numpy()
    return np.empty(n, dtype=np.float64)


def _fill(shape, seed, pinned):
    import paper_2206_08301_b200 as eb
    from paper_2206_08301_b200 import _capi
    n = int(np.prod(shape))
    if pinned:
        import torch
        t = torch.empty(n, dtype=torch.float64, pin_memory=True)
        _pinned_keep.append(t)
        arr = t.numpy()
    else:
        arr = np.empty(n, dtype=np.float64)
    _capi.lib().eb_random_fill_host(arr.ctypes.data_as(_capi._dp), n, seed, 0)
    return arr.reshape(shape)


# ---------------------------------------------------------------- clocks --

class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML
    polled every 2 ms from a thread (the timed region of a default run is only
    tens of ms), with `nvidia-smi -lms 200` as the fallback."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.thread = None
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self.path = tempfile.mktemp(suffix=".csv")
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None

    def _poll(self):
        n = self.nvml
        while not self.stop_flag:
            try:
                self.samples.append(n.nvmlDeviceGetClockInfo(self.handle, n.NVML_CLOCK_SM))
                r = n.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        if self.nvml is not None:
            self.stop_flag = False
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-i", str(self.index), "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.thread is not None:
            self.stop_flag = True
            self.thread.join()
            return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                    "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": len(self.samples), "source": "nvml, 2 ms polling"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi -lms 200"}


# ------------------------------------------------------- reference arm --

# i-rows of X per reference run() in the CPU samples (a few seconds of
# single-threaded reference work each).  Every config's mode-0 output (and
# C2's sweep) is a sum over independent i-slabs of X, so a slab of the REAL
# seed-0 tensor is an exact, proportionally smaller piece of the same
# computation: mode-0 outputs are the slab's output rows, the C2 mode-1 /
# mode-2 outputs are sums of the slabs' partial outputs.
REF_SLAB_ROWS = {"C1": 16, "C2": 8, "C3": 1, "C4": 4, "C5": 1}


class RefWorkload:
    """The config's real inputs (seed-0 X, the config's factor seeds — the
    same tensors the GPU arm stages) cut into i-slabs that successive reference
    steps rotate through; the slab outputs are reassembled and, once every row
    was covered, checked against the reference's own full-size goldens."""

    def __init__(self, config: str):
        import oracle
        from tests.configs import CONFIGS
        c = CONFIGS[config]
        self.config = config
        self.ext = dict(c["extents"](1))
        self.einsums = c["einsums"]
        xin = self.einsums[0].split("->")[0].split(",")[0]
        self.I = self.ext["i"]
        self.X = oracle.random_tensor(oracle.shape_of(xin, self.ext), 0)
        self.factors = []  # per mode: full factor operands
        self.flops_per_row = 0
        for e in self.einsums:
            ins, _ = oracle.parse(e)
            if config == "C2":
                from tests.configs import C2_FACTOR_SEED
                fs = [oracle.random_tensor(oracle.shape_of(t, self.ext), C2_FACTOR_SEED[t[0]])
                      for t in ins[1:]]
            else:
                fs = [oracle.random_tensor(oracle.shape_of(t, self.ext), k + 1)
                      for k, t in enumerate(ins[1:])]
            self.factors.append(fs)
            self.flops_per_row += json.loads(oracle.ref_plan_json(e, self.ext, 1))["tree"][
                "total_flops"] / self.I
        self.out = [None] * len(self.einsums)
        self.covered = np.zeros(self.I, dtype=bool)

    def slab_ops(self, mode, i0, rows):
        """Operands of mode `mode` restricted to X[i0:i0+rows] (factors indexed
        by i sliced alike)."""
        import oracle
        e = self.einsums[mode]
        ins, _ = oracle.parse(e)
        ops = [self.X[i0:i0 + rows]]
        for t, f in zip(ins[1:], self.factors[mode]):
            ops.append(np.ascontiguousarray(f[i0:i0 + rows]) if t[0] == "i" else f)
        ext = dict(self.ext, i=rows)
        return e, ext, ops

    def absorb(self, mode, i0, rows, out):
        e = self.einsums[mode]
        full_shape = tuple(self.ext[c] for c in e.split("->")[1])
        if self.out[mode] is None:
            self.out[mode] = np.zeros(full_shape)
        if e.split("->")[1][0] == "i":
            self.out[mode][i0:i0 + rows] = out
        else:  # C2 modes 1 / 2: the slab's partial sum
            self.out[mode] += out
        self.covered[i0:i0 + rows] = True

    def check(self):
        """Normwise error of the reassembled outputs against the reference's
        goldens (None until every i-row has been covered)."""
        if not self.covered.all():
            return None
        import oracle
        errs = []
        for mode, out in enumerate(self.out):
            tag = f"C2_m{mode}" if self.config == "C2" else self.config
            g = json.load(open(os.path.join(ROOT, "tests", "golden", f"{tag}_summary.json")))
            idx = np.array(g["sample_index"])
            errs.append(oracle.normwise_error(out.ravel()[idx], np.array(g["sample_value"])))
        return max(errs)


def _ref_sample_step(threads: int, rows: int, wl: "RefWorkload", step: int):
    """One bounded sample of the config on the reference implementation:
    `threads` concurrent reference run() calls (P = 1), each on the next slab
    of `rows` i-rows of the real X (C2: all three modes); steps rotate over
    the slabs.  Returns (flops, seconds)."""
    import oracle
    nslab = wl.I // rows
    work = []
    for t in range(threads):
        i0 = ((step * threads + t) % nslab) * rows
        work.append([(m, i0, wl.slab_ops(m, i0, rows)) for m in range(len(wl.einsums))])
    flops = wl.flops_per_row * rows * threads
    results = [[None] * len(wl.einsums) for _ in range(threads)]

    def body(t):
        for m, i0, (e, ext, ops) in work[t]:
            results[t][m] = oracle.ref_run(e, ext, 1, ops)[0]
    ths = [threading.Thread(target=body, args=(t,)) for t in range(threads)]
    t0 = time.perf_counter()
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    dt = time.perf_counter() - t0
    for t in range(threads):
        for m, i0, _ in work[t]:
            wl.absorb(m, i0, rows, results[t][m])
    return flops, dt


def cpu_kind():
    import oracle
    return "reference" if oracle.ref_available() else "port"


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    import oracle
    if not oracle.ref_available():
        oracle.build(ref=True)
    cores = os.cpu_count() or 1
    threads = max(1, min(cores, 32))
    rows = REF_SLAB_ROWS[args.config]
    wl = RefWorkload(args.config)
    step = 0
    for _ in range(args.warmup):
        _ref_sample_step(threads, rows, wl, step)
        step += 1
    tot_f, tot_s = 0, 0.0
    for _ in range(args.steps):
        f, s = _ref_sample_step(threads, rows, wl, step)
        step += 1
        tot_f += f
        tot_s += s
    err = wl.check()
    value = tot_f / tot_s / 1e9
    sample = (f"{args.config} sample per step: {threads} concurrent reference run() calls (P=1, "
              f"single-threaded each, oracle/_ref built from the reference sources), each on the "
              f"next {rows}-row i-slab of the config's own seed-0 X"
              f"{' (all 3 modes)' if args.config == 'C2' else ''}, slabs rotating over all "
              f"{wl.I} rows; GFLOP/s = reference tree flops / wall time")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot_s / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: the same seed-0 X and factor streams as the B200 arm "
                "(reference random_tensor, mt19937_64)",
        "config": {"workload": workload_label(args.config), "sample_rows_per_thread": rows,
                   "threads": threads, "same_inputs_as_b200_arm": True,
                   "rows_covered": int(wl.covered.sum()), "rows_total": wl.I},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": threads,
                         "kind": cpu_kind(), "sample": sample},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        # reassembled slab outputs vs the reference's full-size goldens (sampled
        # elements, normwise); null if the timed steps did not cover every row
        "reassembled_vs_golden": err,
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_label(name):
    return {
        "C1": "C1: order-3 MTTKRP mode-0, X 512^3, R=24",
        "C2": "C2: order-3 CP-ALS MTTKRP sweep (modes 0,1,2), X 1024^3 fp64, factors 1024x32",
        "C3": "C3: order-5 MTTKRP mode-0, X 64^5, R=24",
        "C4": "C4: order-3 TTMc mode-0, X 1024^3, U1/U2 1024x64 (binary chain)",
        "C5": "C5: order-5 TTMc mode-0, X (64P)x64^4, factors 64x16 (weak scaling)",
    }.get(name, name)


CPU_LEG_ROWS = {"C1": 64, "C2": 16, "C3": 1, "C4": 8, "C5": 1}


def cpu_baseline_leg(config="C2"):
    """Rank 0, N = 1: the reference (or the oracle port) on a bounded sample
    of the same inputs, single-threaded as the reference is (README.md:149-150)."""
    import oracle
    if not oracle.ref_available():
        try:
            oracle.build(ref=True)
        except Exception:
            pass
    if oracle.ref_available():
        rows = CPU_LEG_ROWS[config]
        wl = RefWorkload(config)
        f, s = _ref_sample_step(1, rows, wl, 0)
        what = "sweep (3 modes)" if config == "C2" else "run"
        return {"value": f / s / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": "reference",
                "sample": f"{config} {what} on X[0:{rows}] of the config's own seed-0 X, "
                          "reference run() at P=1, one host thread (the reference is "
                          f"single-threaded); {s:.1f} s of CPU work"}
    # Port: the C restatement on a smaller slab.
    ext = dict(i=4, j=1024, k=1024, a=32)
    t0 = time.perf_counter()
    fl = 0
    for e in ("ijk,ja,ka->ia", "ijk,ia,ka->ja", "ijk,ia,ja->ka"):
        ops = oracle.seeded_inputs(e, ext, 0)
        oracle.naive_evaluate(e, ext, ops)
        fl += 2 * 4 * 1024 * 1024 * 32
    s = time.perf_counter() - t0
    return {"value": fl / s / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": "port",
            "sample": "C2 sweep on X[0:4,:,:] with the C oracle (naive_evaluate restatement)"}


# --------------------------------------------------------------- B200 arm --

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip the secondary C1/C3/C4/C5 lines embedded in the default C2 run")
    ap.add_argument("--sweep", default="modes", choices=["modes", "dimtree"],
                    help="C2 only. modes: the reference's three einsums, one schedule each; "
                         "dimtree: modes 0 and 1 from one pass over X (T = X x_k C folded "
                         "into both outputs, eb_exec_run_pair), mode 2 as before — 2/3 of "
                         "the DMMA flops for the same three outputs")
    ap.add_argument("--transport", default="auto",
                    choices=["auto", "virtual", "nccl", "peer", "hybrid"],
                    help="auto: hybrid when WORLD_SIZE > 1 (one process per GPU: MTTKRP "
                         "allreduces on NCCL split communicators, TTMc redistributions fused "
                         "into the producing kernel over CUDA-IPC peer memory), else the "
                         "in-device virtual-rank transport; nccl: NCCL only (grouped "
                         "send/recv redistributions); peer: peer memory only")
    ap.add_argument("--share-gpu", action="store_true",
                    help="functional check of the N-rank path on fewer GPUs: ranks share the "
                         "visible devices (rank r on device r mod count), peer transport, gloo "
                         "for the timing plumbing — the numbers are NOT a multi-GPU measurement")
    args = ap.parse_args()
    if args.share_gpu:
        args.transport = "peer"
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "b200":
        return _self_launch(args.gpus, args.share_gpu)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU "
              f"(torchrun --nproc-per-node {args.gpus}) or drop --gpus", file=sys.stderr)
        return 2
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps

    import torch
    import torch.distributed as dist
    ndev = max(torch.cuda.device_count(), 1)
    dev = local % ndev if args.share_gpu else local
    torch.cuda.set_device(dev)
    if world > 1:
        if args.share_gpu:  # NCCL refuses two ranks on one GPU; gloo carries the plumbing
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    P = world
    import paper_2206_08301_b200 as eb
    from paper_2206_08301_b200 import _capi
    L = _capi.lib()

    label, modes, scaling = workload(args.config, P)
    dimtree = args.sweep == "dimtree"
    if dimtree and args.config != "C2":
        raise SystemExit("--sweep dimtree applies to the C2 CP-ALS sweep only")
    if dimtree:
        label += "; dimension tree: modes 0+1 in one pass over X (eb_exec_run_pair), mode 2 " \
                 "separately — same outputs, 2/3 of the DMMA flops"
    if args.transport == "auto" and world > 1:
        args.transport = "hybrid"
    peer = args.transport in ("peer", "hybrid")
    use_nccl = (world > 1 or args.transport == "nccl" or args.transport == "hybrid") and \
        args.transport != "peer"
    nccl_id, group = None, None
    if world > 1 and use_nccl:
        obj = [eb.Executor.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    elif use_nccl:
        nccl_id = eb.Executor.nccl_unique_id()
    if peer:
        import uuid
        obj = [f"/eb_bench_{uuid.uuid4().hex[:16]}" if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        group = obj[0]
    ranked = use_nccl or peer
    stream = torch.cuda.Stream()
    execs, inputs, grids, flops_tree = [], [], [], 0
    q_bound_total = 0.0  # SOAP I/O lower bound of every mode's partition (soap.cpp:359-425)
    x_shared = []  # per executor: is operand 0 (X) aliased to executor 0's blocks?
    # one process per GPU: stage only this rank's boxes (EB_BENCH_BLOCKS=1
    # forces it for a single NCCL rank, to exercise the path on one GPU)
    blockmode = world > 1 or (ranked and os.environ.get("EB_BENCH_BLOCKS") == "1")
    for mi, (e, ext, build) in enumerate(modes):
        if mi == 0:
            ex = eb.Executor(e, ext, P, 1024.0, rank if ranked else -1, nccl_id,
                             stream=stream.cuda_stream,
                             transport=args.transport if args.transport in ("peer", "hybrid")
                             else "nccl", group=group)
        else:  # same ranks / same NCCL communicator as mode 0
            ex = eb.Executor(e, ext, stream=stream.cuda_stream, like=execs[0])
        shared = False
        if mi > 0 and args.config == "C2":
            # the CP-ALS sweep: one X in HBM for the three modes (eb_exec_share_input)
            ins = build(pinned=False, skip_x=True, ex=ex if blockmode else None)
            ins[0] = inputs[0][0]
            ex.share_input(0, execs[0], 0)
            shared = True
            if dimtree and mi == 1:  # mode 1 also takes mode 0's C blocks (same tensor)
                ex.share_input(2, execs[0], 2)
        else:
            ins = build(pinned=(world == 1 or blockmode), ex=ex if blockmode else None)
        _stage(ex, ins, shared, dimtree and mi == 1, blockmode)
        # reductions on a side stream: mode m's allreduce overlaps mode m+1
        ex.set_async_reduce(True)
        execs.append(ex)
        inputs.append(ins)
        x_shared.append(shared)
        plan = json.loads(eb.plan_json(e, ext, P))
        grids.append([t["grid"] for t in plan["schedule"]["terms"]])
        q_bound_total += float(plan["partition"]["total_q"])
        flops_tree += plan["tree"]["total_flops"]
    torch.cuda.synchronize()

    def step():
        if dimtree:
            if not execs[0].run_pair(execs[1]):
                raise RuntimeError("dimension-tree pair did not qualify")
            execs[2].run()
        else:
            for ex in execs:
                ex.run()
        for ex in execs:  # the step ends when every reduction has landed
            ex.join()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    clocks = ClockSampler(dev if "CUDA_VISIBLE_DEVICES" not in os.environ else
                          int(os.environ["CUDA_VISIBLE_DEVICES"].split(",")[dev]))

    def timed(kernel_events):
        """K steps between a barrier + synchronize on both sides; device time
        of the whole region (CUDA events on the executors' stream).  With
        kernel_events the main contraction launches are also bracketed by
        their own events (eb_timer) — those records sit between programmatic-
        dependent launches and cost a few microseconds of overlap per launch,
        so `value` comes from the pass without them."""
        L.eb_timer_enable(1 if kernel_events else 0)
        L.eb_timer_collect(None, None)
        n0 = L.eb_launch_count()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0.record(stream)
        for _ in range(args.steps):
            step()
        t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        n = L.eb_launch_count() - n0
        kms_, kn_ = ctypes.c_double(0.0), ctypes.c_longlong(0)
        L.eb_timer_collect(ctypes.byref(kms_), ctypes.byref(kn_))
        L.eb_timer_enable(0)
        return t0.elapsed_time(t1), n, kms_, kn_

    clocks.start()
    ms, launches, _, _ = timed(False)
    ms_kpass, _, kms, kn = timed(True)  # the same K steps again: the roofline's kernel time
    comm = _communication(execs, q_bound_total)  # before the dimension-tree / CP-ALS extras
    clk = clocks.stop()
    if world > 1:
        ms = _max_over_ranks(ms)
        ms_kpass = _max_over_ranks(ms_kpass)
    ms_step = ms / args.steps
    value = flops_tree / (ms_step * 1e-3) / 1e9

    # C2 with the reference's per-mode schedules: also time the same sweep with
    # the dimension tree (modes 0+1 from one pass over X), reported beside the
    # headline (which stays on the reference's decomposition).
    alt = None
    als = None
    if args.config == "C2" and not dimtree:
        alt = _time_dimtree(eb, execs, inputs, stream, args, world, flops_tree)
        if world == 1:
            als = _time_cp_als(eb, inputs, stream, args, flops_tree)

    # e2e through the C ABI with host buffers.
    e2e = None
    if not args.no_e2e:
        outs = [np.empty(ex_.output_elems()) for ex_ in execs]
        h2d = 0
        for ins, ex_, sh in zip(inputs, execs, x_shared):
            # bytes this rank copies: its blocks of every operand it stages
            h2d += (sum(a.nbytes for a in _stage_list(ins, sh, dimtree and ex_ is execs[1])
                        if a is not None) if blockmode else
                    _staged_bytes(ex_, ins, P, rank if ranked else -1, eb, skip0=sh,
                                  skip2=dimtree and ex_ is execs[1]))
        d2h = sum(o.nbytes for o in outs) if rank == 0 else 0
        pipelined = world == 1 and not blockmode and not ranked
        reps = max(3, min(args.steps, 8)) if pipelined else max(1, min(args.steps, 3))
        if pipelined:
            # two executor sets on two streams: step k + 1's upload overlaps
            # step k's contraction (every step still uploads its inputs from
            # pinned host memory and reads its outputs back)
            stream2 = torch.cuda.Stream()
            execs2 = []
            for mi, (e, ext, _) in enumerate(modes):
                ex2 = (eb.Executor(e, ext, P, stream=stream2.cuda_stream) if mi == 0 else
                       eb.Executor(e, ext, stream=stream2.cuda_stream, like=execs2[0]))
                if x_shared[mi]:  # (the source must be staged first)
                    ex2.share_input(0, execs2[0], 0)
                    if dimtree and mi == 1:
                        ex2.share_input(2, execs2[0], 2)
                _stage(ex2, inputs[mi], x_shared[mi], dimtree and mi == 1, False)
                execs2.append(ex2)
            sets = [execs, execs2]

            def stage_set(xs):
                for mi_, (ins, ex_, sh) in enumerate(zip(inputs, xs, x_shared)):
                    _stage(ex_, ins, sh, dimtree and mi_ == 1, False)

            def run_set(xs):
                if dimtree:
                    if not xs[0].run_pair(xs[1]):
                        raise RuntimeError("dimension-tree pair did not qualify")
                    xs[2].run()
                else:
                    for ex_ in xs:
                        ex_.run()
                for ex_ in xs:
                    ex_.join()

            stage_set(execs2)  # warm the second set once (allocations), untimed
            run_set(execs2)
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if pipelined:
            stage_set(sets[0])
            for k in range(reps):
                cur = sets[k % 2]
                run_set(cur)
                if k + 1 < reps:
                    stage_set(sets[(k + 1) % 2])
                for ex_, out in zip(cur, outs):
                    ex_.gather(out)
        else:
            for _ in range(reps):
                for mi_, (ins, ex_, sh) in enumerate(zip(inputs, execs, x_shared)):
                    _stage(ex_, ins, sh, dimtree and mi_ == 1, blockmode)
                step()
                for ex_, out in zip(execs, outs):
                    ex_.gather(out if rank == 0 else None)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps
        if world > 1:
            dt = _max_over_ranks(dt)
        e2e = {"value": flops_tree / dt / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": dt * 1e3,
               "host_buffers": "pinned" if (world == 1 or blockmode) else "pageable",
               "steps": reps,
               "pipelined": ("two executor sets on two streams: step k+1's H2D overlaps step "
                             "k's contraction; every step uploads its inputs and reads back "
                             "its outputs inside the timed region") if pipelined else None}
        if world == 1:
            # the e2e roofline: the same bytes through one plain pinned H2D copy
            bw = _h2d_gbs(int(h2d))
            if bw:
                e2e["h2d_copy_gbs"] = bw
                e2e["h2d_only_ms"] = h2d / (bw * 1e9) * 1e3
                e2e["frac_of_h2d_bound"] = (h2d / (bw * 1e9)) / dt

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    # Roofline of the dominant kernel (the fused contraction), live events.
    # All launches of the fused contraction kernel in the timed steps (one per
    # MTTKRP mode for C1-C3, one per TTM step for C4/C5): algorithmic flops of
    # the work they do (the reference tree's flops, this rank's 1/P share)
    # over their CUDA-event time.
    # The per-kernel events break the programmatic-dependent overlap between
    # consecutive launches, so the kernel time they measure can exceed the
    # whole event-free step (C5: two back-to-back TTM-pair launches); the
    # kernel time per step is bounded by that step time.
    kms_step = min(kms.value / args.steps, ms_step)
    kern_ms = kms_step * args.steps / max(kn.value, 1)
    launches_per_step = max(kn.value // max(args.steps, 1), 1)
    # executed DMMA flops: the dimension tree contracts X twice per sweep, not 3x
    kflops = flops_tree * (2.0 / 3.0 if dimtree else 1.0)
    per_launch_flops = kflops / P / launches_per_step
    achieved = (kflops / P) / (kms_step * 1e-3) / 1e12
    peaks = _load_peaks()
    traffic = _traffic(args.config)
    roof = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
            "kernel": ("eb::mttkrp_rf_kernel (U resident in registers, FP64 DMMA.8x8x4, "
                       "16 rows x 8 outer indices per TMA stage)" if args.config == "C3" else
                       "eb::contract_kernel (FP64 DMMA.8x8x4, TMA SWIZZLE_128B ring)"),
            "peak_source": "measured FP64 DMMA peak, profiles/fp64_peak_r01.jsonl "
                           "(MEASURED_PEAKS.json has no FP64 figure)",
            "fp64_achieved_tflops": achieved,
            "kernel_ms_per_launch": kern_ms, "kernel_launches_timed": kn.value,
            "kernel_share_of_step": kms.value / max(ms_kpass, 1e-9),
            "kernel_ms_per_step_events": kms.value / args.steps,
            "kernel_ms_per_step_used": kms_step,
            "kernel_pass_ms_per_step": ms_kpass / args.steps,
            "kernel_timing": "a second pass of the same K steps with the main launches "
                             "bracketed by CUDA events on their stream (value/ms_per_step "
                             "come from the pass without them)",
            "hbm_achieved_gbs": _x_bytes(modes, P) * (2.0 / 3.0 if dimtree else 1.0)
                                / (kms_step * 1e-3) / 1e9,
            "hbm_peak_gbs": peaks.get("hbm_gbs"),
            "algorithmic_flops_per_launch": per_launch_flops,
            "launches_per_step": launches_per_step}
    # The FP64 peak was measured at 1965 MHz (profiles/fp64_peak_r01.jsonl); DMMA
    # throughput scales with the SM clock, so under a power cap the attainable
    # peak is lower: reported beside the fixed denominator, not instead of it.
    run_mhz = (clk or {}).get("sm_mhz") if isinstance(clk, dict) else None
    if run_mhz:
        roof["peak_clock_mhz"] = FP64_PEAK_CLOCK_MHZ
        roof["fp64_peak_at_run_clock"] = FP64_PEAK_TFLOPS * run_mhz / FP64_PEAK_CLOCK_MHZ
        roof["fp64_frac_at_run_clock"] = achieved / roof["fp64_peak_at_run_clock"]
    if args.config == "C5":
        # C5 sits at the HBM side of the ridge (1.316 ms of HBM vs
        # 1.233 ms of FP64 per GPU): the binding roof is bandwidth.  Algorithmic
        # bytes per GPU = SURVEY §8(d): 8 * (#X + sum #U + #out) = 8.6235e9 —
        # the term-0 output t1 is an artefact of the two-term schedule, so its
        # round trip (written once, read once) is reported as excess traffic,
        # not counted as required bytes.
        e0, ext0, _ = modes[0]
        ins0 = e0.split("->")[0].split(",")
        x_el = int(np.prod([ext0[c] for c in ins0[0]])) // P
        u_el = sum(int(np.prod([ext0[c] for c in t])) for t in ins0[1:])
        t1_el = x_el // (ext0["j"] * ext0["k"]) * ext0["b"] * ext0["c"]
        out_el = x_el // (ext0["j"] * ext0["k"] * ext0["l"] * ext0["m"]) * \
            ext0["b"] * ext0["c"] * ext0["d"] * ext0["e"]
        kbytes = 8.0 * (x_el + u_el + out_el)
        excess = 8.0 * 2 * t1_el
        ksec = kms_step * 1e-3
        gbs = kbytes / ksec / 1e9
        hbm_peak = float(peaks.get("hbm_gbs") or 6650.0)
        roof.update({"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s",
                     "frac": gbs / hbm_peak,
                     "kernel": "eb::ttm2_ws_kernel (two fused TTM pairs, FP64 DMMA)",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy test)" if peaks.get("hbm_gbs")
                                    else "fallback (B200_PROFILING.md)",
                     "algorithmic_bytes_per_step": kbytes,
                     "algorithmic_bytes_source": "SURVEY §8(d): 8 * (#X + sum #U + #out) per GPU",
                     "excess_bytes_per_step": excess,
                     "excess_note": "t1 (the term-0 output of the reference's two-term "
                                    "schedule) written and read back once per step",
                     "moved_gbs_incl_excess": (kbytes + excess) / ksec / 1e9,
                     "hbm_achieved_gbs": gbs})
    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference random_tensor streams (mt19937_64, seed 0 for X, "
                "factor seeds 1/2/3), generated on the host",
        "config": {"workload": label, "procs": P, "fast_mem": 1024, "grids": grids,
                   "transport": (args.transport if args.transport in ("peer", "hybrid") else
                                 "nccl" if use_nccl else "virtual"),
                   **({"shared_gpu": "ranks share the visible GPUs: a functional check, "
                                     "not a multi-GPU timing"} if args.share_gpu else {}),
                   "tree_flops_per_step": flops_tree,
                   "l2": "inputs larger than L2 (X is %.2f GB per GPU vs 126 MB L2), no flush "
                         "needed" % (_x_bytes(modes[:1], P) / 1e9)},
        "roofline": roof,
        "communication": comm,
        "e2e": e2e,
        **({"sweep_dimtree": alt} if alt else {}),
        **({"cp_als": als} if als else {}),
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_leg(args.config)
    if world == 1 and args.config == "C2" and not args.no_other_configs:
        line["other_configs"] = _other_configs(args)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _communication(execs, q_bound_total):
    """Reduction / exchange volume of one step against the derived I/O lower
    bound, with the reference's accounting (CommStats, executor.cpp:103-105,
    193-198; einplan_bench_json's volume_to_bound_ratio, bench.cpp:79-87):
    allreduce = block elements x (group - 1), redistribute = transmitted
    volume of the non-self messages, bound = the chosen partition's total_q
    (SOAP, S = 1024), summed over the step's einsums."""
    ar = rd = mx = 0
    for ex in execs:
        st = ex.stats()
        ar += int(st["allreduce_volume"])
        rd += int(st["redistribute_volume"])
        mx += int(st["max_rank_sent"])
    tot = ar + rd
    return {"allreduce_elems": ar, "redistribute_elems": rd, "volume_total_elems": tot,
            "volume_total_bytes": 8 * tot, "max_rank_sent_bytes": 8 * mx,
            "q_bound_total_elems": q_bound_total,
            "volume_to_bound_ratio": (tot / q_bound_total) if q_bound_total > 0 else None,
            "accounting": "reference CommStats / bench.cpp:79-87 (elements; bytes = 8x)"}


def _other_configs(args):
    """The other BASELINE configs measured in the same run (after the timed
    headline, one subprocess each: `bench.py --config C --no-e2e
    --no-cpu-baseline`), summarised: value, ms/step, the binding roof and
    the fraction of it, the clocks they ran at."""
    out = {}
    for c in ("C1", "C3", "C4", "C5"):
        cmd = [sys.executable, os.path.abspath(__file__), "--config", c, "--steps",
               str(max(args.steps, 10)), "--warmup", str(max(args.warmup, 3)), "--no-e2e",
               "--no-cpu-baseline"]
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
            l = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
            ro = l["roofline"]
            out[c] = {"workload": l["config"]["workload"], "value": l["value"], "unit": l["unit"],
                      "ms_per_step": l["ms_per_step"], "bound": ro["bound"],
                      "achieved": ro["achieved"], "peak": ro["peak"], "roof_unit": ro["unit"],
                      "frac": ro["frac"], "kernel": ro.get("kernel"),
                      "gpu_launches": l.get("gpu_launches"), "clocks": l.get("clocks"),
                      "communication": l.get("communication")}
        except Exception as e:  # reported, never fatal for the headline
            out[c] = {"error": f"{type(e).__name__}: {e}"[:300]}
    return out


def _max_over_ranks(x: float) -> float:
    """Max over ranks (the timing rule), on whichever backend carries the
    plumbing (NCCL: a device tensor; gloo: a host one)."""
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _self_launch(n, share_gpu=False):
    """`bench.py --gpus N` without torchrun: re-launch as N ranks (one process
    per GPU) with torch.distributed.run; fail loudly when the box has fewer
    than N GPUs instead of running one rank (unless --share-gpu asks for the
    functional check on fewer GPUs)."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < n and not share_gpu:
        print(f"bench.py: --gpus {n} needs {n} GPUs, this box has {have}", file=sys.stderr)
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the init lines show every rank joining
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def _time_dimtree(eb, execs, inputs, stream, args, world, flops_tree):
    """Device time of the C2 sweep as ONE eb_exec_run_pair (mode 0 + mode 1,
    T = X x_k C contracted once) plus the mode-2 executor, on the same staged
    X / factors; a fourth executor for mode 1 shares X and C from mode 0."""
    import torch
    import torch.distributed as dist
    ex0, ex1, ex2 = execs
    m1 = eb.Executor(ex1.einsum, ex1.extents, stream=stream.cuda_stream, like=ex0)
    m1.share_input(0, ex0, 0)
    m1.share_input(2, ex0, 2)
    if world > 1:
        m1.stage_block(1, inputs[1][1])  # same placement as the mode-1 executor
    else:
        m1.stage([None, inputs[1][1], None])

    m1.set_async_reduce(True)

    def step():
        if not ex0.run_pair(m1):
            raise RuntimeError("dimension-tree pair did not qualify")
        ex2.run()
        for ex in (ex0, m1, ex2):
            ex.join()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        ms = _max_over_ranks(ms)
    ms_step = ms / args.steps
    return {"value": flops_tree / (ms_step * 1e-3) / 1e9, "unit": "GFLOP/s",
            "ms_per_step": ms_step,
            "executed_dmma_tflops": flops_tree * 2 / 3 / (ms_step * 1e-3) / 1e12,
            "frac_of_fp64_peak": flops_tree * 2 / 3 / (ms_step * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
            "note": "same three outputs; modes 0 and 1 share one contraction of X with C "
                    "(2/3 of the per-mode DMMA flops); value counts the reference tree flops"}


def _h2d_gbs(nbytes):
    """Bandwidth of one pinned host -> device copy of `nbytes` (best of 3)."""
    import torch
    try:
        n = max(nbytes // 8, 1)
        h = torch.empty(n, dtype=torch.float64, pin_memory=True)
        d = torch.empty(n, dtype=torch.float64, device="cuda")
        best = None
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            d.copy_(h, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        del h, d
        torch.cuda.empty_cache()
        return n * 8 / (best * 1e-3) / 1e9
    except Exception:
        return None


def _time_cp_als(eb, inputs, stream, args, flops_tree):
    """A full CP-ALS sweep (eb_cp3_als_sweep: the three MTTKRPs plus the
    Gram / Hadamard / SPD-inverse updates, dimension tree) on the C2 tensor,
    X resident; timed like the headline."""
    import torch
    X = torch.from_numpy(inputs[0][0]).to("cuda", non_blocking=False)
    I, J, K = X.shape
    A = torch.from_numpy(np.ascontiguousarray(inputs[1][1])).cuda()  # ia
    B = torch.from_numpy(np.ascontiguousarray(inputs[0][1])).cuda()  # ja
    C = torch.from_numpy(np.ascontiguousarray(inputs[0][2])).cuda()  # ka
    with torch.cuda.stream(stream):
        ws = None
        for _ in range(args.warmup):
            ws = eb.cp3_als_sweep(X, A, B, C, stream=stream.cuda_stream, workspace=ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            eb.cp3_als_sweep(X, A, B, C, stream=stream.cuda_stream, workspace=ws)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    finite = bool(torch.isfinite(A).all() and torch.isfinite(B).all() and torch.isfinite(C).all())
    del X, ws
    torch.cuda.empty_cache()
    return {"ms_per_sweep": ms, "mttkrp_gflops": flops_tree / (ms * 1e-3) / 1e9,
            "factors_finite": finite,
            "note": "one CP-ALS sweep (3 MTTKRPs + Gram/Hadamard/SPD-inverse updates) with the "
                    "dimension tree: 2 passes over X; value counts the 3 reference MTTKRP trees"}


def _x_bytes(modes, P):
    tot = 0
    for e, ext, _ in modes:
        t = e.split("->")[0].split(",")[0]
        tot += 8 * int(np.prod([ext[c] for c in t])) // P
    return tot


def _stage(ex, ins, x_shared, c_shared, blockmode):
    lst = _stage_list(ins, x_shared, c_shared)
    if not blockmode:
        ex.stage(lst)
        return
    for k, a in enumerate(lst):
        if a is not None:
            ex.stage_block(k, a)


def _stage_list(ins, x_shared, c_shared):
    """Host operands to stage: None for the ones aliased from executor 0."""
    out = list(ins)
    if x_shared:
        out[0] = None
    if c_shared:
        out[2] = None
    return out


def _staged_bytes(ex, ins, P, rank, eb, skip0=False, skip2=False):
    if skip0:
        ins = [np.empty(0)] + list(ins[1:])
    if skip2:
        ins = list(ins[:2]) + [np.empty(0)] + list(ins[3:])
    if P == 1:
        return sum(a.nbytes for a in ins)
    # Blocks of this rank: every operand is split over the grid dims it spans
    plan = json.loads(eb.plan_json(ex.einsum, _ext_of(ex, ins), P))
    tot = 0
    for t in plan["schedule"]["terms"]:
        for p in t["placements"]:
            if p["tensor"].startswith("in"):
                k = int(p["tensor"][2:])
                tot += ins[k].nbytes // p["owners"] if ins[k] is not None else 0
    return tot


def _ext_of(ex, ins):
    ext = {}
    for t, a in zip(ex.einsum.split("->")[0].split(","), ins):
        if a is None or a.size == 0:
            continue
        for c, n in zip(t, a.shape):
            ext[c] = n
    return ext


def _traffic(config):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(p)).get(config)
    except Exception:
        return None


if __name__ == "__main__":
    sys.exit(main())
