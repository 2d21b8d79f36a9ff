"""One rank of a multi-process run of the PRODUCT executor over the peer
transport (eb_exec_create_peer: CUDA IPC exchange heaps + a host barrier in
POSIX shared memory).  Launched by tests/test_multiprocess_gpu.py, several
processes on the one GPU of the box.

    python _peer_worker.py CASE PROCS RANK GROUP OUTDIR RUNS

Every rank stages its own blocks (from the global seeded operands, as the
reference's scatter does, executor.cpp:48-65), runs the schedule RUNS times
and takes part in the gather; rank 0 writes the output of every run and the
executor stats to OUTDIR.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: input generation only)
import paper_2206_08301_b200 as eb  # noqa: E402

CASES = {
    # MTTKRP mode 0: one term, reduction groups (allreduce)
    "mttkrp_m0": ("ijk,ja,ka->ia", dict(i=64, j=64, k=64, a=16), 3),
    "mttkrp_m2": ("ijk,ia,ja->ka", dict(i=40, j=36, k=64, a=8), 4),
    # TTMc order 3: two terms, t0 redistributed between the term grids
    "ttmc3": ("ijk,jb,kc->ibc", dict(i=96, j=96, k=96, b=24, c=24), 5),
    # TTMc order 5 (both terms on eb_ttm2)
    "ttmc5": ("ijklm,jb,kc,ld,me->ibcde",
              dict(i=32, j=16, k=16, l=16, m=16, b=12, c=12, d=12, e=12), 6),
    # GEMM chain: reduced intermediates feed a redistribution
    "2mm": ("ij,jk,kl->il", dict(i=40, j=36, k=48, l=28), 7),
    "3mm": ("ij,jk,kl,lm->im", dict(i=24, j=32, k=28, l=36, m=20), 8),
}


def main():
    import time
    case, procs, rank, group, outdir, runs = sys.argv[1:7]
    procs, rank, runs = int(procs), int(rank), int(runs)
    e, ext, seed = CASES[case]
    t0 = time.perf_counter()
    log = lambda what: print(f"rank {rank} {what} {time.perf_counter() - t0:.3f}s", flush=True)
    ex = eb.Executor(e, ext, procs, rank=rank, transport="peer", group=group)
    log("created")
    ex.stage(oracle.seeded_inputs(e, ext, seed))
    log("staged")
    mem = []
    for r in range(runs):
        ex.run()
        log(f"run {r}")
        out = ex.gather()
        log(f"gather {r}")
        mem.append(eb.mem_in_use())
        if rank == 0:
            np.save(os.path.join(outdir, f"out{r}.npy"), out)
    if rank == 0:
        with open(os.path.join(outdir, "stats.json"), "w") as f:
            json.dump({"stats": ex.stats(), "report": json.loads(ex.report_json(out))}, f)
    with open(os.path.join(outdir, f"rank{rank}.json"), "w") as f:
        json.dump({"mem": mem}, f)
    ex.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
