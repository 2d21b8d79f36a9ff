"""The product's N > 1 code path with REAL ranks: 2 and 4 processes on the one
GPU of the box, each one rank of the schedule (eb_exec_create_peer), the
collectives over peer memory (CUDA IPC).  NCCL cannot run several ranks on
one GPU; the peer transport can, and no kernel ever waits on another rank
(each collective synchronises its stream and meets the peers on the host).

Checked against (a) the oracle (reference naive_evaluate restated) and (b)
the virtual-rank run of the same schedule, BITWISE: the peer allreduce sums
the group in ascending rank order from 0.0 like eb_group_sum and the
reference loop (executor.cpp:91-98), and the redistribution copies the same
boxes (redistribute.cpp:185-206); the comm volumes equal the reference
accounting.  Repeated runs must leave the device pool flat.
"""
import json
import os
import subprocess
import sys
import uuid

import numpy as np
import pytest

import oracle
from tests._peer_worker import CASES

HERE = os.path.dirname(os.path.abspath(__file__))
TOL = 1e-12

pytestmark = pytest.mark.gpu


def _run_group(case, procs, tmp_path, runs=3, timeout=600):
    group = f"/eb_t{uuid.uuid4().hex[:16]}"
    env = dict(os.environ, EB_PEER_TIMEOUT_S="240")
    ps = [subprocess.Popen([sys.executable, os.path.join(HERE, "_peer_worker.py"), case,
                            str(procs), str(r), group, str(tmp_path), str(runs)],
                           stdout=subprocess.PIPE, stderr=subprocess.STDOUT, env=env)
          for r in range(procs)]
    logs = []
    for p in ps:
        try:
            out, _ = p.communicate(timeout=timeout)
        except subprocess.TimeoutExpired:
            for q in ps:
                q.kill()
            raise
        logs.append(out.decode(errors="replace"))
    for r, p in enumerate(ps):
        assert p.returncode == 0, f"rank {r} failed:\n{logs[r][-3000:]}"
    outs = [np.load(os.path.join(tmp_path, f"out{k}.npy")) for k in range(runs)]
    st = json.load(open(os.path.join(tmp_path, "stats.json")))
    mem = [json.load(open(os.path.join(tmp_path, f"rank{r}.json")))["mem"] for r in range(procs)]
    return outs, st, mem


def _virtual(eb, e, ext, procs, ops):
    ex = eb.Executor(e, ext, procs)
    ex.stage(ops)
    ex.run()
    return ex.gather(), ex.stats()


@pytest.mark.parametrize("case,procs", [
    ("mttkrp_m0", 2), ("mttkrp_m0", 4), ("mttkrp_m2", 4),
    ("ttmc3", 2), ("ttmc3", 4), ("ttmc5", 4), ("2mm", 4), ("3mm", 4),
    # eight real processes: depth-4 groups, the pushed TTMc exchanges
    ("mttkrp_m0", 8), ("ttmc3", 8), ("ttmc5", 8), ("2mm", 8),
])
def test_peer_processes_match_oracle_and_virtual(eb, case, procs, tmp_path):
    e, ext, seed = CASES[case]
    ops = oracle.seeded_inputs(e, ext, seed)
    if case == "ttmc5":  # the n-ary loop is 4e10 points here: the reference's chain instead
        from tests.test_gpu_parity import _ttmc_o5_chain
        want = _ttmc_o5_chain(ext, ops).ravel()
    else:
        want = oracle.naive_evaluate(e, ext, ops).ravel()
    outs, st, mem = _run_group(case, procs, tmp_path)
    virt, vstats = _virtual(eb, e, ext, procs, ops)
    for out in outs:
        assert oracle.normwise_error(out, want) <= TOL
        assert np.array_equal(out, virt), "peer ranks differ from the virtual ranks"
    stats = st["stats"]
    for k in ("allreduce_volume", "redistribute_volume", "max_rank_sent"):
        assert stats[k] == vstats[k], (k, stats, vstats)
    # the schedule really exchanges something at this P
    assert stats["allreduce_volume"] + stats["redistribute_volume"] > 0, stats
    assert stats["generic_launches"] == vstats["generic_launches"]
    # the device pool does not grow across runs on any rank
    for r, m in enumerate(mem):
        assert m[-1] <= m[1], f"rank {r} pool grew across runs: {m}"


def test_run_json_rank_threads_on_one_gpu(eb, monkeypatch):
    """einplan_run_json with one host thread per rank (EINPLAN_DEVICES=0,0,...
    places every rank thread on GPU 0; the peer transport between threads):
    the same report as the virtual-rank run, bitwise the same output sum, and
    the report says how it ran."""
    e, ext = "ijk,jb,kc->ibc", dict(i=24, j=40, k=36, b=8, c=6)
    for procs in (2, 4):
        monkeypatch.setenv("EINPLAN_EXEC", "virtual")
        st_v, rep_v = eb.Session(e, ext).run_json(procs, 1024.0, seed=3, verify=True)
        monkeypatch.delenv("EINPLAN_EXEC")
        monkeypatch.setenv("EINPLAN_DEVICES", ",".join(["0"] * procs))
        st_t, rep_t = eb.Session(e, ext).run_json(procs, 1024.0, seed=3, verify=True)
        monkeypatch.delenv("EINPLAN_DEVICES")
        assert st_v == st_t == 0
        a, b = json.loads(rep_v), json.loads(rep_t)
        assert a.pop("execution") == {"mode": "virtual", "devices": [0], "transport": "virtual"}
        assert b.pop("execution") == {"mode": "devices", "devices": [0] * procs,
                                      "transport": "peer"}
        assert a == b  # every field, the output sum and the verification error included


def test_run_json_one_rank_uses_the_device(eb):
    """procs = 1 on a 1-GPU box: one rank thread on device 0 (not virtual)."""
    st, rep = eb.Session("ijk,ja,ka->ia", dict(i=16, j=12, k=10, a=4)).run_json(1, 1024.0, seed=1)
    assert st == 0
    ex = json.loads(rep)["execution"]
    assert ex["mode"] == "devices" and ex["devices"] == [0]


def test_run_json_more_ranks_than_gpus_is_virtual(eb):
    import torch
    procs = torch.cuda.device_count() + 1
    st, rep = eb.Session("ijk,ja,ka->ia", dict(i=16, j=12, k=10, a=4)).run_json(
        procs, 1024.0, seed=1)
    assert st == 0
    assert json.loads(rep)["execution"]["mode"] == "virtual"


def test_virtual_runs_keep_the_pool_flat(eb):
    e, ext = "ijk,jb,kc->ibc", dict(i=32, j=48, k=40, b=8, c=6)
    ex = eb.Executor(e, ext, 4)
    ex.stage(oracle.seeded_inputs(e, ext, 5))
    mem = []
    for _ in range(4):
        ex.run()
        ex.gather()
        mem.append(eb.mem_in_use())
    assert mem[-1] <= mem[1], mem


def test_hybrid_transport_single_rank(eb, monkeypatch):
    """The hybrid transport (the default for one process per GPU: NCCL
    allreduce + fused redistribution over peer memory) as rank 0 of 1 — the
    only NCCL world this one-GPU pool can host — through the executor and
    through einplan_run_json."""
    import uuid
    for e, ext in (("ijk,ja,ka->ia", dict(i=64, j=64, k=64, a=16)),
                   ("ijk,jb,kc->ibc", dict(i=96, j=96, k=96, b=24, c=24))):
        ops = oracle.seeded_inputs(e, ext, 13)
        ex = eb.Executor(e, ext, 1, rank=0, transport="hybrid",
                         group=f"/eb_h{uuid.uuid4().hex[:12]}",
                         nccl_id=eb.Executor.nccl_unique_id())
        ex.stage(ops)
        for _ in range(2):
            ex.run()
            got = ex.gather()
            assert oracle.normwise_error(got, oracle.naive_evaluate(e, ext, ops).ravel()) <= TOL
    monkeypatch.setenv("EINPLAN_TRANSPORT", "hybrid")
    st, rep = eb.Session("ijk,jb,kc->ibc", dict(i=24, j=40, k=36, b=8, c=6)).run_json(1, seed=2)
    assert st == 0
    assert json.loads(rep)["execution"]["transport"] == "hybrid"
