"""The N>1 data path on CPU: world-size-2 torch.distributed (gloo) processes,
each acting as one rank of the reference's processor grid.

Each process takes the schedule from the B200 build's planner (plan JSON with
messages — the same plan eb_exec uses), holds only its own placement blocks,
computes its local steps with the CPU oracle on its local index ranges
(local_contract semantics, executor.cpp:112-154), then performs the term's
exchange over gloo exactly as the NCCL transport does on GPUs:
MTTKRP partial outputs are all-reduced within the reduction group
(executor.cpp:80-108); TTMc's intermediate is redistributed with point-to-point
messages from the plan (redistribute.cpp:51-148, 185-206); the output is
gathered from canonical replicas on rank 0 and must equal the single-process
oracle result.
"""
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _coords(grid_dims, rank):
    c = []
    for d in reversed(grid_dims):
        c.append(rank % d)
        rank //= d
    return list(reversed(c))


def _local(term, ext, rank):
    order = list(term["grid"].keys())
    dims = [term["grid"][c] for c in order]
    co = _coords(dims, rank)
    lo = {c: co[i] * term["blocks"][c] for i, c in enumerate(order)}
    ln = {c: min(term["blocks"][c], ext[c] - lo[c]) for c in order}
    return lo, ln


def _block(global_arr, idx, lo, ln):
    sl = tuple(slice(lo[c], lo[c] + ln[c]) for c in idx)
    return np.ascontiguousarray(global_arr[sl])


def _worker(rank, world, port, einsum, ext, fast_mem, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2206_08301_b200 as eb
    plan = json.loads(eb.plan_json(einsum, ext, world, fast_mem, include_messages=True))
    ins, out_idx = oracle.parse(einsum)
    inputs = oracle.seeded_inputs(einsum, ext, 5)            # every rank can regenerate
    steps = plan["tree"]["steps"]
    store = {}                                                 # (term, tensor) -> local block
    for ti, term in enumerate(plan["schedule"]["terms"]):
        lo, ln = _local(term, ext, rank)
        part_term = plan["partition"]["terms"][ti]
        have = {}
        for a in part_term["arrays"]:
            name = a["tensor"]
            if name == part_term["output"]:
                continue
            if name.startswith("in"):
                have[name] = _block(inputs[int(name[2:])], a["indices"], lo, ln)
                continue
            red = [r for r in plan["schedule"]["redistributions"]
                   if r["to_term"] == ti and r["tensor"] == name]
            if not red:
                have[name] = store[name]
                continue
            # redistribution: point-to-point boxes per the plan's messages
            src = store[name]
            shape = [ln[c] for c in a["indices"]]
            dst = np.zeros(shape)
            sends, recvs = [], []
            for m in red[0]["plan"]["messages"]:
                oy = [r["src"] for r in m["ranges"]]
                ox = [r["dst"] for r in m["ranges"]]
                if m["src_rank"] == rank and m["dst_rank"] == rank:
                    dst[tuple(slice(x[0], x[1]) for x in ox)] = \
                        src[tuple(slice(y[0], y[1]) for y in oy)]
                elif m["src_rank"] == rank:
                    box = np.ascontiguousarray(src[tuple(slice(y[0], y[1]) for y in oy)])
                    sends.append(dist.isend(torch.from_numpy(box), m["dst_rank"]))
                elif m["dst_rank"] == rank:
                    buf = torch.empty([y[1] - y[0] for y in oy], dtype=torch.float64)
                    recvs.append((dist.irecv(buf, m["src_rank"]), buf, ox))
            for req, buf, ox in recvs:
                req.wait()
                dst[tuple(slice(x[0], x[1]) for x in ox)] = buf.numpy()
            for s in sends:
                s.wait()
            have[name] = dst
        # local steps of the term (local_contract)
        for sid in sorted(int(s) for s in _term_steps(plan, ti)):
            st = steps[sid]
            lhs_i, rest = st["expr"].split("->")[0], st["expr"].split("->")[1]
            ops_idx = lhs_i.split(",")
            names = [st["lhs"]] + ([st["rhs"]] if "rhs" in st else [])
            lext = {c: ln[c] for c in "".join(ops_idx)}
            res = oracle.naive_evaluate(st["expr"], lext, [have[n] for n in names])
            have[st["result"]] = res
        out_name = part_term["output"]
        partial = have[out_name]
        depth = term["reduction"]["depth"]
        if depth > 1:
            t = torch.from_numpy(np.ascontiguousarray(partial))
            dist.all_reduce(t)          # world == reduction group at P = 2 here
            partial = t.numpy()
        store[out_name] = partial
    # gather canonical replicas of the output on rank 0
    last = plan["schedule"]["terms"][-1]
    lo, ln = _local(last, ext, rank)
    out_i = plan["partition"]["terms"][-1]["arrays"][-1]["indices"]
    mine = store[plan["partition"]["terms"][-1]["output"]]
    boxes = [None] * world
    dist.all_gather_object(boxes, (lo, ln, mine))
    if rank == 0:
        full = np.zeros([ext[c] for c in out_i])
        for lo_r, ln_r, blk in boxes:
            full[tuple(slice(lo_r[c], lo_r[c] + ln_r[c]) for c in out_i)] = blk
        want = oracle.naive_evaluate(einsum, ext, inputs)
        result_q.put(oracle.normwise_error(full, want))
    dist.barrier()
    dist.destroy_process_group()


def _term_steps(plan, ti):
    return plan["schedule"]["terms"][ti].get("steps") or _steps_from_partition(plan, ti)


def _steps_from_partition(plan, ti):
    # partition blocks list result tensor names; map to step ids in tree order
    names = plan["partition"]["blocks"][ti]
    out = []
    for sid, st in enumerate(plan["tree"]["steps"]):
        if st["result"] in names:
            out.append(sid)
    return out


@pytest.mark.parametrize("einsum,ext,fast_mem,kind", [
    ("ijk,ja,ka->ia", dict(i=12, j=10, k=14, a=6), 1024.0, "allreduce"),   # k2, depth 2
    ("ijk,ia,ka->ja", dict(i=16, j=12, k=10, a=4), 1024.0, "allreduce"),
    ("ijk,jb,kc->ibc", dict(i=8, j=8, k=8, b=3, c=3), 16.0, "redistribute"),  # k2 -> b2
    ("ijk,jb,kc->ibc", dict(i=16, j=16, k=16, b=4, c=4), 32.0, "redistribute"),  # k2 -> i2
])
def test_two_rank_gloo_matches_oracle(eb, einsum, ext, fast_mem, kind):
    plan = json.loads(eb.plan_json(einsum, ext, 2, fast_mem))
    assert plan["schedule"]["procs"] == 2
    if kind == "allreduce":
        assert any(t["reduction"]["depth"] > 1 for t in plan["schedule"]["terms"])
    else:
        assert sum(r["plan"]["transmitted_volume"] for r in plan["schedule"]["redistributions"]) > 0
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, einsum, ext, fast_mem, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    err = q.get(timeout=5)
    assert err <= 1e-13, err
