"""Multi-GPU partitioning contract on CPU with world_size 2 over gloo.

Instances shard independently: each rank evaluates a contiguous instance range of the mini-batch
on its own device (here: the dry host runtime, which runs every host step of the B200 path —
fibers, inline depths, schedule, offset tables).  Checked, as §8e states:
  * each shard's schedule equals the reference schedule (orc_schedule_depth, the CPU
    restatement of schedule.cpp:29-62) over the shard's own DFG,
  * the union over ranks of the per-(phase, depth, sig) canonical node sets (instance, emission
    ordinal within the instance) equals the single-device run's,
  * the bench's reductions (max of times, sum of node counts) over gloo.
No tensor crosses ranks: the only collectives are these test/bench reductions.
"""
import os
import sys
import ctypes

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def canonical(nodes, offset):
    """(phase, depth, sig) -> sorted (global instance, emission ordinal) of its nodes."""
    seen, out = {}, {}
    for n in sorted(nodes, key=lambda n: n.id):
        k = seen.get(n.instance, 0)
        seen[n.instance] = k + 1
        out.setdefault((n.phase, n.depth, n.sig_id), []).append((n.instance + offset, k))
    return {k: sorted(v) for k, v in out.items()}


def oracle_schedule(oracle, nodes):
    """Batches (phase, depth, sig, ghost, size, ids) the reference's schedule_depth forms."""
    L = oracle.L
    n = len(nodes)
    ids = np.array([x.id for x in nodes], np.int32)
    ph = np.array([x.phase for x in nodes], np.int32)
    de = np.array([x.depth for x in nodes], np.int32)
    sg = np.array([x.sig_id for x in nodes], np.int32)
    gh = np.array([int(x.ghost) for x in nodes], np.int32)
    ns = np.array([len(x.shared_ins) for x in nodes], np.int32)
    refs = np.array([v for x in nodes for r in x.shared_ins for v in r] or [0], np.int64)
    batches = np.zeros(5 * max(1, n), np.int32)
    order = np.zeros(max(1, n), np.int32)
    ops = ctypes.c_long(0)
    P = lambda a, t: a.ctypes.data_as(ctypes.POINTER(t))
    L.orc_schedule_depth.restype = ctypes.c_int
    nb = L.orc_schedule_depth(n, P(ids, ctypes.c_int), P(ph, ctypes.c_int), P(de, ctypes.c_int), P(sg, ctypes.c_int),
                              P(gh, ctypes.c_int), P(ns, ctypes.c_int), P(refs, ctypes.c_int64), P(batches, ctypes.c_int),
                              P(order, ctypes.c_int), ctypes.byref(ops))
    out, k = [], 0
    for b in range(nb):
        phase, depth, sig, ghost, size = (int(v) for v in batches[5 * b:5 * b + 5])
        out.append((phase, depth, sig, size, bool(ghost), [int(v) for v in order[k:k + size]]))
        k += size
    return out


def _worker(rank, world, port, model, hidden, batch, q):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_10611_b200 import mbx
        from conftest import Oracle, trace_rows
        ctx = mbx.Context(-1, "bf16x3")
        m = mbx.Model(ctx, model, hidden)
        m.make_params(1)
        toks, data = m.make_inputs(1, batch)
        st, sd, lo, hi = mbx.shard_instances(toks, data, batch, rank, world)
        r = m.evaluate_batch(st, sd, hi - lo, record_nodes=True)
        assert trace_rows(r.trace) == oracle_schedule(Oracle(), r.nodes), (rank, "shard schedule")
        mine = canonical(r.nodes, lo)
        allsets = [None] * world
        dist.all_gather_object(allsets, mine)
        if rank == 0:
            full = m.evaluate_batch(toks, data, batch, record_nodes=True)
            union = {}
            for part in allsets:
                for k, v in part.items():
                    union.setdefault(k, []).extend(v)
            union = {k: sorted(v) for k, v in union.items()}
            assert union == canonical(full.nodes, 0), "union of shard node sets != single-device run"
        # bench.py's reductions: max over ranks of the times, sum of the node counts
        t = torch.tensor([float(rank + 1), float(r.trace.total_nodes)], dtype=torch.float64)
        mx, tot = t.clone(), t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        assert mx[0] == world
        if rank == 0:
            full_nodes = m.evaluate_batch(toks, data, batch, record_nodes=False).trace.total_nodes
            assert int(tot[1]) == full_nodes
        q.put((rank, "ok"))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("model,hidden,batch", [("treelstm", 32, 8), ("birnn", 32, 6), ("mvrnn", 32, 5)])
def test_instance_shards_world2(model, hidden, batch):
    import random
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + random.randint(0, 2000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, model, hidden, batch, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res == {0: "ok", 1: "ok"}, res


def test_shard_instances_partition():
    sys.path.insert(0, ROOT)
    from paper_2305_10611_b200 import mbx
    ctx = mbx.Context(-1, "bf16x3")
    m = mbx.Model(ctx, "treelstm", 32)
    toks, data = m.make_inputs(3, 7)
    parts = [mbx.shard_instances(toks, data, 7, r, 3) for r in range(3)]
    assert [(p[2], p[3]) for p in parts] == [(0, 2), (2, 4), (4, 7)]
    assert np.array_equal(np.concatenate([p[0] for p in parts]), toks)
    assert np.array_equal(np.concatenate([p[1] for p in parts]), data)
