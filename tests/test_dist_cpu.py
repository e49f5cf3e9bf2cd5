"""CPU, world_size 2 over gloo: the multi-GPU combination scheme.

Each rank plans the same cost-balanced partition (sthk_plan_partition),
reduces its own rows into 1024-row block partials, the zero-padded block
vectors are all-reduced (gloo here; NCCL in the engine) and summed in fixed
block order. The result must be bitwise identical to the single-rank sum and
the partitions identical on both ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_glue as og
import paper_2005_10123_b200 as pk
from paper_2005_10123_b200 import partition as part


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _data():
    ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                      pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005,
                                      keep=5000)
    p = [0.66, 1.6, 14.0, 0.344, 1440.0, 0.0695]
    o = og.oracle_loglik_grad(ev.xs(), ev.ys(), ev.ts(), ev.windowEnd(), p, per_event=True)
    return ev, p, o["per_event"]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ev, p, terms = _data()
    cuts, sc = part.plan_partition(ev.ts(), p, world)
    allc = [None] * world
    dist.all_gather_object(allc, (cuts.tolist(), sc))
    nb = (ev.size() + part.ROWS_PER_BLOCK - 1) // part.ROWS_PER_BLOCK
    local = part.block_partials(terms, int(cuts[rank]), int(cuts[rank + 1]), nb)
    buf = torch.from_numpy(local)
    dist.all_reduce(buf, op=dist.ReduceOp.SUM)
    total = part.ordered_sum(buf.numpy())
    q.put((rank, total, allc))
    dist.destroy_process_group()


def test_partition_properties():
    ev, p, _ = _data()
    for shards in (1, 2, 3, 8):
        cuts, sc = part.plan_partition(ev.ts(), p, shards)
        assert cuts[0] == 0 and cuts[-1] == ev.size()
        assert np.all(np.diff(cuts) >= 0)
        assert all(c % part.ROWS_PER_BLOCK == 0 or c == ev.size() for c in cuts)
        # (whole 128-source stages; one-stage chunks up to 24k events, else >= 4 stages)
        assert sc % 128 == 0 and (sc >= 512 or (ev.size() <= 24 * 1024 and sc == 128))
        # culling vs dense: same chunking (bitwise-identical results rely on it)
        assert part.plan_partition(ev.ts(), p, shards, dense=True)[1] == sc


def test_partition_balances_cost():
    # dense symmetric sweep: row i costs ~i sources (tiles J <= I), so the
    # balanced cuts shrink with the row index and the per-shard cost is even
    ev = pk.generateBenchmarkCloud(200000, pk.SimWindow(0, 15, 0, 15, 4750), 7)
    p = [1.0, 1.6, 14.0, 0.1, 1.0, 1.0]
    cuts, _ = part.plan_partition(ev.ts(), p, 4, dense=True)
    sizes = np.diff(cuts)
    assert np.all(np.diff(sizes) < 0)
    cost = [(int(b) ** 2 - int(a) ** 2) / 2 for a, b in zip(cuts[:-1], cuts[1:])]
    assert max(cost) < 1.1 * min(cost)


def test_gloo_world2_bitwise():
    ev, p, terms = _data()
    nb = (ev.size() + part.ROWS_PER_BLOCK - 1) // part.ROWS_PER_BLOCK
    single = part.ordered_sum(part.block_partials(terms, 0, ev.size(), nb))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    totals = {r: tot for r, tot, _ in res}
    assert totals[0] == totals[1] == single
    assert res[0][2] == res[1][2]  # identical partition on both ranks
