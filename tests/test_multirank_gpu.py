"""Multi-rank engine on one GPU (BASELINE config 4).

The row partition, the owner-directed exchange of the symmetric sweep's
column sums and the exact combination of the block partials run here with
every rank a separate engine -- own accumulators, trigger partials, plans
and block partials:

  * Engine((0,) * k): k shards in one process sharing cuda:0, combined by
    device copies along exactly the routes the NCCL path uses;
  * two processes on cuda:0, each a rank engine whose collectives go through
    torch.distributed gloo host callbacks (sthk_create_rank_hosted).

Every configuration must reproduce the single-shard result bitwise
(reference: contiguous target blocks summed in order, backend.hpp:139-166)."""
import os
import socket

import numpy as np
import pytest

import paper_2005_10123_b200 as pk

pytestmark = pytest.mark.gpu

THETA_POST = [0.66, 1.6, 14.0, 0.344, 1440.0, 0.0695]
THETA_INIT = [1.0, 1.6, 14.0, 0.1, 1.0, 1.0]


def _cluster(keep):
    ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                      pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005,
                                      keep=keep)
    return ev


def _same(a, b):
    return a[0] == b[0] and a[1] == b[1] and np.array_equal(a[2], b[2])


@pytest.mark.parametrize("k", [2, 3, 8])
def test_c2_emulated_ranks_bitwise(engine, k):
    """C2 (N = 85,000), both Theta: k rank engines on one GPU == one shard,
    loglik, gradient and every per-event term bitwise."""
    ev = _cluster(85000)
    engine.load(ev)
    with pk.Engine((0,) * k) as sh:
        sh.load(ev)
        for theta in (THETA_POST, THETA_INIT):
            engine.set_params(theta)
            sh.set_params(theta)
            a = engine.loglik_grad(per_event=True)
            b = sh.loglik_grad(per_event=True)
            assert _same(a, b) and np.array_equal(a[3], b[3]), (a[0], b[0])
            # the owner-directed exchange ships only rows other shards own, far
            # less than the 6 x N x 8 B a whole-array all-reduce would move
            nbytes = sh.exchange_bytes()
            assert 0 < nbytes < 6 * 8 * ev.size()


@pytest.mark.parametrize("k", [2, 3, 8])
def test_c4_1m_emulated_ranks_bitwise(engine, k):
    """C4 size (N = 1,000,000): the 2/3/8-rank split == one shard, bitwise."""
    n = 1000000
    ev = pk.generateBenchmarkCloud(n, pk.SimWindow(0, 15, 0, 15, 4750), n)
    engine.load(ev)
    engine.set_params(THETA_POST)
    a = engine.loglik_grad()
    with pk.Engine((0,) * k) as sh:
        sh.load(ev)
        sh.set_params(THETA_POST)
        b = sh.loglik_grad()
        assert _same(a, b), (a[0], b[0])
        # per rank and evaluation: well under the 48 MB fx all-reduce
        assert sh.exchange_bytes() < 6 * 8 * n // 4


def test_emulated_ranks_sweep_caches_bitwise(engine):
    """MH-style moves (mu0, theta, omega, h; tauX, tauT fixed as in the
    reference sampler) on 4 rank engines: the cached background (a shard's
    own rows), trigger-only sweeps and finalize-only moves reproduce full
    single-shard evaluations bitwise; a tauT move re-sweeps."""
    ev = _cluster(30000)
    rng = np.random.default_rng(5)
    engine.load(ev)
    engine.set_background_cache(False)
    try:
        with pk.Engine((0,) * 4) as sh:
            sh.load(ev)
            theta = list(THETA_POST)
            hits = 0
            for it in range(24):
                k = [0, 3, 4, 5, 2][it % 5]
                theta[k] *= float(np.exp(0.05 * rng.standard_normal()))
                engine.set_params(theta)
                sh.set_params(theta)
                a = engine.loglik_grad()
                b = sh.loglik_grad()
                hits += sh.stats()["cache_hit"]
                assert _same(a, b), (it, a[0], b[0])
            assert hits > 0
    finally:
        engine.set_background_cache(True)


@pytest.mark.parametrize("mode", ["rows", "dense", "far_off"])
def test_emulated_ranks_kernel_variants_bitwise(engine, mode):
    """The row kernel (no column sums: no exchange), dense sweeps and the
    all-FP64 path split across 3 ranks == one shard of the same variant."""
    ev = _cluster(20000)
    engine.load(ev)
    with pk.Engine((0, 0, 0)) as sh:
        sh.load(ev)
        for eng in (engine, sh):
            if mode == "rows":
                eng.set_kernel(0)
            elif mode == "dense":
                eng.set_dense(True)
            else:
                eng.set_far_tier(False)
        try:
            for theta in (THETA_POST, THETA_INIT):
                engine.set_params(theta)
                sh.set_params(theta)
                assert _same(engine.loglik_grad(), sh.loglik_grad())
            if mode == "rows":
                assert sh.exchange_bytes() == 0
        finally:
            engine.set_kernel(1)
            engine.set_dense(False)
            engine.set_far_tier(True)


def test_emulated_ranks_excitation_and_batch(engine):
    """Per-event excitation split and grouped batches through 3 ranks."""
    ev = _cluster(15000)
    engine.load(ev)
    grid = [[0.66, 1.6, 14, th, om, 0.0695] for th in (0.2, 0.344) for om in (720.0, 1440.0)]
    with pk.Engine((0, 0, 0)) as sh:
        sh.load(ev)
        engine.set_params(THETA_POST)
        sh.set_params(THETA_POST)
        for u, v in zip(engine.excitation(), sh.excitation()):
            assert np.array_equal(u, v)
        la, oa, ga = engine.loglik_batch(grid, grad=True)
        lb, ob, gb = sh.loglik_batch(grid, grad=True)
        assert np.array_equal(la, lb) and np.array_equal(oa, ob) and np.array_equal(ga, gb)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _hosted_worker(rank, world, port, keep, q):
    import torch.distributed as dist
    from paper_2005_10123_b200.hostcomm import TorchDistComm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ev = _cluster(keep)
        comm = TorchDistComm()
        out = []
        with pk.Engine((0,), rank=rank, world=world, comm=comm) as eng:
            eng.load(ev)
            for theta in (THETA_POST, THETA_INIT):
                eng.set_params(theta)
                ll, ok, g, pe = eng.loglik_grad(per_event=True)
                out.append((ll, ok, g.tolist(), pe.tolist(), eng.exchange_bytes()))
            # MH-style: theta / omega moves over the cached background
            for theta in ([0.7, 1.6, 14, 0.3, 1440, 0.0695], [0.7, 1.6, 14, 0.3, 1300, 0.0695]):
                eng.set_params(theta)
                ll, ok, g, _ = eng.loglik_grad()
                out.append((ll, ok, g.tolist(), None, eng.stats()["cache_hit"]))
        q.put((rank, out, None))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, None, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_hosted_gloo_ranks_bitwise(engine, world):
    """`world` processes on cuda:0, each a rank engine (sthk_create_rank_hosted)
    whose fx exchange and block all-reduce run over gloo: every rank returns
    the single-engine loglik and gradient bitwise and its own rows' per-event
    terms."""
    import torch.multiprocessing as mp
    keep = 20000
    ev = _cluster(keep)
    engine.load(ev)
    ref = []
    for theta in (THETA_POST, THETA_INIT, [0.7, 1.6, 14, 0.3, 1440, 0.0695],
                  [0.7, 1.6, 14, 0.3, 1300, 0.0695]):
        engine.set_params(theta)
        ref.append(engine.loglik_grad(per_event=True))
    cuts, _ = pk.partition.plan_partition(ev.ts(), THETA_POST, world)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_hosted_worker, args=(r, world, port, keep, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, out, err in res:
        assert err is None, err
        lo, hi = int(cuts[rank]), int(cuts[rank + 1])
        for j, (ll, ok, g, pe, extra) in enumerate(out):
            r = ref[j]
            assert ll == r[0] and ok == r[1] and np.array_equal(np.array(g), r[2]), (rank, j)
            if pe is not None:
                assert np.array_equal(np.array(pe)[lo:hi], r[3][lo:hi])
            if j == 0 and rank > 0:
                assert extra > 0  # (fx bytes sent to earlier owners)
        # background cached across the omega move (the theta move before it
        # re-sweeps: from Θ_init's tiled trigger terms to row windows, the
        # near split -- hence the background's grouping -- changes)
        assert out[3][4] == 1
