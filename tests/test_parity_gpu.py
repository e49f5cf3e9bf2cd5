"""GPU parity: the sm_100a engine vs the long-double oracle and the verbatim
reference engine (oracle/_ref). Tolerances from BASELINE.json north_star:
<= 1e-10 relative on loglik, <= 1e-8 per gradient component (scale-aware
norm sum_i |d l_i / d p_k| near stationary points)."""
import math
import os

import numpy as np
import pytest

import oracle_glue as og
import paper_2005_10123_b200 as pk

pytestmark = pytest.mark.gpu

LL_TOL = 1e-10
G_TOL = 1e-8


def _rand_params(rng):
    return pk.Params(rng.uniform(0.3, 2.0), rng.uniform(0.5, 2.0), rng.uniform(2.0, 20.0),
                     rng.uniform(0.05, 0.8), rng.uniform(0.3, 3.0), rng.uniform(0.1, 1.0))


def _check(engine, ev, p, ll_tol=LL_TOL, g_tol=G_TOL):
    r, g = pk.logLikelihoodGradient(ev, p, engine=engine)
    o = og.oracle_loglik_grad(ev.xs(), ev.ys(), ev.ts(), ev.windowEnd(), p.as_array())
    assert r.valid == o["valid"]
    if not o["valid"]:
        assert r.logLik == -math.inf
        return r, g, o
    assert abs(r.logLik - o["loglik"]) <= ll_tol * abs(o["loglik"]), (r.logLik, o["loglik"])
    # scale-aware gradient norm: |g_k - g_k^oracle| <= tol * sum_i |d l_i/d p_k|
    # (|g_k| itself can be ~0 near a stationary point)
    scale = np.maximum(o["grad_abs"], 1e-300)
    err = np.abs(g - o["grad"]) / scale
    assert np.all(err <= g_tol), (g, o["grad"], err)
    # plain per-component relative error wherever the component is not
    # dominated by cancellation (|g_k| >= 1e-6 sum_i |d l_i / d p_k|)
    well = np.abs(o["grad"]) >= 1e-6 * o["grad_abs"]
    rel = np.abs(g - o["grad"]) / np.maximum(np.abs(o["grad"]), 1e-300)
    assert np.all(rel[well] <= g_tol), (g, o["grad"], rel)
    return r, g, o


def test_single_event_closed_form(engine):
    # test_likelihood.cpp:42-56
    ev = pk.EventSet([0.0], [0.0], [1.0], 1.0)
    p = pk.Params(1, 1, 1, 1, 1, 1)
    r = pk.logLikelihood(ev, p, engine=engine)
    assert r.valid
    assert abs(r.logLik - (-3.0981603456825612)) <= 1e-13


def test_five_event_fixture(engine):
    # test_likelihood.cpp:84-104
    ev = pk.EventSet([0.1, 0.9, -0.4, 0.2, 1.1], [-0.2, 0.3, 0.5, 0.9, -0.8],
                     [0.4, 1.1, 1.9, 3.0, 4.2], 5.0)
    p = pk.Params(0.6, 0.9, 3.0, 0.5, 1.1, 0.35)
    r, g, o = _check(engine, ev, p)
    assert abs(r.logLik - (-19.396372326920137)) <= 1e-10 * 19.4


def test_random_instances(engine):
    # test_likelihood.cpp:106-121 shape: N in {2,3,10,100}, 8 reps each
    rng = np.random.default_rng(2024)
    inst = 0
    for n in (2, 3, 10, 100):
        for _ in range(8):
            ev = pk.generateBenchmarkCloud(n, pk.SimWindow(0, 4, 0, 4, 60), 1000 + inst)
            _check(engine, ev, _rand_params(rng))
            inst += 1


@pytest.mark.parametrize("n", [127, 128, 129, 1000, 4099])
def test_tile_edges(engine, n):
    ev = pk.generateBenchmarkCloud(n, pk.SimWindow(0, 4, 0, 4, 60), n)
    _check(engine, ev, pk.Params(0.6, 0.9, 3.0, 0.5, 1.1, 0.35))


def test_dc_shaped_culling_exact(engine):
    ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                      pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005,
                                      keep=6000)
    for p in (pk.Params(0.66, 1.6, 14, 0.344, 1440, 0.0695), pk.Params(1, 1.6, 14, 0.1, 1, 1)):
        engine.load(ev)
        engine.set_params(p)
        engine.set_dense(False)
        a = engine.loglik_grad()
        engine.set_dense(True)
        b = engine.loglik_grad()
        engine.set_dense(False)
        assert a[0] == b[0] and np.array_equal(a[2], b[2])
        _check(engine, ev, p)


def test_matches_reference_engine(engine):
    if not og.ref_available():
        pytest.skip("oracle/_ref not built")
    ev = pk.generateBenchmarkCloud(1000, pk.SimWindow(0, 4, 0, 4, 60), 1000)
    p = pk.Params(0.6, 0.9, 3.0, 0.5, 1.1, 0.35)
    ref, ok, _ = og.ref_loglik(ev.xs(), ev.ys(), ev.ts(), ev.windowEnd(), p.as_array(), 4, 8)
    r = pk.logLikelihood(ev, p, engine=engine)
    assert ok and r.valid
    assert abs(r.logLik - ref) <= LL_TOL * abs(ref)


@pytest.mark.parametrize("k", [2, 3, 8])
def test_partition_bitwise_invariant(engine, k):
    """Row partition across k shards -- k separate rank engines on one device
    (own accumulators, plans and partials) combined along the multi-GPU
    routes -- gives bitwise-identical results."""
    ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                      pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005,
                                      keep=20000)
    engine.load(ev)
    with pk.Engine((0,) * k) as sh:
        sh.load(ev)
        for p in (pk.Params(0.66, 1.6, 14, 0.344, 1440, 0.0695), pk.Params(1, 1.6, 14, 0.1, 1, 1)):
            engine.set_params(p)
            sh.set_params(p)
            a = engine.loglik_grad(per_event=True)
            b = sh.loglik_grad(per_event=True)
            assert a[0] == b[0] and np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3])
            if p.omega == 1440:  # (the second Theta reuses the cached background)
                assert sh.exchange_bytes() > 0


def test_pair_counters_and_results_through_mapped_memory(engine):
    """Results and (timing) pair counters reach the host through device-mapped
    memory written by the last kernel (fused final sum for one shard, the
    final-sum kernel for several), which also re-zeroes the counters: repeated
    timed evaluations report the same counts, equal across shard counts, and
    the result matches an untimed evaluation bitwise."""
    ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                      pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005,
                                      keep=12000)
    engine.load(ev)
    engine.set_params(pk.Params(0.66, 1.6, 14, 0.344, 1440, 0.0695))
    engine.set_background_cache(False)
    keys = ("pairs_bg", "pairs_tr", "pairs_any", "exec_bg", "exec_geom", "exec_sym", "exec_far")
    sh = pk.Engine((0, 0, 0))
    sh.load(ev)
    sh.set_params(pk.Params(0.66, 1.6, 14, 0.344, 1440, 0.0695))
    sh.set_background_cache(False)
    try:
        base = engine.loglik_grad()
        counts = []
        for eng in (engine, engine, sh, sh, engine):
            eng.set_timing(True)
            r = eng.loglik_grad()
            st = eng.stats()
            eng.set_timing(False)
            counts.append(tuple(st[q] for q in keys))
            assert r[0] == base[0] and np.array_equal(r[2], base[2])
        assert counts[0][0] > 0 and len(set(counts)) == 1, counts
        for eng in (engine, sh):
            eng.loglik_grad()  # untimed: counters untouched, reported as 0
            assert all(eng.stats()[q] == 0 for q in keys)
    finally:
        sh.close()
        engine.set_timing(False)
        engine.set_background_cache(True)


def test_per_event_sums_to_total(engine):
    # test_likelihood.cpp:134-146
    ev = pk.generateBenchmarkCloud(120, pk.SimWindow(0, 4, 0, 4, 60), 5)
    r = pk.logLikelihood(ev, pk.Params(0.9, 1.1, 5.0, 0.4, 1.3, 0.5), keepPerEvent=True,
                         engine=engine)
    assert r.valid and r.perEvent.size == 120
    assert abs(r.perEvent.sum() - r.logLik) <= 1e-12 * 120


def test_underflow_invalid_and_invalid_params(engine):
    # test_likelihood.cpp:148-175
    ev = pk.EventSet([0.0, 1.0], [0.0, 0.0], [0.0, 1.0])
    r, g = pk.logLikelihoodGradient(ev, pk.Params(5e-324, 1e120, 1e120, 0.0, 1.0, 1.0),
                                    engine=engine)
    assert not r.valid and r.logLik == -math.inf and np.all(np.isnan(g))
    with pytest.raises(ValueError):
        pk.logLikelihood(ev, pk.Params(omega=-1.0), engine=engine)


def test_batch_bitwise_equals_single(engine):
    # test_likelihood.cpp:224-247
    ev = pk.generateBenchmarkCloud(100, pk.SimWindow(0, 4, 0, 4, 60), 55)
    rng = np.random.default_rng(56)
    plist = [_rand_params(rng) for _ in range(3)]
    plist.append(plist[0])
    engine.load(ev)
    ll, ok, g = engine.loglik_batch([p.as_array() for p in plist], grad=True)
    for i, p in enumerate(plist):
        engine.set_params(p)
        s = engine.loglik_grad()
        assert ll[i] == s[0] and np.array_equal(g[i], s[2])
    assert ll[0] == ll[3]
    with pytest.raises(ValueError):
        engine.loglik_batch(np.zeros((0, 6)))


def test_ties_strict_time_rule(engine):
    """Equal timestamps never excite each other (kernels.hpp:44): the C2
    tie-stress variant (times floored to whole seconds), vs the oracle."""
    ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                      pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005,
                                      keep=3000)
    t = np.floor(ev.ts() * 86400.0) / 86400.0
    ev2 = pk.EventSet(ev.xs(), ev.ys(), t)
    assert np.sum(np.diff(t) == 0) > 0
    for p in (pk.Params(0.66, 1.6, 14, 0.344, 1440, 0.0695), pk.Params(1, 1.6, 14, 0.1, 1, 1)):
        _check(engine, ev2, p)


@pytest.mark.parametrize("mode", [0, 1])
def test_both_kernels_vs_oracle(engine, mode):
    """Rows kernel (ordered pairs) and symmetric-background kernel each match
    the oracle on C1 and on DC-shaped data at both thetas."""
    engine.set_kernel(mode)
    try:
        ev = pk.generateBenchmarkCloud(1000, pk.SimWindow(0, 4, 0, 4, 60), 1000)
        _check(engine, ev, pk.Params(0.6, 0.9, 3.0, 0.5, 1.1, 0.35))
        ev2, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                           pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005,
                                           keep=5000)
        for p in (pk.Params(0.66, 1.6, 14, 0.344, 1440, 0.0695), pk.Params(1, 1.6, 14, 0.1, 1, 1)):
            _check(engine, ev2, p)
        rng = np.random.default_rng(99)
        for n in (1, 2, 7, 129, 300):
            evr = pk.generateBenchmarkCloud(n, pk.SimWindow(0, 4, 0, 4, 60), 500 + n)
            _check(engine, evr, _rand_params(rng))
    finally:
        engine.set_kernel(1)


def test_kernel_modes_agree_and_cull_exact(engine):
    ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                      pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005,
                                      keep=30000)
    engine.load(ev)
    for p in (pk.Params(0.66, 1.6, 14, 0.344, 1440, 0.0695), pk.Params(1, 1.6, 14, 0.1, 1, 1)):
        engine.set_params(p)
        res = {}
        for mode in (0, 1):
            engine.set_kernel(mode)
            engine.set_dense(False)
            a = engine.loglik_grad()
            engine.set_dense(True)
            b = engine.loglik_grad()
            engine.set_dense(False)
            assert a[0] == b[0] and np.array_equal(a[2], b[2])  # culling is exact
            res[mode] = a
        engine.set_kernel(1)
        assert abs(res[0][0] - res[1][0]) <= 1e-13 * abs(res[0][0])
        assert np.allclose(res[0][2], res[1][2], rtol=1e-11, atol=0)


def test_background_cache_bitwise_transparent(engine):
    """Reusing background sums (tauX, tauT unchanged) gives bitwise the same
    loglik / gradient / per-event terms as full evaluations."""
    ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                      pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005,
                                      keep=12000)
    seq = [pk.Params(0.66, 1.6, 14, 0.344, 1440, 0.0695), pk.Params(0.7, 1.6, 14, 0.344, 1440, 0.0695),
           pk.Params(0.7, 1.6, 14, 0.2, 1440, 0.0695), pk.Params(0.7, 1.6, 14, 0.2, 3.0, 0.0695),
           pk.Params(0.7, 1.6, 14, 0.2, 3.0, 0.5), pk.Params(0.7, 1.2, 14, 0.2, 3.0, 0.5),
           pk.Params(0.7, 1.2, 14, 0.2, 1.0, 0.5)]
    for mode in (1, 0):
        engine.set_kernel(mode)
        engine.load(ev)
        outs = {}
        for cache in (False, True):
            engine.set_background_cache(cache)
            res, hits = [], []
            for grad in (True, False):
                for p in seq:
                    engine.set_params(p)
                    r = engine.loglik_grad(per_event=True) if grad else engine.loglik(per_event=True)
                    res.append(r)
                    hits.append(engine.stats()["cache_hit"])
            outs[cache] = (res, hits)
        engine.set_background_cache(True)
        engine.set_kernel(1)
        for a, b in zip(outs[False][0], outs[True][0]):
            assert a[0] == b[0]
            assert np.array_equal(a[-1], b[-1])
            if len(a) == 4:
                assert np.array_equal(a[2], b[2])
        # hits: tauX change at index 5 forces a full sweep, and so does a move
        # of omega across a trigger-free-split threshold (1440 -> 3 moves the
        # split structure); grad->value reuses
        assert sum(outs[True][1]) >= 8 and sum(outs[False][1]) == 0


def _ulp_err(got, want):
    return np.abs(got - want) / np.spacing(np.abs(want))


def test_exp_l_accuracy(engine):
    """The pair kernels' exp (2048-entry table + degree-3 polynomial, sthk_device.cuh)
    against an extended-precision exp: <= 2 ulp (the reference's Pack exp bound,
    test_pack.cpp:21-46) over the live range, exact +0 below -708.40 (the flush the
    exact culling relies on), 1 at 0."""
    import ctypes
    lib = pk.load_library()
    rng = np.random.default_rng(7)
    x = np.concatenate([-rng.uniform(0, 708.3, 200_000), -rng.uniform(0, 1e-3, 20_000),
                        -np.logspace(-12, 2.85, 20_000), [0.0, -708.3, -708.41, -745.0, -1e6]])
    out = np.empty_like(x)
    dp = ctypes.POINTER(ctypes.c_double)
    rc = lib.sthk_debug_exp(0, x.ctypes.data_as(dp), x.size, out.ctypes.data_as(dp))
    assert rc == 0
    live = x >= -708.3
    want = np.exp(x[live].astype(np.longdouble)).astype(np.float64)
    # one extra rounding: the argument is scaled to L units (x * 2048/ln2)
    # in double, an error of ~|x| * 2^-53 relative, i.e. up to ~700 * 1.1e-16
    arg_err = np.abs(x[live]) * 2.0 ** -53 / np.spacing(1.0) * 2
    err = _ulp_err(out[live], want)
    assert np.all(err <= 2.0 + arg_err), float(np.max(err - arg_err))
    small = live & (x > -1.0)
    assert np.max(_ulp_err(out[small], np.exp(x[small].astype(np.longdouble)).astype(np.float64))) <= 2.0
    assert out[x.size - 5] == 1.0
    assert np.all(out[x < -708.41] == 0.0)


def test_trigger_cache_and_plan_cache_bitwise_transparent(engine):
    """MH-style moves with the sweep caches on: mu0 / theta moves reuse the
    trigger sums too (finalize only), h moves reuse the work plan; every
    result is bitwise the result of a full evaluation."""
    ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                      pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005,
                                      keep=9000)
    base = [0.66, 1.6, 14, 0.344, 1440, 0.0695]
    seq = []
    rng = np.random.default_rng(3)
    cur = list(base)
    for _ in range(24):
        k = [0, 3, 4, 5][int(rng.integers(4))]
        cur = list(cur)
        cur[k] *= float(np.exp(0.05 * rng.standard_normal()))
        seq.append((pk.Params(*cur), bool(rng.integers(2))))
    seq.append((pk.Params(*cur), True))   # repeat: grad after a possibly value-only sweep
    seq.append((pk.Params(*cur), False))
    engine.load(ev)
    out = {}
    for cache in (False, True):
        engine.set_background_cache(cache)
        res, hits = [], []
        for p, grad in seq:
            engine.set_params(p)
            r = engine.loglik_grad(per_event=True) if grad else engine.loglik(per_event=True)
            res.append(r)
            st = engine.stats()
            hits.append((st["cache_hit"], st["trigger_cache_hit"]))
        out[cache] = (res, hits)
    engine.set_background_cache(True)
    for a, b in zip(out[False][0], out[True][0]):
        assert a[0] == b[0]
        assert np.array_equal(a[-1], b[-1])
        if len(a) == 4:
            assert np.array_equal(a[2], b[2])
    assert sum(h[1] for h in out[False][1]) == 0
    assert sum(h[1] for h in out[True][1]) >= 4


def test_grouped_batch_shares_sweeps_bitwise(engine):
    """f3: a profile/grid batch (mu0, theta varied over a few (omega, h)
    pairs, shuffled) evaluated in one call is bitwise the single calls with
    every cache off, for value and gradient batches."""
    ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                      pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005,
                                      keep=7000)
    rng = np.random.default_rng(11)
    plist = []
    for om, h in [(1440.0, 0.0695), (500.0, 0.1), (1440.0, 0.2)]:
        for _ in range(5):
            plist.append([rng.uniform(0.3, 1.0), 1.6, 14.0, rng.uniform(0.1, 0.6), om, h])
    plist.append([0.7, 1.3, 12.0, 0.3, 800.0, 0.08])
    order = rng.permutation(len(plist))
    plist = [plist[i] for i in order]
    engine.load(ev)
    engine.set_background_cache(True)
    llb, okb, gb = engine.loglik_batch(plist, grad=True)
    llv, okv, _ = engine.loglik_batch(plist)
    engine.set_background_cache(False)
    try:
        for i, p in enumerate(plist):
            engine.set_params(p)
            s = engine.loglik_grad()
            assert llb[i] == s[0] and np.array_equal(gb[i], s[2])
            v = engine.loglik()
            assert llv[i] == v[0]
    finally:
        engine.set_background_cache(True)
    res = pk.logLikelihoodBatch(ev, [pk.Params(*p) for p in plist], engine=engine)
    assert [r.logLik for r in res] == list(llv)


def test_engine_event_checks_match_reference_messages(engine):
    """sthk_load_events runs the EventSet checks on the device (tile-box pass)
    and reports the reference's message for the first failing index."""
    cases = [
        (([0, 1, 2], [0, 1, 2], [1.0, 0.5, np.nan], 5.0), "times not sorted at index 1"),
        (([0, np.inf, 2], [0, 1, 2], [1.0, 0.5, 0.2], 5.0), "non-finite entry at index 1"),
        (([0, 1], [0, 1], [1.0, -1.0], 5.0), "negative time at index 1"),
        (([0, 1], [0, 1], [-1.0, 2.0], 5.0), "negative time at index 0"),
        (([0, 1, 2], [0, 1, 2], [0.0, 1.0, 2.0], 1.5), "windowEnd precedes last event"),
    ]
    big_t = np.sort(np.random.default_rng(1).uniform(0, 100, 5000))
    big_t[4321] = big_t[4320] - 1e-9
    cases.append(((np.zeros(5000), np.zeros(5000), big_t, 200.0), "times not sorted at index 4321"))
    import torch

    def pinned(a):  # (pinned host arrays take the zero-copy load kernel)
        return torch.from_numpy(np.asarray(a, float)).pin_memory().numpy()

    for (x, y, t, we), msg in cases:
        for conv in (lambda a: np.asarray(a, float), pinned):
            with pytest.raises(ValueError, match=msg):
                engine.load_events(conv(x), conv(y), conv(t), we)
    # a failed load leaves the engine without events; a good load recovers
    ev = pk.generateBenchmarkCloud(300, pk.SimWindow(0, 4, 0, 4, 60), 5)
    engine.load(ev)
    engine.set_params(pk.Params(0.6, 0.9, 3.0, 0.5, 1.1, 0.35))
    assert engine.loglik()[1]


def test_far_tier_matches_all_fp64(engine):
    """The FP32 far tier (stages whose every exponent is provably < -40) changes
    nothing the FP64 sums can see: far on vs far off (every pair in FP64) agree to
    1e-13 on loglik and 1e-11 (scale-aware) on the gradient, at the C2 posterior and
    at the sampler's initial point (ω = 1: far causal trigger stages), value and grad."""
    ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                      pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005,
                                      keep=30000)
    engine.load(ev)
    for theta in ([0.66, 1.6, 14, 0.344, 1440, 0.0695], [1, 1.6, 14, 0.1, 1, 1],
                  [0.5, 0.7, 3.0, 0.3, 20.0, 0.3]):
        engine.set_params(theta)
        out = {}
        for far in (1, 0):
            engine.set_far_tier(bool(far))
            engine.set_timing(True)
            out[far] = (engine.loglik_grad(), engine.stats()["exec_far"], engine.loglik()[0])
            engine.set_timing(False)
        engine.set_far_tier(True)
        (a, nfar, va), (b, nfar0, vb) = out[1], out[0]
        assert nfar > 0 and nfar0 == 0, (theta, nfar)
        assert abs(a[0] - b[0]) <= 1e-13 * abs(b[0]) and abs(va - vb) <= 1e-13 * abs(vb)
        o = og.oracle_loglik_grad(ev.xs(), ev.ys(), ev.ts(), ev.windowEnd(), np.array(theta))
        assert np.all(np.abs(a[2] - b[2]) <= 1e-11 * o["grad_abs"]), (a[2], b[2])


def test_far_tier_guard_off_for_extreme_coordinates(engine):
    """FP32 coordinates must stay small in kernel units: a spatial extent of
    ~1e4 tauX turns the far tier off (every pair FP64); a time span of ~500 tauT
    keeps it on (times are tile-relative, only the 128-event tile span counts);
    results match the oracle either way."""
    rng = np.random.default_rng(4)
    n = 12000
    for xs, tspan, want_far in ((5.0, 1800.0, True), (3e4, 1800.0, False)):
        t = np.sort(rng.uniform(0, tspan, n))
        ev = pk.EventSet(rng.uniform(0, xs, n), rng.uniform(0, 5, n), t)
        # (tauT = 60 days: the far band [tfar, dBf] = [8.9, 9.7] tauT holds a few
        # whole 128-event stages at this event density)
        p = pk.Params(0.6, 0.9, 60.0, 0.3, 2.0, 0.3)
        engine.load(ev)
        engine.set_params(p)
        engine.set_timing(True)
        r = engine.loglik_grad()
        assert (engine.stats()["exec_far"] > 0) == want_far
        engine.set_timing(False)
        o = og.oracle_loglik_grad(ev.xs(), ev.ys(), ev.ts(), ev.windowEnd(), p.as_array())
        assert abs(r[0] - o["loglik"]) <= 1e-10 * abs(o["loglik"])


def test_far_schedule_bitwise_invariant(engine):
    """The near (FP64) and far (FP32) kernels write disjoint trigger partials and
    add background sums as integers: concurrent or sequential schedules, any CTA
    counts, give bitwise-identical results."""
    ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                      pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005,
                                      keep=20000)
    engine.load(ev)
    engine.set_background_cache(False)
    try:
        res = []
        for sched in ((True, 3, 6), (False, 3, 6), (True, 1, 3), (True, 2, 1)):
            engine.set_far_schedule(*sched)
            for theta in ([0.66, 1.6, 14, 0.344, 1440, 0.0695], [1, 1.6, 14, 0.1, 1, 1]):
                engine.set_params(theta)
                r = engine.loglik_grad()
                res.append((sched, theta[4], r[0], tuple(r[2])))
        base = {om: (ll, g) for s, om, ll, g in res if s == (True, 3, 6)}
        for s, om, ll, g in res:
            assert (ll, g) == base[om], s
    finally:
        engine.set_far_schedule(True, 3, 6)
        engine.set_background_cache(True)


def _clustered_events(rng, n, t_end, tau_hot=0.5):
    """Bursty synthetic set: a Poisson background plus tight space-time bursts."""
    k = max(1, n // 20)
    cx, cy, ct = rng.uniform(0, 10, k), rng.uniform(0, 10, k), rng.uniform(0, t_end, k)
    pick = rng.integers(0, k, n // 2)
    x = np.concatenate([rng.uniform(0, 10, n - n // 2), cx[pick] + 0.05 * rng.standard_normal(n // 2)])
    y = np.concatenate([rng.uniform(0, 10, n - n // 2), cy[pick] + 0.05 * rng.standard_normal(n // 2)])
    t = np.concatenate([rng.uniform(0, t_end, n - n // 2),
                        np.clip(ct[pick] + tau_hot * rng.exponential(1.0, n // 2), 0, t_end)])
    return pk.EventSet.sortedByTime(x, y, t)


@pytest.mark.parametrize("seed", range(8))
def test_random_regimes_vs_oracle(engine, seed):
    """Fuzz across parameter regimes (small / large tauT, omega from 0.05 to 5000,
    theta up to 0.95, tiny h) and bursty data: the full engine (far tier, caches,
    both kernels' stage modes) against the long-double oracle at the north-star
    tolerances."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1500, 6000))
    ev = _clustered_events(rng, n, float(rng.choice([50.0, 500.0, 3000.0])))
    p = pk.Params(float(rng.uniform(0.05, 3.0)), float(rng.uniform(0.2, 3.0)),
                  float(np.exp(rng.uniform(np.log(0.5), np.log(60.0)))),
                  float(rng.uniform(0.0, 0.95)),
                  float(np.exp(rng.uniform(np.log(0.05), np.log(5000.0)))),
                  float(np.exp(rng.uniform(np.log(0.01), np.log(2.0)))))
    _check(engine, ev, p)


def test_bgonly_kernel_consistent(engine):
    """Near stages beyond the trigger window run in the trigger-free kernel (from
    36k events). With
    it on, results are bitwise identical with the caches on or off; against the
    single near kernel they differ only by the grouping of the per-item FP64 row
    partials (<= 1e-14 relative)."""
    ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                      pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005,
                                      keep=70000)
    engine.load(ev)
    seq = [[0.66, 1.6, 14, 0.344, 1440, 0.0695], [0.7, 1.6, 14, 0.344, 1440, 0.0695],
           [0.7, 1.6, 14, 0.344, 30.0, 0.0695], [1, 1.6, 14, 0.1, 1, 1]]
    out = {}
    try:
        for split in (True, False):
            engine.set_bgonly_kernel(split)
            for cache in (False, True):
                engine.set_background_cache(cache)
                res = []
                for p in seq:
                    engine.set_params(p)
                    r = engine.loglik_grad()
                    res.append((r[0], tuple(r[2])))
                out[(split, cache)] = res
    finally:
        engine.set_bgonly_kernel(True)
        engine.set_background_cache(True)
    assert out[(True, True)] == out[(True, False)]
    assert out[(False, True)] == out[(False, False)]
    for (a, ga), (b, gb) in zip(out[(True, False)], out[(False, False)]):
        assert abs(a - b) <= 1e-14 * abs(b)
        assert np.allclose(ga, gb, rtol=1e-11, atol=0)


def _c2(keep=85000):
    ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                      pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005,
                                      keep=keep)
    return ev


@pytest.mark.parametrize("theta", [(0.66, 1.6, 14, 0.344, 1440, 0.0695), (1, 1.6, 14, 0.1, 1, 1)])
def test_full_size_c2_matches_reference_engine(engine, theta):
    """The bench workload itself (C2, N = 85,000) against the verbatim reference
    engine on all host cores: loglik to 1e-10 and every per-event term to 1e-12
    (absolute, or relative above 1)."""
    if not og.ref_available():
        pytest.skip("oracle/_ref not built")
    ev = _c2()
    lanes = 8 if og.has_avx512() else 4
    ref, ok, ref_pe = og.ref_loglik(ev.xs(), ev.ys(), ev.ts(), ev.windowEnd(), np.array(theta),
                                    os.cpu_count() or 1, lanes, per_event=True)
    engine.load(ev)
    engine.set_params(list(theta))
    ll, valid, pe = engine.loglik(per_event=True)
    assert ok and valid
    assert abs(ll - ref) <= LL_TOL * abs(ref), (ll, ref)
    assert np.all(np.abs(pe - ref_pe) <= 1e-12 * np.maximum(1.0, np.abs(ref_pe)))


def test_full_size_properties(engine):
    """Size-independent properties at the bench size (C2, N = 85,000, loglik +
    gradient): repeat-bitwise, culled == dense bitwise, 4 emulated ranks bitwise,
    per-event terms summing to the total, far tier vs all-FP64 to 1e-13."""
    ev = _c2()
    engine.load(ev)
    engine.set_params([0.66, 1.6, 14, 0.344, 1440, 0.0695])
    engine.set_background_cache(False)
    try:
        a = engine.loglik_grad(per_event=True)
        b = engine.loglik_grad(per_event=True)
        assert a[0] == b[0] and np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3])
        engine.set_dense(True)
        d = engine.loglik_grad()
        engine.set_dense(False)
        assert d[0] == a[0] and np.array_equal(d[2], a[2])
        with pk.Engine((0,) * 4) as sh:
            sh.load(ev)
            sh.set_params([0.66, 1.6, 14, 0.344, 1440, 0.0695])
            s = sh.loglik_grad(per_event=True)
        assert s[0] == a[0] and np.array_equal(s[2], a[2]) and np.array_equal(s[3], a[3])
        assert abs(math.fsum(a[3]) - a[0]) <= 1e-12 * abs(a[0])
        engine.set_far_tier(False)
        f = engine.loglik_grad()
        engine.set_far_tier(True)
        assert abs(f[0] - a[0]) <= 1e-13 * abs(a[0])
        assert np.all(np.abs(f[2] - a[2]) <= 1e-11 * np.abs(a[2]) + 1e-9)
    finally:
        engine.set_dense(False)
        engine.set_far_tier(True)
        engine.set_background_cache(True)


def test_c3_250k_matches_reference_engine(engine):
    """The largest C3 sweep point (generateBenchmarkCloud, N = 250,000) against
    the verbatim reference engine on all host cores, loglik to 1e-10."""
    if not og.ref_available():
        pytest.skip("oracle/_ref not built")
    n = 250000
    ev = pk.generateBenchmarkCloud(n, pk.SimWindow(0, 15, 0, 15, 4750), n)
    theta = np.array([0.66, 1.6, 14, 0.344, 1440, 0.0695])
    ref, ok, _ = og.ref_loglik(ev.xs(), ev.ys(), ev.ts(), ev.windowEnd(), theta,
                               os.cpu_count() or 1, 8 if og.has_avx512() else 4)
    engine.load(ev)
    engine.set_params(list(theta))
    ll, valid, _ = engine.loglik()
    assert ok and valid and abs(ll - ref) <= LL_TOL * abs(ref), (ll, ref)


def test_c4_1m_properties(engine):
    """C4 size (N = 1,000,000, one GPU): bitwise repeatable, per-event terms
    summing to the total (the 2/3/8-rank split: test_multirank_gpu.py)."""
    n = 1000000
    ev = pk.generateBenchmarkCloud(n, pk.SimWindow(0, 15, 0, 15, 4750), n)
    engine.load(ev)
    engine.set_params([0.66, 1.6, 14, 0.344, 1440, 0.0695])
    engine.set_background_cache(False)
    try:
        a = engine.loglik_grad(per_event=True)
        b = engine.loglik_grad()
        assert a[1] and a[0] == b[0]
        assert np.array_equal(a[2], b[2])
        assert abs(math.fsum(a[3]) - a[0]) <= 1e-12 * abs(a[0])
    finally:
        engine.set_background_cache(True)


@pytest.mark.parametrize("theta", [(0.66, 1.6, 14, 0.344, 1440, 0.0695), (1, 1.6, 14, 0.1, 1, 1)])
def test_c2_shaped_gradient_vs_oracle(engine, theta):
    """Gradient parity on C2-shaped data (first 30,000 events of the bench set:
    the far tier, the trigger-free split and culling all active) against the
    long-double oracle: loglik to 1e-10, each component to 1e-8 of its
    scale (sum of |per-event contributions|) and, away from a stationary point,
    to 1e-8 relative."""
    ev = _c2(keep=30000)
    o = og.oracle_loglik_grad(ev.xs(), ev.ys(), ev.ts(), ev.windowEnd(), np.array(theta))
    engine.load(ev)
    engine.set_params(list(theta))
    ll, valid, g, _ = engine.loglik_grad()
    assert valid and o["valid"]
    assert abs(ll - o["loglik"]) <= LL_TOL * abs(o["loglik"])
    assert np.all(np.abs(g - o["grad"]) <= 1e-8 * o["grad_abs"]), (g, o["grad"])
    big = np.abs(o["grad"]) > 1e-3 * o["grad_abs"]
    assert np.all(np.abs(g - o["grad"])[big] <= 1e-8 * np.abs(o["grad"])[big])


@pytest.mark.parametrize("theta", [(0.66, 1.6, 14, 0.344, 1440, 0.0695), (1, 1.6, 14, 0.1, 1, 1)])
def test_c2_full_size_gradient_vs_oracle(engine, theta):
    """The bench's own GRAD kernels at the bench size (C2, N = 85,000: far tier,
    trigger-free split and culling all active) against the long-double oracle:
    loglik to 1e-10, every gradient component to 1e-8 of its scale and, away
    from a stationary point, to 1e-8 relative."""
    ev = _c2()
    o = og.oracle_loglik_grad(ev.xs(), ev.ys(), ev.ts(), ev.windowEnd(), np.array(theta))
    engine.load(ev)
    engine.set_params(list(theta))
    ll, valid, g, _ = engine.loglik_grad()
    assert valid and o["valid"]
    assert abs(ll - o["loglik"]) <= LL_TOL * abs(o["loglik"]), (ll, o["loglik"])
    assert np.all(np.abs(g - o["grad"]) <= G_TOL * o["grad_abs"]), (g, o["grad"])
    big = np.abs(o["grad"]) > 1e-3 * o["grad_abs"]
    assert np.all(np.abs(g - o["grad"])[big] <= G_TOL * np.abs(o["grad"])[big]), (g, o["grad"])


def test_c3_250k_theta_init_matches_reference_engine(engine):
    """The largest C3 point at the sampler's initial Theta (omega = 1: the causal
    trigger live over ~50 days) against the verbatim reference engine."""
    if not og.ref_available():
        pytest.skip("oracle/_ref not built")
    n = 250000
    ev = pk.generateBenchmarkCloud(n, pk.SimWindow(0, 15, 0, 15, 4750), n)
    theta = np.array([1.0, 1.6, 14, 0.1, 1.0, 1.0])
    ref, ok, _ = og.ref_loglik(ev.xs(), ev.ys(), ev.ts(), ev.windowEnd(), theta,
                               os.cpu_count() or 1, 8 if og.has_avx512() else 4)
    engine.load(ev)
    engine.set_params(list(theta))
    ll, valid, _ = engine.loglik()
    assert ok and valid and abs(ll - ref) <= LL_TOL * abs(ref), (ll, ref)


def test_c4_1m_matches_reference_engine(engine):
    """C4 (N = 1,000,000) against the verbatim reference engine on every host
    core (dense O(N^2) on the CPU: a few minutes), loglik to 1e-10."""
    if not og.ref_available():
        pytest.skip("oracle/_ref not built")
    n = 1000000
    ev = pk.generateBenchmarkCloud(n, pk.SimWindow(0, 15, 0, 15, 4750), n)
    theta = np.array([0.66, 1.6, 14, 0.344, 1440, 0.0695])
    engine.load(ev)
    engine.set_params(list(theta))
    ll, valid, _ = engine.loglik()
    ref, ok, _ = og.ref_loglik(ev.xs(), ev.ys(), ev.ts(), ev.windowEnd(), theta,
                               os.cpu_count() or 1, 8 if og.has_avx512() else 4)
    assert ok and valid and abs(ll - ref) <= LL_TOL * abs(ref), (ll, ref)


@pytest.mark.parametrize("seed", range(4))
def test_far_tier_stress_bursty_random_theta(engine, seed):
    """Adversarial far tier: N >= 30k bursty events, random Theta from regimes
    where the far tier is live (asserted through its pair counter): far on vs
    every pair in FP64 within the claimed 1e-13 (loglik) and against the
    long-double oracle at the north-star tolerances."""
    rng = np.random.default_rng(77 + seed)
    n = int(rng.integers(30000, 40000))
    ev = _clustered_events(rng, n, float(rng.choice([800.0, 2000.0, 4000.0])), tau_hot=2.0)
    for _ in range(12):
        p = pk.Params(float(rng.uniform(0.2, 3.0)), float(rng.uniform(0.3, 3.0)),
                      float(np.exp(rng.uniform(np.log(1.0), np.log(30.0)))),
                      float(rng.uniform(0.05, 0.95)),
                      float(np.exp(rng.uniform(np.log(0.3), np.log(3000.0)))),
                      float(np.exp(rng.uniform(np.log(0.02), np.log(1.0)))))
        engine.load(ev)
        engine.set_params(p)
        engine.set_timing(True)
        a = engine.loglik_grad()
        nfar = engine.stats()["exec_far"]
        engine.set_timing(False)
        if nfar > 0:
            break
    assert nfar > 0, "no far-tier work at any drawn Theta"
    engine.set_far_tier(False)
    try:
        b = engine.loglik_grad()
    finally:
        engine.set_far_tier(True)
    assert a[1] == b[1]
    if b[1]:
        assert abs(a[0] - b[0]) <= 1e-13 * abs(b[0]), (a[0], b[0])
    _check(engine, ev, p)


def test_trigger_cache_far_split_flip_bitwise(engine):
    """with the trigger sums cached, a theta / mu0 step that
    moves the trigger boost across the far tier's trigger window (tauT = 14,
    omega = 0.5: dTf crosses tfar near boost 7.3) must not reuse a sweep whose
    far trigger partials were never stored. Cached == full evaluation, bitwise,
    along a theta ladder across the crossing."""
    ev = _c2(keep=30000)
    engine.load(ev)
    seq = []
    for mu0 in (0.5, 1.0, 2.0):  # boost = ln(9300 theta / mu0): 5.4 .. 11.4
        for th in np.geomspace(0.05, 5.0, 9):
            seq.append([mu0, 1.6, 14.0, float(th), 0.5, 0.0695])
    full, cached = [], []
    engine.set_background_cache(False)
    for p in seq:
        engine.set_params(p)
        full.append(engine.loglik_grad())
    engine.set_background_cache(True)
    hits = 0
    for p in seq:
        engine.set_params(p)
        cached.append(engine.loglik_grad())
        hits += engine.stats()["trigger_cache_hit"]
    assert hits > 0
    for p, a, b in zip(seq, full, cached):
        assert a[0] == b[0] and np.array_equal(a[2], b[2]), p


def test_extreme_trigger_boost_keeps_trigger_in_fp64(engine):
    """trNorm / (mu0 bgNorm) ~ e^45 puts trigger terms that
    matter below the FP32 flush point; they must stay in the FP64 near list.
    Against the long-double oracle and the all-FP64 path."""
    ev = _c2(keep=20000)
    # boost = ln(theta omega / (2 pi h^2) / (mu0 (2pi)^-1.5 / (tauX^2 tauT)))
    p = pk.Params(1e-13, 1.6, 14.0, 0.9, 0.5, 0.01)
    cB = p.mu0 * (2 * np.pi) ** -1.5 / (p.tauX ** 2 * p.tauT)
    cT = p.theta * p.omega / (2 * np.pi * p.h ** 2)
    assert np.log(cT / cB) > 40
    r, g, o = _check(engine, ev, p)
    engine.set_far_tier(False)
    try:
        b = engine.loglik_grad()
    finally:
        engine.set_far_tier(True)
    if o["valid"]:
        assert abs(r.logLik - b[0]) <= 1e-13 * abs(b[0])


def test_rejects_more_events_than_fixed_point_range(engine):
    """The fixed-point background sums hold per-row totals below 2^23 (a row's
    S_B can reach N): loads beyond 2^23 events are refused, not wrapped."""
    n = (1 << 23) + 1
    t = np.arange(n, dtype=np.float64) * 1e-3
    z = np.zeros(n)
    with pytest.raises(ValueError, match="at most 2\\^23 events"):
        engine.load_events(z, z, t, float(t[-1]))
    ev = pk.generateBenchmarkCloud(300, pk.SimWindow(0, 4, 0, 4, 60), 5)
    engine.load(ev)  # (the engine still works)


def test_far_list_in_fp64_same_windows(engine):
    """sthk_set_far_tier(2): the far list evaluated by the FP64 kernel with the
    far tier's windows. Against the FP32 far tier it differs only by the far
    terms' FP32 rounding (<= 1e-13 on loglik); against no far tier at all only
    by terms below half an ulp of lambda."""
    ev = _c2(keep=40000)
    engine.load(ev)
    for theta in ([0.66, 1.6, 14, 0.344, 1440, 0.0695], [1, 1.6, 14, 0.1, 1, 1]):
        engine.set_params(theta)
        res = {}
        try:
            for mode in (1, 2, 0):
                engine.set_far_tier(mode)
                engine.set_timing(True)
                res[mode] = (engine.loglik_grad(), engine.stats()["exec_far"])
                engine.set_timing(False)
        finally:
            engine.set_far_tier(1)
        (a, fa), (b, fb), (c, fc) = res[1], res[2], res[0]
        assert fa > 0 and fb == 0 and fc == 0
        assert abs(a[0] - b[0]) <= 1e-13 * abs(b[0]) and abs(b[0] - c[0]) <= 1e-14 * abs(c[0])
        o = og.oracle_loglik_grad(ev.xs(), ev.ys(), ev.ts(), ev.windowEnd(), np.array(theta))
        assert np.all(np.abs(b[2] - c[2]) <= 1e-12 * o["grad_abs"])


@pytest.mark.parametrize("n", [3000, 40000])
def test_graph_replay_bitwise_equals_direct_launches(n):
    """One-shard evaluations run as cached CUDA graphs (kernel arguments
    updated in place) give bitwise the results of direct launches, across the
    evaluation shapes of an MH chain (full sweep, trigger-only sweep, finalize
    only), per-event terms and the excitation split included; the graph cache
    builds each shape once."""
    ev = _c2(n)
    rng = np.random.default_rng(n)
    theta = [0.66, 1.6, 14, 0.344, 1440, 0.0695]
    seq = [list(theta)]
    for _ in range(24):
        k = [0, 3, 4, 5][int(rng.integers(4))]
        cand = list(seq[-1])
        cand[k] *= float(np.exp(0.05 * rng.standard_normal()))
        seq.append(cand)
    out = {}
    for graphs in (True, False):
        e = pk.Engine((0,))
        e.set_graphs(graphs)
        e.load(ev)
        res = []
        for i, p in enumerate(seq):
            e.set_params(p)
            if i % 5 == 4:
                ll, ok, pe = e.loglik(per_event=True)
                res.append((ll, ok, tuple(pe)))
            else:
                ll, ok, g, _ = e.loglik_grad()
                res.append((ll, ok, tuple(g)))
        e.set_background_cache(False)
        e.set_params(seq[-1])
        res.append(tuple(e.loglik_grad()[2]))
        mu, xi, pi = e.excitation()
        res.append((tuple(mu), tuple(pi)))
        st = e.stats()
        out[graphs] = res
        if graphs:
            assert st["graph_launches"] > 0
            assert st["graph_builds"] <= 10, st["graph_builds"]
        e.close()
    assert out[True] == out[False]


_PIVOT_SCRIPT = r"""
import hashlib, json, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
import paper_2005_10123_b200 as pk
out = []
for n, th in ((85000, [0.66, 1.6, 14, 0.344, 1440, 0.0695]), (85000, [1, 1.6, 14, 0.1, 1, 1]),
              (6000, [0.66, 1.6, 14, 0.344, 1440, 0.0695])):
    ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                      pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005, keep=n)
    e = pk.Engine((0,))
    e.set_background_cache(False)
    e.load(ev)
    e.set_params(th)
    ll, ok, g, pe = e.loglik_grad(per_event=True)
    out.append([ll.hex(), [float(v).hex() for v in g], hashlib.sha256(pe.tobytes()).hexdigest()])
    e.close()
print(json.dumps(out))
"""


def test_tile_pivot_plan_bitwise_equals_strided_plan():
    """The plan's tile-granular searches (tile last times as pivots, no global
    rounds) and the exact strided-pivot searches give the same stage sets,
    hence bitwise-identical loglik, gradient and per-event terms."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for strided in ("0", "1"):
        env = dict(os.environ, STHK_PLAN_STRIDED=strided)
        r = subprocess.run([sys.executable, "-c", _PIVOT_SCRIPT, root], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[strided] = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["0"] == res["1"]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_shell_bound_culls_bursty_against_oracle(engine, seed):
    """The half-ulp culls bound the skipped terms by shells of the load-time
    window statistics. Bursty data puts many events just beyond
    each cut; against the long-double oracle (which keeps every term above
    e^-100 of the self term) the loglik must agree to 1e-12 relative -- far
    inside the 1e-10 contract, at the level of FP64 accumulation noise -- with
    the far tier active, at long trigger windows (small omega) and with a
    large trigger boost."""
    rng = np.random.default_rng(100 + seed)
    bursts = rng.uniform(0, 3000, 60)
    t = np.sort(np.concatenate([b + np.cumsum(rng.exponential(0.05, 400)) for b in bursts]))
    n = t.size
    x = rng.normal(7.5, 2.0, n) + rng.normal(0, 0.3, n)
    y = rng.normal(7.5, 2.0, n) + rng.normal(0, 0.3, n)
    ev = pk.EventSet(x, y, t)
    engine.load(ev)
    for theta in ([0.66, 1.6, 14, 0.344, 1440, 0.0695],   # C2 posterior
                  [0.8, 1.2, 9.0, 0.4, 0.2, 0.5],          # 0.2/day: trigger window ~ 230 days
                  [1e-3, 1.0, 20.0, 0.9, 3.0, 0.05]):      # large boost (trNorm >> mu0 bgNorm)
        engine.set_params(theta)
        engine.set_timing(True)
        ll, ok, g, _ = engine.loglik_grad()
        st = engine.stats()
        engine.set_timing(False)
        o = og.oracle_loglik_grad(ev.xs(), ev.ys(), ev.ts(), ev.windowEnd(), np.array(theta))
        assert ok and o["valid"]
        assert abs(ll - o["loglik"]) <= 1e-12 * abs(o["loglik"]), (theta, ll, o["loglik"], st["exec_far"])
        assert np.all(np.abs(g - o["grad"]) <= 1e-10 * o["grad_abs"]), (theta, g, o["grad"])


def test_pinned_zero_copy_load_bitwise_equals_pageable_load(engine):
    """Pinned host arrays are read by the load kernel itself over PCIe
    (zero-copy); pageable ones are copied first. Same device data, same load
    statistics, bitwise-identical results (C2 at both Theta and a partial tile)."""
    import torch
    for keep in (85000, 85000 - 77):
        ev = _c2(keep)
        res = []
        for pin in (False, True):
            x, y, t = ev.xs(), ev.ys(), ev.ts()
            if pin:
                x, y, t = (torch.from_numpy(np.array(a, dtype=np.float64)).pin_memory().numpy() for a in (x, y, t))
            engine.load_events(x, y, t, ev.windowEnd())
            out = []
            for th in ([0.66, 1.6, 14, 0.344, 1440, 0.0695], [1, 1.6, 14, 0.1, 1, 1]):
                engine.set_params(th)
                ll, ok, g, pe = engine.loglik_grad(per_event=True)
                out.append((ll, ok, tuple(g), pe.tobytes()))
            res.append(out)
        assert res[0] == res[1]


def test_load_beside_a_running_evaluation_copies_and_matches(engine):
    """A load issued while another engine's evaluation runs on the device
    copies the pinned arrays with the copy engines (the zero-copy gather
    would wait for SM slots); an idle device gets the zero-copy gather.
    Both loads give bitwise-identical results, and the pipelined two-engine
    pattern of bench.py's end-to-end arm returns every step's result."""
    import torch
    import paper_2005_10123_b200 as pk
    ev = _c2(85000)
    x, y, t = (torch.from_numpy(np.array(a, dtype=np.float64)).pin_memory().numpy()
               for a in (ev.xs(), ev.ys(), ev.ts()))
    th = [0.66, 1.6, 14, 0.344, 1440, 0.0695]
    engine.set_background_cache(False)
    engine.load_events(x, y, t, ev.windowEnd())
    assert engine.stats()["load_zero_copy"] == 1
    engine.set_params(th)
    ref = engine.loglik_grad()
    with pk.Engine((0,)) as other:
        other.set_background_cache(False)
        other.load_events(x, y, t, ev.windowEnd())
        other.set_params(th)
        copied = 0
        for _ in range(4):
            other.enqueue(grad=True)
            engine.load_events(x, y, t, ev.windowEnd())
            copied += 1 - engine.stats()["load_zero_copy"]
            engine.set_params(th)
            engine.enqueue(grad=True)
            r_other = other.result()
            r_eng = engine.result()
            for r in (r_other, r_eng):
                assert r[0] == ref[0] and r[1] == ref[1] and tuple(r[2]) == tuple(ref[2])
        assert copied >= 1  # (the first evaluation of 85k events lasts ~0.4 ms)
    engine.set_background_cache(True)


@pytest.mark.parametrize("n", [1, 2, 3, 127, 128, 129, 255, 256, 257, 1023, 1025])
def test_tile_boundary_sizes_against_oracle(engine, n):
    """Event counts around the 128-event tile and 1024-row block boundaries
    (partial tiles, a single event, one row per block): loglik and gradient
    against the long-double oracle, through the graph path and both load
    paths (pinned zero-copy and pageable)."""
    import torch
    rng = np.random.default_rng(n)
    t = np.sort(rng.uniform(0, 40, n))
    x, y = rng.uniform(0, 3, n), rng.uniform(0, 3, n)
    p = np.array([0.7, 0.8, 4.0, 0.4, 1.5, 0.3])
    o = og.oracle_loglik_grad(x, y, t, float(t[-1]) + 1.0, p)
    for pin in (False, True):
        arrs = [np.array(a) for a in (x, y, t)]
        if pin:
            arrs = [torch.from_numpy(a).pin_memory().numpy() for a in arrs]
        engine.load_events(*arrs, float(t[-1]) + 1.0)
        engine.set_params(p)
        ll, ok, g, _ = engine.loglik_grad()
        assert ok == o["valid"]
        assert abs(ll - o["loglik"]) <= 1e-12 * abs(o["loglik"]), (n, pin, ll, o["loglik"])
        assert np.all(np.abs(g - o["grad"]) <= 1e-10 * o["grad_abs"] + 1e-300), (n, pin, g, o["grad"])


def test_full_size_metamorphic_identities(engine):
    """Size-independent identities of the model, checked on the C2 workload
    itself (85,000 events) without an oracle:
      * translation and rotation of space leave loglik and gradient unchanged;
      * scaling space by s with tauX, h scaled alike: loglik - 2 N ln s, and
        d/dtauX, d/dh scale by 1/s;
      * scaling time by s (t, T, tauT scaled; omega / s): loglik - N ln s,
        d/dtauT by 1/s, d/domega by s.
    (to 1e-11 relative: the inputs are rounded differently)"""
    ev = _c2()
    x, y, t, T = ev.xs(), ev.ys(), ev.ts(), ev.windowEnd()
    n = t.size
    for theta in ([0.66, 1.6, 14, 0.344, 1440, 0.0695], [1, 1.6, 14, 0.1, 1, 1]):
        p = np.array(theta)

        def run(xx, yy, tt, TT, pp):
            engine.load_events(np.ascontiguousarray(xx), np.ascontiguousarray(yy),
                               np.ascontiguousarray(tt), TT)
            engine.set_params(pp)
            ll, ok, g, _ = engine.loglik_grad()
            assert ok
            return ll, g.copy()

        ll0, g0 = run(x, y, t, T, p)
        gs = np.abs(g0) + 1e-300

        ang = 0.7
        xr = np.cos(ang) * x - np.sin(ang) * y + 123.456
        yr = np.sin(ang) * x + np.cos(ang) * y - 78.9
        ll1, g1 = run(xr, yr, t, T, p)
        assert abs(ll1 - ll0) <= 1e-11 * abs(ll0), (theta, ll0, ll1)
        assert np.all(np.abs(g1 - g0) <= 1e-9 * gs), (theta, g0, g1)

        s = 1.7
        ps = p.copy()
        ps[1] *= s
        ps[5] *= s
        ll2, g2 = run(s * x, s * y, t, T, ps)
        assert abs(ll2 - (ll0 - 2 * n * np.log(s))) <= 1e-11 * abs(ll0), (theta, ll0, ll2)
        want = g0.copy()
        want[1] /= s
        want[5] /= s
        assert np.all(np.abs(g2 - want) <= 1e-9 * gs), (theta, want, g2)

        st = 2.3
        pt = p.copy()
        pt[2] *= st
        pt[4] /= st
        ll3, g3 = run(x, y, st * t, st * T, pt)
        assert abs(ll3 - (ll0 - n * np.log(st))) <= 1e-11 * abs(ll0), (theta, ll0, ll3)
        want = g0.copy()
        want[2] /= st
        want[4] *= st
        assert np.all(np.abs(g3 - want) <= 1e-9 * gs), (theta, want, g3)


def test_c4_1m_scaling_identities(engine):
    """The space and time scaling identities (see the C2 test above) on the C4
    workload, N = 1,000,000: loglik - 2 N ln s and - N ln s, to 1e-11."""
    ev = pk.generateBenchmarkCloud(1_000_000, pk.SimWindow(0, 15, 0, 15, 4750), 1_000_000)
    x, y, t, T = ev.xs(), ev.ys(), ev.ts(), ev.windowEnd()
    n = t.size
    p = np.array([0.66, 1.6, 14, 0.344, 1440, 0.0695])

    def run(xx, yy, tt, TT, pp):
        engine.load_events(np.ascontiguousarray(xx), np.ascontiguousarray(yy),
                           np.ascontiguousarray(tt), TT)
        engine.set_params(pp)
        ll, ok = engine.loglik()[:2]
        assert ok
        return ll

    ll0 = run(x, y, t, T, p)
    s = 1.7
    ps = p.copy()
    ps[1] *= s
    ps[5] *= s
    assert abs(run(s * x, s * y, t, T, ps) - (ll0 - 2 * n * np.log(s))) <= 1e-11 * abs(ll0)
    st = 2.3
    pt = p.copy()
    pt[2] *= st
    pt[4] /= st
    assert abs(run(x, y, st * t, st * T, pt) - (ll0 - n * np.log(st))) <= 1e-11 * abs(ll0)


_ROWS_SCRIPT = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
import paper_2005_10123_b200 as pk
out = []
for n, th in ((85000, [0.66, 1.6, 14, 0.344, 1440, 0.0695]), (85000, [0.66, 1.6, 14, 0.344, 300, 0.2]),
              (85000, [1, 1.6, 14, 0.1, 1, 1]), (4000, [0.66, 1.6, 14, 0.344, 1440, 0.0695])):
    ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                      pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005, keep=n)
    e = pk.Engine((0,))
    e.set_background_cache(False)
    e.load(ev)
    e.set_params(th)
    ll, ok, g, pe = e.loglik_grad(per_event=True)
    out.append([ll, list(map(float, g)), e.stats()["trigger_rows"]])
    e.close()
print(json.dumps(out))
"""


def test_trigger_rows_match_tiled_sweep_and_oracle(engine):
    """Trigger underflow windows 709/ω shorter than every 128-event tile's
    time span (Θ_post, ω = 1440: half a day) are summed by row windows
    (trig_rows_kernel): taken at Θ_post, not at Θ_init (ω = 1); the results
    match the tiled sweep (STHK_TRIG_ROWS=0) to 1e-13 relative (loglik) and
    1e-10 scale-aware (gradient), and the oracle with tied timestamps; a
    trigger-only sweep over a cached background (h, ω moves) is bitwise the
    full sweep."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for rows in ("0", "1"):
        env = dict(os.environ, STHK_TRIG_ROWS=rows)
        r = subprocess.run([sys.executable, "-c", _ROWS_SCRIPT, root], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[rows] = json.loads(r.stdout.strip().splitlines()[-1])
    assert [c[2] for c in res["0"]] == [0, 0, 0, 0]
    assert [c[2] for c in res["1"]][0::2] == [1, 0] and res["1"][3][2] == 1
    for a, b in zip(res["0"], res["1"]):
        assert abs(a[0] - b[0]) <= 1e-13 * abs(a[0])
        scale = max(abs(v) for v in a[1])
        for ga, gb in zip(a[1], b[1]):
            assert abs(ga - gb) <= 1e-10 * scale
    # ties (strict t_j < t_i) against the oracle, on the row-window path
    ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                      pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005,
                                      keep=3000)
    t = np.floor(ev.ts() * 86400.0) / 86400.0
    ev2 = pk.EventSet(ev.xs(), ev.ys(), t)
    p = pk.Params(0.66, 1.6, 14, 0.344, 1440, 0.0695)
    _check(engine, ev2, p)
    engine.set_params(p)
    engine.loglik_grad()
    assert engine.stats()["trigger_rows"] == 1
    # cached trigger-only sweeps (h, omega moves and back) == full sweeps, bitwise
    ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                      pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005,
                                      keep=40000)
    engine.load(ev)
    seq = [[0.66, 1.6, 14, 0.344, 1440, 0.0695], [0.66, 1.6, 14, 0.344, 1440, 0.072],
           [0.66, 1.6, 14, 0.344, 1300, 0.072], [0.7, 1.6, 14, 0.3, 1300, 0.072],
           [0.66, 1.6, 14, 0.344, 1440, 0.0695]]
    out = {}
    for cache in (False, True):
        engine.set_background_cache(cache)
        rr = []
        for th in seq:
            engine.set_params(th)
            r = engine.loglik_grad(per_event=True)
            st = engine.stats()
            rr.append((r[0], tuple(r[2]), r[3].tobytes(), st["trigger_rows"], st["cache_hit"]))
        out[cache] = rr
    engine.set_background_cache(True)
    for a, b in zip(out[False], out[True]):
        assert a[:4] == b[:4] and a[3] == 1
    assert sum(b[4] for b in out[True]) >= 3


def test_trigger_rows_long_windows_against_oracle(engine):
    """Row windows near their limit: ω chosen so that 709/ω is 0.9 of the
    shortest tile's time span, ≈ 115 sources per row in the window (uniform
    times, 6,000 events), against the long-double oracle; and a bursty
    variant (half the events packed into short bursts)."""
    rng = np.random.default_rng(77)
    n, T = 6000, 100.0
    t = np.sort(rng.uniform(0, T, n))
    x, y = rng.uniform(0, 4, n), rng.uniform(0, 4, n)
    span = min(t[k + 127] - t[k] for k in range(0, n - 127, 128))
    omega = 709.0 / (0.9 * span)
    for p in ([0.7, 1.2, 6.0, 0.5, omega, 1.0], [0.7, 1.2, 6.0, 0.5, omega, 0.2]):
        ev = pk.EventSet(x, y, t)
        _check(engine, ev, pk.Params(*p))
        engine.set_params(p)
        engine.loglik_grad()
        assert engine.stats()["trigger_rows"] == 1
    # bursty: 40 bursts of 75 events within 0.01 days each, plus a uniform half
    tb = np.concatenate([rng.uniform(0, T, 3000)] +
                        [c + rng.uniform(0, 0.01, 75) for c in rng.uniform(0, T, 40)])
    tb = np.sort(tb)
    ev = pk.EventSet(rng.uniform(0, 4, tb.size), rng.uniform(0, 4, tb.size), tb)
    for omega_b in (2000.0, 20000.0):
        p = pk.Params(0.7, 1.2, 6.0, 0.5, omega_b, 0.5)
        _check(engine, ev, p)
