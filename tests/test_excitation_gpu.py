"""GPU: excitation probabilities vs the long-double oracle
sums, and the reference's posteriorExcitation semantics
(excitation.cpp:13-130, test_excitation.cpp)."""
import math
import os

import numpy as np
import pytest

import oracle_glue as og
import paper_2005_10123_b200 as pk

pytestmark = pytest.mark.gpu


def _oracle_split(ev, p):
    o = og.oracle_loglik_grad(ev.xs(), ev.ys(), ev.ts(), ev.windowEnd(), p.as_array(), sums=True)
    s = o["sums"]
    bgNorm = (2 * math.pi) ** -1.5 / (p.tauX ** 2 * p.tauT)
    trNorm = p.theta * p.omega / (2 * math.pi * p.h ** 2)
    mu = p.mu0 * bgNorm * s[:, 0]
    xi = trNorm * s[:, 3]
    return mu, xi, xi / (mu + xi)


def _tp():
    return pk.Params(0.7, 1.1, 6.0, 0.4, 1.5, 0.2)


@pytest.mark.parametrize("n,seed", [(3, 1), (50, 9), (200, 21), (2000, 5)])
def test_excitation_matches_oracle(engine, n, seed):
    ev = pk.generateBenchmarkCloud(n, pk.SimWindow(0, 4, 0, 4, 30), seed)
    p = _tp()
    ex = pk.excitationProbabilities(ev, p, engine=engine)
    mu, xi, pi = _oracle_split(ev, p)
    assert np.allclose(ex.mu, mu, rtol=1e-12, atol=0)
    assert np.all(np.abs(ex.xi - xi) <= 1e-12 * (np.abs(xi) + 1e-300) + 1e-300)
    assert np.all(np.abs(ex.pi - pi) <= 1e-12)
    assert ex.xi[0] == 0.0 and ex.pi[0] == 0.0 and ex.mu[0] > 0
    assert np.all((ex.pi == 0) == (ex.xi == 0))


def test_theta_zero_and_invalid(engine):
    ev = pk.generateBenchmarkCloud(60, pk.SimWindow(0, 4, 0, 4, 30), 10)
    p = _tp()
    p.theta = 0.0
    ex = pk.excitationProbabilities(ev, p, engine=engine)
    assert np.all(ex.pi == 0.0) and np.all(ex.xi == 0.0)
    bad = _tp()
    bad.h = 0.0
    with pytest.raises(ValueError):
        pk.excitationProbabilities(ev, bad, engine=engine)


def test_consistent_with_likelihood_rates(engine):
    ev = pk.generateBenchmarkCloud(150, pk.SimWindow(0, 4, 0, 4, 30), 33)
    p = _tp()
    ex = pk.excitationProbabilities(ev, p, engine=engine)
    r = pk.logLikelihood(ev, p, keepPerEvent=True, engine=engine)
    D = ev.windowEnd() - ev.ts()
    from scipy.special import ndtr
    comp = p.mu0 * (ndtr(D / p.tauT) - ndtr(-ev.ts() / p.tauT)) - p.theta * np.expm1(-p.omega * D)
    lam = np.exp(r.perEvent + comp)
    assert np.allclose(ex.mu + ex.xi, lam, rtol=1e-12, atol=0)


def test_posterior_excitation_semantics(engine, tmp_path):
    ev = pk.generateBenchmarkCloud(200, pk.SimWindow(0, 4, 0, 4, 30), 50)
    rng = np.random.default_rng(51)
    draws = []
    for _ in range(10):
        p = _tp()
        p.theta, p.omega, p.h = rng.uniform(0.05, 0.8), rng.uniform(0.5, 3.0), rng.uniform(0.05, 0.5)
        draws.append(p)
    post = pk.posteriorExcitation(ev, draws, thinTo=10, engine=engine)
    acc = np.zeros(ev.size())
    for p in draws:
        acc += pk.excitationProbabilities(ev, p, engine=engine).pi
    acc /= 10.0
    assert np.array_equal(post.meanPi, acc)
    assert post.perDraw.shape == (10, ev.size())
    assert pk.thinIndices(10, 3) == [0, 3, 6] and pk.thinIndices(3, 10) == [0, 1, 2]
    small = pk.posteriorExcitation(ev, draws[:2], memoryCapEntries=10, engine=engine)
    assert small.perDraw.size == 0
    bad = _tp()
    bad.omega = -2.0
    with pytest.raises(RuntimeError, match="draw 1"):
        pk.posteriorExcitation(ev, [draws[0], bad, draws[0]], engine=engine)
    path = os.path.join(str(tmp_path), "pi.tsv")
    pk.posteriorExcitation(ev, [draws[0]] * 7, thinTo=3, dumpPath=path, engine=engine)
    lines = open(path).read().strip().split("\n")
    assert lines[0].startswith("# sthawkes pi draws v1, events=200") and len(lines) == 4


def test_posterior_excitation_batch_bitwise_and_errors(engine, tmp_path):
    """The batched device path (sthk_excitation_batch: MH-style draws sharing
    tauX, tauT share one background sweep) reproduces the reference's
    one-call-per-draw loop bitwise -- meanPi, perDraw rows, the dump file --
    also across chunked calls (sum_pi in/out), and stops at the same draw
    with the same message on an underflowed rate."""
    ev = pk.generateBenchmarkCloud(3000, pk.SimWindow(0, 8, 0, 8, 400), 9)
    rng = np.random.default_rng(3)
    draws, p = [], [0.6, 0.9, 3.0, 0.4, 2.0, 0.3]
    for _ in range(40):  # an MH-like walk: one coordinate moves per draw
        k = [0, 3, 4, 5][int(rng.integers(4))]
        p = list(p)
        p[k] *= float(np.exp(0.05 * rng.standard_normal()))
        draws.append(pk.Params(*p))
    path_b = os.path.join(str(tmp_path), "batch.tsv")
    post = pk.posteriorExcitation(ev, draws, thinTo=25, dumpPath=path_b, engine=engine)
    idx = pk.thinIndices(len(draws), 25)
    acc, rows = np.zeros(ev.size()), []
    for d in idx:
        pi = pk.excitationProbabilities(ev, draws[d], engine=engine).pi
        acc += pi
        rows.append(pi)
    acc /= float(len(idx))
    assert np.array_equal(post.meanPi, acc)
    assert np.array_equal(post.perDraw, np.array(rows))
    ref_lines = ["# sthawkes pi draws v1, events=3000"] + [
        str(d) + "".join("\t%.17g" % v for v in r) for d, r in zip(idx, rows)]
    assert open(path_b).read() == "\n".join(ref_lines) + "\n"
    # chunked: two device calls, sums carried through sum_pi
    P = np.array([draws[d].as_array() for d in idx])
    engine.load(ev)
    s1, _, b1 = engine.excitation_batch(P[:11])
    s2, r2, b2 = engine.excitation_batch(P[11:], sum_pi=s1, per_draw=True)
    assert b1 == b2 == -1 and np.array_equal(s2 / float(len(idx)), acc)
    assert np.array_equal(r2, np.array(rows[11:]))
    # an underflowing draw (mu0 * S_B and the trigger both below the smallest
    # double) stops the batch at its index, after the earlier draws' dump lines
    bad = pk.Params(5e-324, 0.9, 3.0, 0.0, 2.0, 0.3)
    seq = [draws[0], draws[1], bad, draws[2]]
    path_e = os.path.join(str(tmp_path), "err.tsv")
    with pytest.raises(RuntimeError, match="posteriorExcitation: draw 2: .*underflowed"):
        pk.posteriorExcitation(ev, seq, dumpPath=path_e, engine=engine)
    assert len(open(path_e).read().strip().split("\n")) == 3


def test_excitation_row_windows_against_oracle_and_batch(engine):
    """Excitation split with the trigger sums by row windows (ω = 200/day:
    709/ω = 3.5 days, shorter than every tile) against the oracle; then MH
    draws moving ω and h -- trigger-only evaluations fused into finalize --
    through the batched posterior path, bitwise equal to single calls."""
    ev = pk.generateBenchmarkCloud(3000, pk.SimWindow(0, 8, 0, 8, 400), 12)
    p = pk.Params(0.7, 1.1, 6.0, 0.4, 200.0, 0.3)
    ex = pk.excitationProbabilities(ev, p, engine=engine)
    assert engine.stats()["trigger_rows"] == 1
    mu, xi, pi = _oracle_split(ev, p)
    assert np.allclose(ex.mu, mu, rtol=1e-12, atol=0)
    assert np.all(np.abs(ex.xi - xi) <= 1e-12 * (np.abs(xi) + 1e-300) + 1e-300)
    assert np.all(np.abs(ex.pi - pi) <= 1e-12)
    rng = np.random.default_rng(8)
    draws, q = [], [0.7, 1.1, 6.0, 0.4, 200.0, 0.3]
    for _ in range(12):
        k = [0, 3, 4, 5][int(rng.integers(4))]
        q = list(q)
        q[k] *= float(np.exp(0.05 * rng.standard_normal()))
        draws.append(pk.Params(*q))
    post = pk.posteriorExcitation(ev, draws, thinTo=12, engine=engine)
    rows = [pk.excitationProbabilities(ev, d, engine=engine).pi for d in draws]
    assert np.array_equal(post.perDraw, np.array(rows))
