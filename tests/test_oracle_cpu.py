"""CPU: pin the long-double oracle (oracle/hawkes_oracle.c) against the
reference's known answers and golden vectors, and check its gradient against
finite differences of the verbatim reference engine."""
import json
import math
import os

import numpy as np
import pytest

import oracle_glue as og

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _oracle(d, **kw):
    return og.oracle_loglik_grad(d["x"], d["y"], d["t"], d["T"], d["params"], **kw)


def test_single_event_known_answer():
    # test_likelihood.cpp:42-56: log((2pi)^-3/2) - (0.5 - Phi(-1))
    d = _load("ref_kats.json")["single_event"]
    o = _oracle(d)
    assert o["valid"]
    assert abs(o["loglik"] - (-3.0981603456825612)) <= 1e-13
    assert abs(o["loglik"] - d["loglik"]) <= 1e-13


def test_five_event_fixture():
    d = _load("ref_kats.json")["five_event"]
    o = _oracle(d, per_event=True)
    assert abs(o["loglik"] - d["loglik"]) <= 1e-12 * abs(d["loglik"])
    assert np.allclose(o["per_event"], d["per_event"], rtol=1e-12, atol=0)


def test_theta_zero_instance():
    d = _load("ref_kats.json")["theta_zero"]
    o = _oracle(d)
    assert abs(o["loglik"] - d["loglik"]) <= 1e-10 * abs(d["loglik"])
    assert o["grad"][4] == 0.0 and o["grad"][5] == 0.0  # no trigger sensitivity


def test_underflow_is_invalid_not_error():
    d = _load("ref_kats.json")["underflow"]
    o = _oracle(d)
    assert d["valid"] is False
    assert o["valid"] is False and o["loglik"] == -math.inf
    assert np.all(np.isnan(o["grad"]))


def test_invalid_params_rejected():
    with pytest.raises(ValueError):
        og.oracle_loglik_grad([0.0], [0.0], [1.0], 1.0, [1, 1, 1, 0.1, -1.0, 1])
    with pytest.raises(ValueError):
        og.oracle_loglik_grad([0.0], [0.0], [1.0], 1.0, [1, 1, 1, -0.1, 1.0, 1])


def test_random_instances_vs_reference_golden():
    # the 32 instances of test_likelihood.cpp:106-121, reference at 1e-10
    for d in _load("ref_random.json"):
        o = _oracle(d)
        assert o["valid"] == d["valid"]
        for key in ("loglik_serial", "loglik_t4s4"):
            assert abs(o["loglik"] - d[key]) <= 1e-10 * abs(d[key]), (d["n"], d["seed"])


def test_c1_vs_reference_golden():
    d = _load("ref_c1.json")
    o = _oracle(d, per_event=True)
    assert abs(o["loglik"] - d["loglik_serial"]) <= 1e-12 * abs(d["loglik_serial"])
    assert abs(o["loglik"] - d["loglik_t8s8"]) <= 1e-12 * abs(d["loglik_t8s8"])
    assert np.max(np.abs(o["per_event"] - np.array(d["per_event"]))) <= 1e-12


def _ref_or_skip():
    if not og.ref_available():
        pytest.skip("oracle/_ref (verbatim reference build) not present")


def test_oracle_vs_live_reference_random():
    _ref_or_skip()
    rng = np.random.default_rng(7)
    for k in range(6):
        n = int(rng.integers(2, 300))
        x, y, t, we = og.ref_sim_cloud(n, [0, 4, 0, 4, 60], 50 + k)
        p = [rng.uniform(0.3, 2), rng.uniform(0.5, 2), rng.uniform(2, 20), rng.uniform(0.05, 0.8),
             rng.uniform(0.3, 3), rng.uniform(0.1, 1)]
        ref, ok, _ = og.ref_loglik(x, y, t, we, p)
        o = og.oracle_loglik_grad(x, y, t, we, p)
        assert ok == o["valid"]
        assert abs(o["loglik"] - ref) <= 1e-10 * abs(ref)


@pytest.mark.parametrize("params", [[0.6, 0.9, 3.0, 0.5, 1.1, 0.35], [1.0, 1.6, 14.0, 0.1, 1.0, 1.0]])
def test_oracle_gradient_vs_reference_finite_differences(params):
    """the gradient oracle is pinned against Richardson
    central differences of the verbatim reference logLikelihood (serial)."""
    _ref_or_skip()
    x, y, t, we = og.ref_sim_cloud(300, [0, 4, 0, 4, 60], 7)
    o = og.oracle_loglik_grad(x, y, t, we, params)
    p0 = np.array(params, dtype=np.float64)

    def f(p):
        return og.ref_loglik(x, y, t, we, p)[0]

    for k in range(6):
        h = 1e-3 * p0[k]

        def cd(hh):
            pp, pm = p0.copy(), p0.copy()
            pp[k] += hh
            pm[k] -= hh
            return (f(pp) - f(pm)) / (2 * hh)
        fd = (4 * cd(h / 2) - cd(h)) / 3  # Richardson
        assert abs(fd - o["grad"][k]) <= 1e-7 * o["grad_abs"][k], (k, fd, o["grad"][k])


def test_normal_cdf_known_answer():
    # test_kernels.cpp:157-162 compensator KAT uses Phi(1)-Phi(0)=0.3413447460685429
    lib = og.oracle_lib()
    assert abs((lib.oracle_normal_cdf(1.0) - lib.oracle_normal_cdf(0.0)) - 0.3413447460685429) <= 1e-16
