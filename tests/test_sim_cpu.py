"""CPU: the synthetic-data generators (include/sthk_sim.h) reproduce the
reference generators bit for bit (golden checksums from the reference)."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle_glue as og
import paper_2005_10123_b200 as pk

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.float64).tobytes()).hexdigest()


def test_cloud_matches_reference_golden():
    sim = json.load(open(os.path.join(GOLD, "ref_sim.json")))
    for key, d in sim.items():
        if not key.startswith("cloud"):
            continue
        ev = pk.generateBenchmarkCloud(d["n"], pk.SimWindow(*d["window"]), d["seed"])
        assert sha(ev.xs()) == d["sha_x"] and sha(ev.ys()) == d["sha_y"] and sha(ev.ts()) == d["sha_t"]


def test_cluster_c2_matches_reference_golden():
    d = json.load(open(os.path.join(GOLD, "ref_sim.json")))["cluster_c2"]
    ev, par = pk.simulateClusterProcess(pk.Params(*d["params"]), pk.SimWindow(*d["window"]),
                                        d["rate"], d["seed"])
    assert ev.size() == d["n"] == 86138
    assert sha(ev.xs()) == d["sha_x"] and sha(ev.ts()) == d["sha_t"]
    assert hashlib.sha256(par.astype(np.int32).tobytes()).hexdigest() == d["sha_parent"]
    ev85, _ = pk.simulateClusterProcess(pk.Params(*d["params"]), pk.SimWindow(*d["window"]),
                                        d["rate"], d["seed"], keep=85000)
    assert ev85.windowEnd() == d["t_85000"]


def test_c1_events_match_golden():
    d = json.load(open(os.path.join(GOLD, "ref_c1.json")))
    ev = pk.generateBenchmarkCloud(1000, pk.SimWindow(*d["window"]), d["seed"])
    assert np.array_equal(ev.xs(), np.array(d["x"])) and np.array_equal(ev.ts(), np.array(d["t"]))


def test_live_reference_generators():
    if not og.ref_available():
        pytest.skip("oracle/_ref not built")
    for n, seed in [(1, 3), (17, 4), (4096, 5)]:
        x, y, t, we = og.ref_sim_cloud(n, [0, 15, 0, 15, 4750], seed)
        ev = pk.generateBenchmarkCloud(n, pk.SimWindow(0, 15, 0, 15, 4750), seed)
        assert np.array_equal(x, ev.xs()) and np.array_equal(y, ev.ys()) and np.array_equal(t, ev.ts())
    p = [1.0, 1.6, 14.0, 0.3, 1.0, 0.1]
    x, y, t, par = og.ref_sim_cluster(p, [0, 10, 0, 10, 250], 0.07, 321)
    ev, par2 = pk.simulateClusterProcess(pk.Params(*p), pk.SimWindow(0, 10, 0, 10, 250), 0.07, 321)
    assert np.array_equal(t, ev.ts()) and np.array_equal(par, par2)
