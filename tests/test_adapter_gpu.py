"""GPU: the drop-in boundary. The reference's own callers, compiled verbatim
and linked against the B200 engine through the C++ adapter
(paper_2005_10123_b200/adapter/hawkes_b200_adapter.cpp):

  * tests/test_likelihood.cpp of the reference (11 cases, incl. the oracle
    comparisons at 1e-10, backend invariance, per-event sums, underflow and
    invalid-parameter behaviour, batch bitwise equality);
  * the reference MH driver (sampler.cpp runChain): the chain driven by the
    GPU engine takes the same accept/reject decisions and draws as the chain
    driven by the reference CPU engine.
"""
import json
import os
import subprocess

import pytest

import oracle_glue as og

pytestmark = pytest.mark.gpu


def _exe(name):
    p = os.path.join(og.REF_DIR, name)
    if not os.path.exists(p):
        pytest.skip(f"{p} not built (needs /root/reference at build time)")
    return p


def test_reference_likelihood_suite_on_b200():
    out = subprocess.run([_exe("test_likelihood_b200")], capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "11/11 passed" in out.stdout


def test_reference_excitation_suite_on_b200():
    out = subprocess.run([_exe("test_excitation_b200")], capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "13/13 passed" in out.stdout


def _chain(exe, *args):
    out = subprocess.run([exe, *args], capture_output=True, text=True, timeout=1200)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_mh_chain_matches_reference_cpu_chain():
    ref = _exe("mh_chain_ref_v4" if og.has_avx512() else "mh_chain_ref_v3")
    args = ["--n", "1500", "--data", "c2", "--iters", "300", "--burnin", "30", "--seed", "7"]
    gpu = _chain(_exe("mh_chain_b200"), *args)
    cpu = _chain(ref, *args, "--threads", "0", "--lanes", "8" if og.has_avx512() else "4")
    assert gpu["accepted"] == cpu["accepted"] and gpu["proposed"] == cpu["proposed"]
    assert gpu["draws_fnv1a"] == cpu["draws_fnv1a"]
    assert abs(gpu["final_logpost"] - cpu["final_logpost"]) <= 1e-10 * abs(cpu["final_logpost"])


def test_reference_timing_harness_on_b200():
    """The reference's timeLikelihood (bench.cpp, verbatim; it fails hard on any
    drift between repeats) over the adapter, full evaluations, C2 at N=20k."""
    exe = _exe("timing_b200")
    env = dict(os.environ, STHK_SWEEP_CACHE="0")
    out = subprocess.run([exe, "--n", "20000", "--repeats", "5", "--warmups", "1"],
                         capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    rec = json.loads(out.stdout.strip().splitlines()[-1])
    assert rec["impl"] == "b200" and rec["n"] == 20000 and rec["median_s"] > 0


def test_adapter_event_cache_exact_under_address_reuse():
    """A set destroyed and rebuilt at the same heap addresses with one event
    moved (at an index the old sampled check skipped) gets its own likelihood,
    equal to the same data at other addresses (the reference API
    is stateless)."""
    out = subprocess.run([_exe("adapter_cache_b200")], capture_output=True, text=True, timeout=600)
    rec = json.loads(out.stdout.strip().splitlines()[-1])
    assert out.returncode == 0, (rec, out.stderr[-2000:])
    assert rec["ll_b"] == rec["ll_b_elsewhere"] == rec["ll_b_again"] != rec["ll_a"]


def test_mh_chain_full_10k_iterations_matches_reference_cpu_chain():
    """a full 10,000-iteration chain at N=1,500 (C2 data) takes
    bitwise the same draws on the B200 engine as on the reference CPU engine."""
    ref = _exe("mh_chain_ref_v4" if og.has_avx512() else "mh_chain_ref_v3")
    args = ["--n", "1500", "--data", "c2", "--iters", "10000", "--burnin", "1000", "--seed", "1"]
    gpu = _chain(_exe("mh_chain_b200"), *args)
    cpu = _chain(ref, *args, "--threads", "0", "--lanes", "8" if og.has_avx512() else "4")
    assert gpu["accepted"] == cpu["accepted"] and gpu["proposed"] == cpu["proposed"]
    assert gpu["draws_fnv1a"] == cpu["draws_fnv1a"]
    assert abs(gpu["final_logpost"] - cpu["final_logpost"]) <= 1e-10 * abs(cpu["final_logpost"])


def test_mh_chain_first_iterations_at_c2_match_reference_cpu_chain():
    """The bench-size chain (C2, N=85,000): the first 20 iterations of the
    reference runChain take identical accept/reject decisions and draws on
    the B200 engine and on the reference CPU engine (all host cores)."""
    ref = _exe("mh_chain_ref_v4" if og.has_avx512() else "mh_chain_ref_v3")
    args = ["--n", "85000", "--data", "c2", "--iters", "20", "--burnin", "2", "--seed", "1"]
    gpu = _chain(_exe("mh_chain_b200"), *args)
    cpu = _chain(ref, *args, "--threads", "0", "--lanes", "8" if og.has_avx512() else "4")
    assert gpu["accepted"] == cpu["accepted"] and gpu["proposed"] == cpu["proposed"]
    assert gpu["draws_fnv1a"] == cpu["draws_fnv1a"]
    assert abs(gpu["final_logpost"] - cpu["final_logpost"]) <= 1e-10 * abs(cpu["final_logpost"])
