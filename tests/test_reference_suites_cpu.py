"""CPU: the reference's own GoogleTest suites, compiled verbatim against the
oracle/shim API shims, must pass -- this is what makes oracle/_ref a faithful
build of the reference (64/64)."""
import os
import subprocess

import pytest

import oracle_glue as og

SUITES = {"test_kernels": 24, "test_pack": 6, "test_likelihood": 11, "test_backends": 11,
          "test_simulator": 12, "test_excitation": 13}


@pytest.mark.parametrize("suite", sorted(SUITES))
def test_reference_suite_passes(suite):
    exe = os.path.join(og.REF_DIR, suite)
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert f"{SUITES[suite]}/{SUITES[suite]} passed" in out.stdout
