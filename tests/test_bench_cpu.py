"""bench.py launcher contract (CPU): --gpus N without torchrun relaunches one
process per GPU, and fails loudly when the box has fewer GPUs than asked."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_more_than_available_fails_loudly():
    import torch
    have = torch.cuda.device_count()
    ask = max(have + 1, 2)
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(ask),
                        "--steps", "3"], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2
    assert f"--gpus {ask} needs {ask} GPUs" in r.stderr
    assert r.stdout.strip() == ""


def test_world_size_mismatch_fails_loudly():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4",
                        "--steps", "3"], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr
