"""bench.py's multi-GPU launcher refuses to mislabel a run: --gpus N needs N
visible GPUs and, under torchrun, WORLD_SIZE == N (exit 2, no JSON line)."""

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True,
                          text=True, timeout=300, env=env)


def test_gpus_more_than_visible_fails_loudly():
    r = _run(["--gpus", "2", "--no-cpu"], {"CUDA_VISIBLE_DEVICES": ""})
    assert r.returncode == 2
    assert "CUDA device(s) visible" in r.stderr
    assert r.stdout.strip() == ""


def test_world_size_mismatch_fails_loudly():
    r = _run(["--gpus", "2", "--no-cpu"], {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0",
                                          "CUDA_VISIBLE_DEVICES": ""})
    assert r.returncode == 2
    assert "WORLD_SIZE=1" in r.stderr
    assert r.stdout.strip() == ""
