"""distributed.py with the real GPU transforms under an NCCL process group
(torchrun, one process per visible GPU -- the round-end box has one, so
world size 1 there; the collectives still run through NCCL).  Compared with
the CPU oracle on the same seeded inputs.  The multi-rank host logic is
covered on CPU by test_distributed_gloo.py."""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
def test_distributed_paths_under_nccl(tmp_path, oracle):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    n = torch.cuda.device_count()
    out = tmp_path / "r.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}",
           os.path.join(ROOT, "tests", "helpers", "nccl_worker.py"), str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    got = np.load(out)
    assert int(got["world"]) == n
    O = oracle
    rng = np.random.default_rng(11)
    M, nm, tol = 20000, (24, 20, 16), 1e-9
    coords = [rng.uniform(-np.pi, np.pi, M) for _ in range(3)]
    c = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    ref = O.exec_type1(coords, c, nm, tol=tol)
    nrm = np.linalg.norm(ref)
    for k in ("grid", "modes", "grid_all"):
        assert np.linalg.norm(got[k] - ref) <= 1e-12 * nrm, k
    cb = rng.standard_normal((5, M)) + 1j * rng.standard_normal((5, M))
    ref1 = np.stack([O.exec_type1(coords[:2], ci, nm[:2], tol=tol) for ci in cb])
    assert np.linalg.norm(got["batch1"] - ref1) <= 1e-12 * np.linalg.norm(ref1)
    shp = (3,) + tuple(reversed(nm[:2]))
    fb = rng.standard_normal(shp) + 1j * rng.standard_normal(shp)
    ref2 = np.stack([O.exec_type2(coords[:2], fi, tol=tol, isign=-1) for fi in fb])
    assert np.linalg.norm(got["batch2"] - ref2) <= 1e-12 * np.linalg.norm(ref2)
