"""Point-split type 1 with the reduction fused into the spreader
(distributed.exec_type1_peer_reduced): every rank's tile flushes RED into
the root's peer-mapped fine grid.  Two PROCESSES under torchrun, so the grid
is really mapped through CUDA IPC (both on cuda:0 on a one-GPU box; their
kernels never wait on one another), compared with the CPU oracle on the same
seeded inputs; plus esn_plan_spread_add in one process."""

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
def test_peer_reduced_two_processes(tmp_path, oracle):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = tmp_path / "r.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}",
           os.path.join(ROOT, "tests", "helpers", "peer_worker.py"), str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    got = np.load(out)
    assert int(got["world"]) == 2
    O = oracle
    rng = np.random.default_rng(23)
    for tag, dim, nm, tol, rtol in (("d3", 3, (24, 20, 16), 1e-9, 1e-12), ("f3", 3, (20, 18, 22), 1e-4, 2e-5),
                                    ("d2", 2, (40, 36), 1e-6, 1e-12)):
        M = 30000
        coords = [rng.uniform(-np.pi, np.pi, M) for _ in range(dim)]
        c = rng.standard_normal(M) + 1j * rng.standard_normal(M)
        ref = O.exec_type1(coords, c, nm, tol=tol)
        assert np.linalg.norm(got[tag] - ref) <= rtol * np.linalg.norm(ref), tag


@pytest.mark.gpu
def test_spread_add_accumulates_shards(esn):
    """Two shards added into one zeroed grid = the spread of their union
    (up to the order of the atomic adds); the batched owner-computes
    spreader refuses (plain stores)."""
    import torch
    from paper_1808_06736_b200.plan import Plan
    from paper_1808_06736_b200.errors import SizeError
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(5)
    M, nm = 40000, (30, 28, 26)
    xs = [torch.from_numpy(rng.uniform(-np.pi, np.pi, M)).to(dev) for _ in range(3)]
    c = torch.from_numpy(rng.standard_normal(M) + 1j * rng.standard_normal(M)).to(dev)
    plan = Plan(1, 3, nmodes=nm, tol=1e-8, device=dev)
    shape = tuple(reversed([int(v) for v in plan.nfine]))
    whole = torch.empty(shape, dtype=torch.complex128, device=dev)
    plan.setpts(xs)
    plan.spread(c, whole)
    acc = torch.zeros(shape, dtype=torch.complex128, device=dev)
    h = M // 3
    for lo, hi in ((0, h), (h, M)):
        plan.setpts([x[lo:hi].contiguous() for x in xs])
        plan.spread_add(c[lo:hi].contiguous(), acc)
    plan.check()
    assert torch.linalg.norm(acc - whole) <= 1e-13 * torch.linalg.norm(whole)
    pb = Plan(1, 2, nmodes=(64, 64), tol=1e-4, device=dev, dtype="float32", ntransf=32)
    x2 = [x[:1000].float().contiguous() for x in xs[:2]]
    pb.setpts(x2)
    cb = torch.zeros((32, 1000), dtype=torch.complex64, device=dev)
    g = torch.zeros((32,) + tuple(reversed([int(v) for v in pb.nfine])), dtype=torch.complex64, device=dev)
    with pytest.raises(SizeError):
        pb.spread_add(cb, g)
