"""Worker for tests/test_gpu_peer.py: run under torchrun with WORLD ranks.
The ranks share the visible GPUs round-robin (on a one-GPU box both ranks
use cuda:0 -- two processes, so the root's fine grid really is mapped through
CUDA IPC), the process group is gloo (it carries only the handle and the
barriers; NCCL refuses two ranks on one device).  Writes rank 0's modes."""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_1808_06736_b200 as E  # noqa: E402
from paper_1808_06736_b200.distributed import (exec_type1_peer_reduced, release_peer_grids,  # noqa: E402
                                               shard_range)


def main(out_path):
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    rng = np.random.default_rng(23)
    res = {}
    for tag, dim, nm, tol, dtype in (("d3", 3, (24, 20, 16), 1e-9, "float64"), ("f3", 3, (20, 18, 22), 1e-4, "float32"),
                                     ("d2", 2, (40, 36), 1e-6, "float64")):
        M = 30000
        coords = [rng.uniform(-np.pi, np.pi, M) for _ in range(dim)]
        c = rng.standard_normal(M) + 1j * rng.standard_normal(M)
        lo, hi = shard_range(M, rank, world)
        mine = [torch.from_numpy(x[lo:hi]).to(dev) for x in coords]
        cm = torch.from_numpy(c[lo:hi]).to(dev)
        opts = E.TransformOptions(tolerance=tol, device=dev, dtype=dtype)
        for rep in range(2):  # the second call reuses the cached grid and mapping
            out = exec_type1_peer_reduced(mine, cm, nm, opts, dst=0)
        if rank == 0:
            res[tag] = out.cpu().numpy()
        else:
            assert out is None
    if rank == 0:
        np.savez(out_path, world=world, **res)
    dist.barrier()
    release_peer_grids()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
