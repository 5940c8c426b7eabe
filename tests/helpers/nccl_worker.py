"""Worker for tests/test_gpu_distributed.py: run under torchrun (1 process
per GPU, NCCL).  Runs every multi-GPU path of distributed.py with the REAL
GPU transforms under a NCCL process group and writes rank 0's results to
the .npz named in argv[1]; the test compares them with the CPU oracle."""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_1808_06736_b200 as E  # noqa: E402
from paper_1808_06736_b200.distributed import (exec_type1_grid_reduced, exec_type1_point_sharded,  # noqa: E402
                                               exec_type1_transform_sharded, exec_type2_transform_sharded,
                                               shard_range)


def main(out_path):
    local = int(os.environ["LOCAL_RANK"])
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    assert dist.get_backend() == "nccl"
    rng = np.random.default_rng(11)
    M, nm, tol = 20000, (24, 20, 16), 1e-9
    coords = [rng.uniform(-np.pi, np.pi, M) for _ in range(3)]
    c = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    lo, hi = shard_range(M, rank, world)
    mine = [torch.from_numpy(x[lo:hi]).to(dev) for x in coords]
    cm = torch.from_numpy(c[lo:hi]).to(dev)
    opts = E.TransformOptions(tolerance=tol, device=dev)
    res = {}
    g = exec_type1_grid_reduced(mine, cm, nm, opts, dst=0)
    p = exec_type1_point_sharded(mine, cm, nm, opts, dst=0)
    ga = exec_type1_grid_reduced(mine, cm, nm, opts, dst=None)
    T = 5
    cb = rng.standard_normal((T, M)) + 1j * rng.standard_normal((T, M))
    co2 = [torch.from_numpy(x).to(dev) for x in coords[:2]]
    b1 = exec_type1_transform_sharded(co2, torch.from_numpy(cb).to(dev), nm[:2], opts)
    fb = rng.standard_normal((3,) + tuple(reversed(nm[:2]))) + 1j * rng.standard_normal((3,) + tuple(reversed(nm[:2])))
    o2 = E.TransformOptions(tolerance=tol, isign=-1, device=dev)
    b2 = exec_type2_transform_sharded(co2, torch.from_numpy(fb).to(dev), o2)
    torch.cuda.synchronize()
    if rank == 0:
        res = dict(grid=g.cpu().numpy(), modes=p.cpu().numpy(), grid_all=ga.cpu().numpy(),
                   batch1=b1.cpu().numpy(), batch2=b2.cpu().numpy(), world=world)
        np.savez(out_path, **res)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
