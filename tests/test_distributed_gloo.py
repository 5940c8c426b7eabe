"""Multi-process host logic of the multi-GPU paths (distributed.py) on CPU:
world_size 2, gloo backend, 127.0.0.1.  The per-rank transform is injected
as the CPU oracle (test infrastructure); the sharding, the point-split
modes reduction and the transform-split all-gather are the product code."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_compute(coords, c, nm, opts):
    import esn_oracle as O
    c = c.numpy() if isinstance(c, torch.Tensor) else np.asarray(c)
    cs = [np.asarray(x) for x in coords]
    if c.ndim == 2:
        out = np.stack([O.exec_type1(cs, ci, nm, tol=opts["tol"]) for ci in c])
    else:
        out = O.exec_type1(cs, c, nm, tol=opts["tol"])
    return torch.from_numpy(np.ascontiguousarray(out))


def _oracle_compute2(coords, f, opts):
    import esn_oracle as O
    f = f.numpy() if isinstance(f, torch.Tensor) else np.asarray(f)
    cs = [np.asarray(x) for x in coords]
    out = np.stack([O.exec_type2(cs, fi, tol=opts["tol"], isign=-1) for fi in f])
    return torch.from_numpy(np.ascontiguousarray(out))


def _oracle_spread(coords, c, nm, opts):
    """First half of the oracle's type 1 (esn_oracle.exec_type1 up to the
    spread), returning (grid tensor, state) like spread_type1_grid."""
    import esn_oracle as O
    params = O.select_params(opts["tol"])
    sizes = O.fine_grid_sizes(nm, 2.0, params.w)
    gs = [O.grid_coords(np.asarray(x), n)[0] for x, n in zip(coords, sizes)]
    perm, _ = O.bin_sort(gs, sizes)
    grid = O.spread(gs, perm, np.asarray(c), sizes, params)
    return torch.from_numpy(np.ascontiguousarray(grid)), (params, sizes)


def _oracle_finish(state, grid, nm, opts):
    import esn_oracle as O
    params, sizes = state
    big = O.fft_forward(grid.numpy())
    bins = [np.mod(O.centered(k), n) for k, n in zip(nm, sizes)]
    out = np.ascontiguousarray(big[np.ix_(*reversed(bins))])
    O._apply_separable(out, O._axis_corr(params, nm, sizes))
    return torch.from_numpy(out)


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p in (root, os.path.join(root, "oracle"), os.path.join(root, "tests", "golden")):
        sys.path.insert(0, p)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1808_06736_b200.distributed import (exec_type1_grid_reduced, exec_type1_point_sharded,
                                                       exec_type1_transform_sharded,
                                                       exec_type2_transform_sharded, shard_range)
        rng = np.random.default_rng(5)
        M, nm = 3000, (12, 10)
        coords = [rng.uniform(-np.pi, np.pi, M) for _ in range(2)]
        c = rng.standard_normal(M) + 1j * rng.standard_normal(M)
        lo, hi = shard_range(M, rank, world)
        mine = [x[lo:hi] for x in coords]
        opts = {"tol": 1e-9}
        full = exec_type1_point_sharded(mine, c[lo:hi], nm, opts, dst=0, compute=_oracle_compute)
        allr = exec_type1_point_sharded(mine, c[lo:hi], nm, opts, dst=None, compute=_oracle_compute)
        T = 5
        cb = rng.standard_normal((T, M)) + 1j * rng.standard_normal((T, M))
        batched = exec_type1_transform_sharded(coords, torch.from_numpy(cb), nm, opts, compute=_oracle_compute)
        gfull = exec_type1_grid_reduced(mine, c[lo:hi], nm, opts, dst=0, spread=_oracle_spread,
                                        finish=_oracle_finish)
        gall = exec_type1_grid_reduced(mine, c[lo:hi], nm, opts, dst=None, spread=_oracle_spread,
                                       finish=_oracle_finish)
        # batched type 2: transforms split, (T, M) all-gathered
        fb = rng.standard_normal((3,) + tuple(reversed(nm))) + 1j * rng.standard_normal((3,) + tuple(reversed(nm)))
        batched2 = exec_type2_transform_sharded(coords, torch.from_numpy(fb), opts, compute=_oracle_compute2)
        # T < world: the rank without a transform still joins the gather
        one = exec_type1_transform_sharded(coords, torch.from_numpy(cb[:1]), nm, opts, compute=_oracle_compute)
        q.put((rank, None if full is None else full.numpy(), allr.numpy(), batched.numpy(),
               None if gfull is None else gfull.numpy(), gall.numpy(), batched2.numpy(), one.numpy()))
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions():
    from paper_1808_06736_b200.distributed import shard_range
    for total in (0, 1, 7, 64, 1000):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1


def test_point_and_transform_sharding_world2(oracle):
    import esn_oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, *vals = q.get(timeout=300)
        res[r] = tuple(vals)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(5)
    M, nm = 3000, (12, 10)
    coords = [rng.uniform(-np.pi, np.pi, M) for _ in range(2)]
    c = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    ref = O.exec_type1(coords, c, nm, tol=1e-9)
    # point split + reduce == the unsplit transform (linearity), to rounding
    assert np.linalg.norm(res[0][0] - ref) <= 1e-12 * np.linalg.norm(ref)
    assert res[1][0] is None
    for r in (0, 1):
        assert np.linalg.norm(res[r][1] - ref) <= 1e-12 * np.linalg.norm(ref)
    # fine-grid reduce variant: root (or every rank for all-reduce) finishes
    assert np.linalg.norm(res[0][3] - ref) <= 1e-12 * np.linalg.norm(ref)
    assert res[1][3] is None
    for r in (0, 1):
        assert np.linalg.norm(res[r][4] - ref) <= 1e-12 * np.linalg.norm(ref)
    cb = rng.standard_normal((5, M)) + 1j * rng.standard_normal((5, M))
    refb = np.stack([O.exec_type1(coords, ci, nm, tol=1e-9) for ci in cb])
    for r in (0, 1):
        np.testing.assert_array_equal(res[r][2], refb)
        np.testing.assert_array_equal(res[r][6], refb[:1])
    fb = rng.standard_normal((3,) + tuple(reversed(nm))) + 1j * rng.standard_normal((3,) + tuple(reversed(nm)))
    refb2 = np.stack([O.exec_type2(coords, fi, tol=1e-9, isign=-1) for fi in fb])
    for r in (0, 1):
        np.testing.assert_array_equal(res[r][5], refb2)
