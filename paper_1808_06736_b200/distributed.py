"""Multi-GPU execution (one process per GPU, torch.distributed over NCCL).

SURVEY.md section 8(e):

* one large type-1 transform (config c3) splits its POINTS across ranks,
  in two variants: exec_type1_point_sharded -- each rank
  spreads its shard into its own fine grid, FFTs and deconvolves, and the
  partial MODE arrays are summed with one NCCL reduce (exact by linearity
  of spreading, FFT and the diagonal correction; the mode array is
  sigma^d = 8x smaller than the fine grid); exec_type1_grid_reduced --
  the partial FINE GRIDS are reduced and only the root runs FFT + deconv;
* batched transforms (config c5, and batched type 2) split their
  TRANSFORMS across ranks: every rank sorts the shared point set itself and
  runs its slice of strength / mode vectors -- no data-path collective; the
  slices are gathered at the end (exec_type1_transform_sharded,
  exec_type2_transform_sharded);
* exec_type1_peer_reduced fuses that reduction into the spreader: the root's
  fine grid is peer-mapped (CUDA IPC over NVLink) on every rank and each
  rank's tile flushes RED straight into it -- no per-rank grids, no reduce
  collective;
* type 2 and single-GPU configs run as independent replicas (each rank owns
  its own targets; type-2 outputs are independent per point).

``compute`` is injectable so the host-side sharding / reduction logic is
testable on CPU with the gloo backend; production calls use the GPU
transforms of this package.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced shard [lo, hi) of ``total`` items for ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    base, extra = divmod(int(total), world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def _world(group):
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def _gpu_type1(coords, strengths, num_modes, opts):
    from .transforms import exec_type1
    return exec_type1(coords, strengths, num_modes, opts)[0]


def _as_real_view(t: torch.Tensor) -> torch.Tensor:
    return torch.view_as_real(t) if t.is_complex() else t


def exec_type1_point_sharded(coords, strengths, num_modes, opts, *, group=None, dst: int | None = 0,
                             compute=None):
    """Type 1 over points distributed across ranks.

    Every rank passes ITS shard of points / strengths (any split); the
    result -- the transform of the union of all shards -- is returned on
    ``dst`` (all ranks when ``dst`` is None, via all-reduce).  Other ranks
    get their partial modes back (useful for overlap), or None when
    ``dst`` is a different rank.
    """
    compute = compute or _gpu_type1
    rank, world = _world(group)
    part = compute(coords, strengths, num_modes, opts)
    if world == 1:
        return part
    t = part if isinstance(part, torch.Tensor) else torch.as_tensor(part)
    t = t.contiguous()
    buf = _as_real_view(t)
    if dst is None:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
        return t
    dist.reduce(buf, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return t if rank == dst else None


def _gpu_spread(coords, strengths, num_modes, opts):
    from .transforms import spread_type1_grid
    return spread_type1_grid(coords, strengths, num_modes, opts)


def _gpu_finish(state, grid, num_modes, opts):
    from .transforms import finish_type1_grid
    return finish_type1_grid(state, grid)


def exec_type1_grid_reduced(coords, strengths, num_modes, opts, *, group=None, dst: int | None = 0,
                            spread=None, finish=None):
    """Type 1 over points distributed across ranks, reducing the FINE GRID
    (first variant): every rank spreads its shard
    into a full fine grid, the grids are summed with one NCCL reduce (exact:
    spreading is linear) and ``dst`` alone runs the FFT + deconvolution.  The
    message is sigma^d x the mode array of exec_type1_point_sharded, which
    in exchange skips the FFT on the other ranks.  ``spread(coords, c, nm,
    opts) -> (grid, state)`` and ``finish(state, grid, nm, opts) -> modes``
    are injectable (CPU tests)."""
    spread = spread or _gpu_spread
    finish = finish or _gpu_finish
    rank, world = _world(group)
    grid, state = spread(coords, strengths, num_modes, opts)
    if world > 1:
        buf = _as_real_view(grid)
        if dst is None:
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
        else:
            dist.reduce(buf, dst=dst, op=dist.ReduceOp.SUM, group=group)
            if rank != dst:
                return None
    return finish(state, grid, num_modes, opts)


_PEER_GRIDS: dict = {}  # (device, bytes) -> peer.PeerBuffer of the root's fine grid, reused across calls


def release_peer_grids():
    """Free the cached peer-mappable fine grids of this process and unmap
    the peers' grids it opened (call on every rank, after a barrier: nobody
    may still be adding into a grid that is freed)."""
    from . import peer
    for key in list(_PEER_GRIDS):
        _PEER_GRIDS.pop(key).free()
    peer.close_all_peers()


def exec_type1_peer_reduced(coords, strengths, num_modes, opts, *, group=None, dst: int = 0):
    """Type 1 over points distributed across ranks with the reduction FUSED
    into the spreader (B200: NVLink 5 / NVSwitch peer
    memory).  ``dst`` owns the fine grid in peer-mappable memory
    (peer.PeerBuffer, CUDA IPC); every rank sorts its shard and its spread
    kernel flushes its tiles with REDs straight into that grid -- the
    partial sums never exist as per-rank grids and no reduce collective
    runs; ``dst`` then runs the FFT + deconvolution.  Exact up to the
    floating-point order of the atomic adds (as between two runs of a
    single-GPU spread).  The process group carries only the 64-byte handle
    and two barriers, so any backend works.  Returns the modes on ``dst``,
    None elsewhere."""
    from . import peer
    from .transforms import finish_type1_grid, prepare_type1_spread
    rank, world = _world(group)
    plan, c, xs, shape = prepare_type1_spread(coords, strengths, num_modes, opts)
    dev = c.device
    nbytes = c.element_size()
    for v in shape:
        nbytes *= int(v)
    grid = None
    if rank == dst:
        key = (str(dev), nbytes)
        buf = _PEER_GRIDS.get(key)
        if buf is None:
            buf = _PEER_GRIDS[key] = peer.PeerBuffer(nbytes, dev)
        grid = buf.tensor(c.dtype, shape)
        with torch.cuda.device(dev):
            grid.zero_()
            torch.cuda.current_stream(dev).synchronize()  # zeroed before any peer adds
        target = grid
    if world > 1:
        box = [buf.handle if rank == dst else None]
        dist.broadcast_object_list(box, src=dst, group=group)  # (also: the grid is zeroed)
        if rank != dst:
            target = peer.open_peer(box[0], dev)
    with plan.lock:
        plan.spread_add(c, target)
        st, idx, d = plan.check_info()  # waits for this rank's flushes
    if world > 1:
        dist.barrier(group=group)  # every rank's REDs have landed
    if st:  # (after the barrier: a rank with bad data must not strand the others)
        from .transforms import raise_data_error
        raise_data_error(st, idx, d, xs, "strength")
    if rank != dst:
        return None
    return finish_type1_grid(plan, grid)


def _empty_slice_spec(part, ref, opts, group):
    """dtype / device of this rank's all-gather buffer.  A rank without a
    transform (T < world) has no result to copy them from: it uses the plan
    precision and the device the backend needs (NCCL: this rank's CUDA
    device; gloo: host), so every rank joins with matching buffers."""
    if part is not None:
        return part.dtype, part.device
    prec = getattr(opts, "dtype", "float64")
    dtype = torch.complex64 if prec == "float32" else torch.complex128
    if dist.get_backend(group) == "nccl":
        return dtype, torch.device("cuda", torch.cuda.current_device())
    return (ref.dtype if ref.is_complex() else dtype), torch.device("cpu")


def _gather_transform_slices(part, T, rank, world, group, tail_shape, dtype, device):
    """All-gather per-rank (T_r, ...) slices into the full (T, ...) array.
    Every rank joins the collective, including ranks whose slice is empty
    (T < world): they contribute a zero pad, so no rank can block."""
    shapes = [shard_range(T, r, world) for r in range(world)]
    width = max(h - l for l, h in shapes)
    pad = torch.zeros((width,) + tuple(tail_shape), dtype=dtype, device=device)
    if part is not None and part.shape[0]:
        pad[: part.shape[0]] = part
    slabs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather([_as_real_view(s) for s in slabs], _as_real_view(pad), group=group)
    return torch.cat([s[: h - l] for s, (l, h) in zip(slabs, shapes)], dim=0)


def exec_type1_transform_sharded(coords, strengths_all, num_modes, opts, *, group=None, compute=None):
    """Batched type 1 (strengths (T, M)) with the T transforms split across
    ranks; every rank returns the full (T, N_d..N_1) result (all-gather).
    T and world are the same on every rank, so argument errors are raised
    on all ranks before any collective; ranks left without a transform
    (T < world) still join the all-gather with an empty slice."""
    compute = compute or _gpu_type1
    rank, world = _world(group)
    if strengths_all.ndim != 2 or strengths_all.shape[0] < 1:
        raise ValueError(f"batched strengths must be (T >= 1, M), got {tuple(strengths_all.shape)}")
    T = strengths_all.shape[0]
    lo, hi = shard_range(T, rank, world)
    part = compute(coords, strengths_all[lo:hi], num_modes, opts) if hi > lo else None
    if world == 1:
        return part
    nm = tuple(num_modes) if not isinstance(num_modes, int) else (num_modes,)
    tail = tuple(reversed(nm))
    ref = strengths_all if isinstance(strengths_all, torch.Tensor) else torch.as_tensor(strengths_all)
    part = None if part is None else (part if isinstance(part, torch.Tensor) else torch.as_tensor(part))
    dtype, device = _empty_slice_spec(part, ref, opts, group)
    return _gather_transform_slices(part, T, rank, world, group, tail, dtype, device)


def _gpu_type2(coords, modes, opts):
    from .transforms import exec_type2
    return exec_type2(coords, modes, opts)[0]


def exec_type2_transform_sharded(coords, modes_all, opts, *, group=None, compute=None):
    """Batched type 2 (mode arrays (T, N_d..N_1)) with the T transforms split
    across ranks (north_star: batched transforms shard across the GPUs):
    every rank interpolates its slice at the shared targets -- no
    data-path collective -- and the (T_r, M) slices are all-gathered, so
    every rank returns the full (T, M) result."""
    compute = compute or _gpu_type2
    rank, world = _world(group)
    if modes_all.ndim < 2 or modes_all.shape[0] < 1:
        raise ValueError(f"batched modes must be (T >= 1, N_d..N_1), got {tuple(modes_all.shape)}")
    T = modes_all.shape[0]
    M = int(coords[0].shape[0])
    lo, hi = shard_range(T, rank, world)
    part = compute(coords, modes_all[lo:hi], opts) if hi > lo else None
    if world == 1:
        return part
    ref = modes_all if isinstance(modes_all, torch.Tensor) else torch.as_tensor(modes_all)
    part = None if part is None else (part if isinstance(part, torch.Tensor) else torch.as_tensor(part))
    if part is not None and part.ndim == 1:
        part = part[None]
    dtype, device = _empty_slice_spec(part, ref, opts, group)
    return _gather_transform_slices(part, T, rank, world, group, (M,), dtype, device)
