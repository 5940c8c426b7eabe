"""Spreading (points -> fine grid) and interpolation (fine grid -> points)
on the GPU: the spreadinterp.py:187-306 seam of the reference.

build_point_set keeps the raw coordinates on device; the fold, grid
scaling and bin sort run inside the setpts kernels of a spread/interp plan
(esn_spreader_create + esn_plan_setpts).  spread zeroes the grid itself
(spreadinterp.py:205-206); interp returns values in ORIGINAL point order.
Both directions evaluate identical kernel values, so the pair is adjoint
to rounding (the atomic accumulation order of spread is not fixed, so
results are reproducible to rounding, not bitwise).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _device as D
from .errors import SizeError
from .kernel import KernelParams
from .plan import Plan, raise_data_error

SUBPROBLEM_CAP = 8192  # GPU default max points per spread subproblem


@dataclass(frozen=True)
class NuPointSet:
    """Raw coordinates on device (dimension 1 first) plus fine sizes."""

    coords: tuple
    sizes: tuple
    check_bounds: bool = False

    @property
    def dim(self) -> int:
        return len(self.coords)

    @property
    def count(self) -> int:
        return int(self.coords[0].numel())


def build_point_set(coords, sizes, check_bounds: bool = False) -> NuPointSet:
    if len(coords) != len(sizes):
        raise SizeError(f"{len(coords)} coordinate arrays for {len(sizes)} sizes")
    dev = D.device_of(None)
    m = len(coords[0]) if not D.is_torch(coords[0]) else coords[0].numel()
    xs = []
    for d, raw in enumerate(coords):
        t = D.as_real_1d(raw, "x", dev)
        if t.dim() != 1 or t.numel() != m:
            raise SizeError(f"coordinate array {d + 1} has shape {tuple(t.shape)}, expected ({m},)")
        xs.append(t.to(torch.float64))
    return NuPointSet(coords=tuple(xs), sizes=tuple(int(s) for s in sizes), check_bounds=check_bounds)


def ensure_sorted(points: NuPointSet, threads: int = 1) -> NuPointSet:
    """The GPU sort runs inside every spread/interp plan; nothing to attach."""
    return points


def _fill_stats(stats: dict, p: Plan, kw: dict) -> None:
    """spreadinterp.py:165-184: ``busy_per_thread`` (seconds per worker) and
    ``tasks`` (work items).  On the GPU the worker is the device stream the
    plan runs on (key 0; its busy time is the spread / interp kernel's
    CUDA-event time) and the tasks are the sort's subproblems, which the
    persistent kernels claim dynamically.  Stage times (sort / spread / fft /
    correct) are added as well."""
    timed = kw.get("timing", True)
    stats["busy_per_thread"] = {0: p.hot_kernel_seconds() if timed else 0.0}
    stats["tasks"] = p.tasks()
    if timed:
        stats.update(p.stage_times())


def _spreader(points: NuPointSet, params: KernelParams, use_exact: bool, ntransf: int, **kw):
    p = Plan(0, points.dim, nfine=points.sizes, ntransf=ntransf, params=params,
             use_exact_kernel=use_exact, check_bounds=points.check_bounds, sigma=params.sigma,
             **kw)
    p.setpts(list(points.coords))
    return p


def spread(points: NuPointSet, strengths, params: KernelParams, threads: int = 1,
           use_exact: bool = False, stats: dict | None = None, **kw):
    """b_l = sum_j c_j psi~(l h - x_j); returns (n_d, ..., n_1) complex."""
    like_torch = D.is_torch(strengths)
    dev = D.device_of(None)
    c = D.as_complex(strengths, dev, torch.complex128 if kw.get("dtype", "float64") == "float64"
                     else torch.complex64)
    m = points.count
    ntransf = 1 if c.dim() == 1 else c.shape[0]
    if c.shape[-1:] != (m,) or c.dim() > 2:
        raise SizeError(f"strengths shape {tuple(c.shape)} does not match M={m}")
    shape = tuple(reversed(points.sizes))
    if c.dim() == 2:
        shape = (ntransf,) + shape
    p = _spreader(points, params, use_exact, ntransf, **kw)
    grid = torch.empty(shape, dtype=p.cplx, device=dev)
    p.spread(c, grid)
    st, idx, d = p.check_info()
    if st:
        raise_data_error(st, idx, d, points.coords, "strength")
    if stats is not None:
        _fill_stats(stats, p, kw)
    p.close()
    return D.to_output(grid, like_torch)


def interp(points: NuPointSet, grid, params: KernelParams, threads: int = 1,
           use_exact: bool = False, stats: dict | None = None, **kw):
    """c_j = sum_l b_l psi~(l h - x_j), output in original point order."""
    like_torch = D.is_torch(grid)
    dev = D.device_of(None)
    shape = tuple(reversed(points.sizes))
    gshape = tuple(grid.shape)
    if gshape == shape:
        ntransf = 1
    elif len(gshape) == len(shape) + 1 and gshape[1:] == shape:
        ntransf = gshape[0]
    else:
        raise SizeError(f"grid shape {gshape}, expected {shape}")
    g = D.as_complex(grid, dev, torch.complex128 if kw.get("dtype", "float64") == "float64"
                     else torch.complex64)
    p = _spreader(points, params, use_exact, ntransf, **kw)
    out = torch.empty(((ntransf,) if ntransf > 1 else ()) + (points.count,), dtype=p.cplx, device=dev)
    p.interp(g, out)
    st, idx, d = p.check_info()
    if st:
        raise_data_error(st, idx, d, points.coords)
    if stats is not None:
        _fill_stats(stats, p, kw)
    p.close()
    return D.to_output(out, like_torch)
