"""Fine-grid geometry, centered mode indexing and the GPU bin sort
(mirrors esnufft.grid, grid.py:1-254).

Conventions: dimension 1 is the fastest axis of every array (shape
(n_d, ..., n_1), C order); node l of a size-n axis sits at l 2 pi / n;
points fold so x / h lands in [0, n).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _lib
from .errors import SizeError

BOX_FAST = 16
BOX_SLOW = 4
SPARSE_SORT_RATIO = 0.1
COORD_LIMIT = 3.0 * np.pi
TWO_PI = 2.0 * np.pi


def next_smooth(n: int) -> int:
    """Least 5-smooth integer >= n (grid.py:34-58)."""
    n = int(n)
    if n < 1:
        raise SizeError(f"next_smooth needs n >= 1, got {n}")
    out = ctypes.c_int64()
    _lib.check(_lib.lib.esn_next_smooth(n, ctypes.byref(out)))
    return int(out.value)


def centered_indices(num_modes: int) -> np.ndarray:
    if num_modes < 1:
        raise SizeError(f"mode count must be >= 1, got {num_modes}")
    lo = -(num_modes // 2)
    return np.arange(lo, lo + num_modes, dtype=np.int64)


@dataclass(frozen=True)
class ModeIndexSet:
    """Centered mode indices per dimension; arrays are (N_d, ..., N_1)."""

    num_modes: tuple

    def __post_init__(self):
        if not 1 <= len(self.num_modes) <= 3:
            raise SizeError(f"1..3 dimensions supported, got {len(self.num_modes)}")
        for n in self.num_modes:
            if n < 1:
                raise SizeError(f"mode counts must be >= 1, got {self.num_modes}")

    @property
    def dim(self) -> int:
        return len(self.num_modes)

    @property
    def total(self) -> int:
        return int(np.prod(self.num_modes))

    @property
    def shape(self) -> tuple:
        return tuple(reversed(self.num_modes))

    def axis_indices(self, axis: int) -> np.ndarray:
        return centered_indices(self.num_modes[axis - 1])

    def fft_bins(self, axis: int, n: int) -> np.ndarray:
        k = self.axis_indices(axis)
        if n < len(k):
            raise SizeError(f"fine grid size {n} smaller than mode count {len(k)}")
        return np.mod(k, n)


def fine_grid_sizes(num_modes, sigma: float, w: int) -> tuple:
    """n_i = next_smooth(max(ceil(sigma N_i), 2 w)) (grid.py:141-149)."""
    for nm in num_modes:
        if nm < 1:
            raise SizeError(f"mode counts must be >= 1, got {tuple(num_modes)}")
    out = (ctypes.c_int64 * 3)()
    _lib.check(_lib.lib.esn_fine_grid_sizes(len(num_modes), _lib.i64_array(num_modes),
                                            float(sigma), int(w), out))
    return tuple(int(out[d]) for d in range(len(num_modes)))


def fold_coords(x, check_bounds: bool = False, n: int | None = None):
    """Fold coordinates into [0, 2 pi) on the GPU (grid.py:152-168); with n,
    return grid units x n / 2 pi instead (spreadinterp.py:99-100)."""
    from .errors import BoundsViolationError
    dev = D.device_of(None)
    like_torch = D.is_torch(x)
    t = D.as_real_1d(x, "x", dev)
    if check_bounds:
        bad = t.abs() > COORD_LIMIT
        if bool(bad.any()):
            i = int(torch.nonzero(bad)[0, 0])
            raise BoundsViolationError(f"coordinate {float(t[i])!r} at index {i} outside [-3 pi, 3 pi]")
    nn = 0 if n is None else int(n)
    g = torch.empty(t.numel(), dtype=torch.float64, device=dev)
    cd = _lib.ESN_F32 if t.dtype == torch.float32 else _lib.ESN_F64
    _lib.check(_lib.lib.esn_fold_coords(t.numel(), cd, ctypes.c_void_p(t.data_ptr()) if t.numel() else None,
                                        nn, ctypes.c_void_p(g.data_ptr()) if t.numel() else None,
                                        ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    return D.to_output(g, like_torch)


@dataclass(frozen=True)
class BinSortPermutation:
    """perm[i] = original index of the i-th point in sorted order; boxes =
    per-point flat box index (original order); box_counts per dim."""

    perm: np.ndarray
    boxes: np.ndarray
    box_counts: tuple


def bin_sort(grid_coords, sizes, threads: int = 1) -> BinSortPermutation:
    """Counting sort of points (grid units in [0, n)) by 16x4x4 boxes on the
    GPU (grid.py:202-254).  Bin membership and box indices match the
    reference exactly; the order inside a box is the GPU's (the reference
    spec guarantees only bin grouping, SPEC.md bin_sort post)."""
    from .plan import Plan
    from .kernel import params_for_width
    m = len(grid_coords[0])
    for c in grid_coords:
        if len(c) != m:
            raise SizeError("coordinate arrays must share a length")
    dim = len(sizes)
    dev = D.device_of(None)
    box = [BOX_FAST] + [BOX_SLOW] * (dim - 1)
    # w = 2 makes the footprint origin floor(g - 1 + 1) = floor(g): the
    # reference's box coordinate
    p = Plan(0, dim, nfine=tuple(sizes), device=dev, params=params_for_width(2, 2.0),
             bin_size=box, method="global", timing=False)
    xs = [D.as_real_1d(g, "g", dev).to(torch.float64) for g in grid_coords]
    p.setpts(xs, grid_units=True)
    perm, keys, _ = p.sort_view()
    torch.cuda.synchronize(dev)
    counts = tuple(-(-sizes[d] // box[d]) for d in range(dim))
    out = BinSortPermutation(perm=perm.cpu().numpy().astype(np.int64),
                             boxes=keys.cpu().numpy().astype(np.int64), box_counts=counts)
    p.close()
    return out
