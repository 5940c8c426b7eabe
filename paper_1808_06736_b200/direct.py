"""Direct-summation transforms and error metrics on the GPU (mirrors the
public part of esnufft.oracle, oracle.py:101-209).

These O(M N) float64 sums run in the esn_direct CUDA kernel; they are an
independent route to the same transforms (no spreading, no FFT), useful for
sampled accuracy checks of large transforms.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _lib
from .errors import DataError, ResourceError, SizeError

DIRECT_COST_CAP = 100_000_000_000  # the GPU affords 1000x the CPU cap (oracle.py:23)
ROUNDOFF = 1.1e-16


def _dev_real(arrs, dev):
    out = [D.as_real_1d(a, "x", dev).to(torch.float64) for a in arrs]
    m = out[0].numel()
    for d, a in enumerate(out):
        if a.dim() != 1 or a.numel() != m:
            raise SizeError(f"coordinate array {d + 1} has shape {tuple(a.shape)}")
        if not bool(torch.isfinite(a).all()):
            raise DataError(f"non-finite coordinate in dimension {d + 1}")
    return out


def _direct(xs, c, ss, isign):
    dev = c.device
    m, nk = xs[0].numel(), ss[0].numel()
    if m * nk > DIRECT_COST_CAP:
        raise ResourceError(f"direct summation cost {m * nk:.3g} exceeds cap {DIRECT_COST_CAP:.3g}")
    out = torch.empty(nk, dtype=torch.complex128, device=dev)
    P = [ctypes.c_void_p(t.data_ptr()) if t.numel() else None for t in xs] + [None] * (3 - len(xs))
    S = [ctypes.c_void_p(t.data_ptr()) if t.numel() else None for t in ss] + [None] * (3 - len(ss))
    _lib.check(_lib.lib.esn_direct(len(xs), m, P[0], P[1], P[2],
                                   ctypes.c_void_p(c.data_ptr()) if c.numel() else None,
                                   nk, S[0], S[1], S[2], int(isign),
                                   ctypes.c_void_p(out.data_ptr()) if nk else None,
                                   ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    return out


def direct_type3(coords, strengths, targets, isign: int = 1):
    dev = D.device_of(None)
    like_torch = D.is_torch(strengths)
    xs = _dev_real(coords, dev)
    ss = _dev_real(targets, dev) if len(targets[0]) else [D.as_real_1d(t, "s", dev) for t in targets]
    if len(ss) != len(xs):
        raise SizeError(f"{len(ss)} target arrays for {len(xs)} dims")
    c = D.as_complex(strengths, dev, torch.complex128)
    if tuple(c.shape) != (xs[0].numel(),):
        raise SizeError(f"strengths shape {tuple(c.shape)}")
    return D.to_output(_direct(xs, c, ss, isign), like_torch)


def _mesh(num_modes, dev):
    axes = [torch.arange(n, dtype=torch.float64, device=dev) - n // 2 for n in num_modes]
    grids = torch.meshgrid(*axes, indexing="ij")
    return [g.reshape(-1).contiguous() for g in grids]


def direct_type1(coords, strengths, num_modes, isign: int = 1):
    if np.isscalar(num_modes):
        num_modes = (int(num_modes),)
    num_modes = tuple(int(n) for n in num_modes)
    dev = D.device_of(None)
    like_torch = D.is_torch(strengths)
    xs = _dev_real(coords, dev)
    if len(num_modes) != len(xs):
        raise SizeError(f"{len(num_modes)} mode counts for {len(xs)} dims")
    c = D.as_complex(strengths, dev, torch.complex128)
    flat = _direct(xs, c, _mesh(num_modes, dev), isign)
    return D.to_output(flat.reshape(num_modes).permute(*reversed(range(len(num_modes)))).contiguous(),
                       like_torch)


def direct_type2(coords, mode_coeffs, isign: int = 1):
    dev = D.device_of(None)
    like_torch = D.is_torch(mode_coeffs)
    xs = _dev_real(coords, dev)
    f = D.as_complex(mode_coeffs, dev, torch.complex128)
    if f.dim() != len(xs):
        raise SizeError(f"mode array rank {f.dim()} for {len(xs)} dims")
    num_modes = tuple(reversed(f.shape))
    fk = f.permute(*reversed(range(f.dim()))).reshape(-1).contiguous()
    return D.to_output(_direct(_mesh(num_modes, dev), fk, xs, isign), like_torch)


@dataclass(frozen=True)
class ErrorReport:
    rel_l2: float
    max_abs_diff: float
    floor: float


def rel_l2(approx, exact, n_terms: int | None = None) -> ErrorReport:
    a = (approx.cpu().numpy() if D.is_torch(approx) else np.asarray(approx)).astype(np.complex128).reshape(-1)
    e = (exact.cpu().numpy() if D.is_torch(exact) else np.asarray(exact)).astype(np.complex128).reshape(-1)
    if a.shape != e.shape:
        raise SizeError(f"shape mismatch {a.shape} vs {e.shape}")
    denom = float(np.linalg.norm(e))
    if denom == 0.0:
        raise DataError("reference vector is identically zero")
    diff = a - e
    return ErrorReport(rel_l2=float(np.linalg.norm(diff)) / denom,
                       max_abs_diff=float(np.max(np.abs(diff))) if len(diff) else 0.0,
                       floor=(n_terms or 0) * ROUNDOFF)


ALIASING_PROBE_CAP = 64


def aliasing_probe(num_modes: int, points, params):
    """|fast - direct| for unit strengths at each point (oracle.py:157-180)."""
    from .transforms import TransformOptions, exec_type1
    x = np.ascontiguousarray(np.asarray(points, dtype=np.float64))
    m = len(x)
    if num_modes > ALIASING_PROBE_CAP or m > ALIASING_PROBE_CAP:
        raise ResourceError(f"probe sizes capped at {ALIASING_PROBE_CAP}, got N={num_modes}, M={m}")
    eye = np.eye(m, dtype=np.complex128)
    fast, _ = exec_type1((x,), eye, (num_modes,), TransformOptions(params=params))
    exact = np.stack([direct_type1((x,), eye[j], (num_modes,)) for j in range(m)])
    mags = np.abs(fast - exact).T
    return mags, float(mags.max())
