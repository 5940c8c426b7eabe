"""The nonuniform transforms on B200 (mirrors esnufft.transforms).

Type 1: f_k = sum_j c_j exp(isign i k.x_j)  (spread -> cuFFT -> deconvolve)
Type 2: c_j = sum_k f_k exp(isign i k.x_j)  (amplify -> cuFFT -> interpolate)
Type 3: f_k = sum_j c_j exp(isign i s_k.x_j) (spread -> inner type 2 ->
        per-target phi-hat correction), transforms.py:221-351.

Same signatures, argument conventions, defaults, exception classes and stage
keys as the reference (transforms.py:44-404).  Inputs may be numpy arrays
(returned as numpy) or CUDA torch tensors (returned as torch tensors, no
host round trip).  Extensions: a leading ntransf axis on strengths / modes
(batched transforms sharing one point set), ``dtype="float32"``, and GPU
knobs (method, bin_size, max_subprob, device).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _device as D
from . import _lib
from .errors import BadToleranceError, DataError, ResourceError, SizeError
from .grid import ModeIndexSet, fine_grid_sizes, next_smooth
from .kernel import MAX_TOLERANCE, MIN_TOLERANCE, KernelParams, kernel_ft, select_params
from .plan import PLANS, Plan, _ptr, raise_data_error

DEFAULT_GRID_CAP = 2 ** 31
TWO_PI = 2.0 * math.pi


@dataclass(frozen=True)
class TransformOptions:
    """Knobs shared by all transforms (transforms.py:44-80) plus GPU knobs.

    threads is accepted for drop-in compatibility and ignored (the GPU path
    has no host thread pool).  dtype: "float64" (reference semantics) or
    "float32".  method: "auto" | "tile" | "global" spreader.
    """

    tolerance: float = 1e-6
    isign: int = 1
    sigma: float = 2.0
    threads: int = 0
    check_bounds: bool = False
    use_exact_kernel: bool = False
    max_grid_values: int = DEFAULT_GRID_CAP
    params: KernelParams | None = None
    dtype: str = "float64"
    method: str = "auto"
    bin_size: tuple | None = None
    max_subprob: int = 0
    device: object = None

    def __post_init__(self):
        if self.isign not in (1, -1):
            raise SizeError(f"isign must be +1 or -1, got {self.isign}")
        if self.threads < 0:
            raise SizeError(f"threads must be >= 0, got {self.threads}")
        if self.max_grid_values < 1:
            raise SizeError("max_grid_values must be positive")
        if not (MIN_TOLERANCE <= self.tolerance <= MAX_TOLERANCE):
            raise BadToleranceError(
                f"tolerance {self.tolerance:g} outside [{MIN_TOLERANCE:g}, {MAX_TOLERANCE:g}]")
        if self.dtype not in ("float64", "float32"):
            raise SizeError(f"dtype must be 'float64' or 'float32', got {self.dtype!r}")
        if self.method not in ("auto", "tile", "global"):
            raise SizeError(f"method must be auto/tile/global, got {self.method!r}")

    def kernel_params(self) -> KernelParams:
        if self.params is not None:
            return self.params
        return select_params(self.tolerance, self.sigma)


def _new_timings() -> dict:
    return {"sort": 0.0, "spread": 0.0, "fft": 0.0, "correct": 0.0}


def _merge_timings(dst: dict, src: dict) -> None:
    for k, v in src.items():
        dst[k] = dst.get(k, 0.0) + v


def _as_mode_tuple(num_modes, dim: int) -> tuple:
    if np.isscalar(num_modes):
        nm = (int(num_modes),) * dim
    else:
        nm = tuple(int(n) for n in num_modes)
    if len(nm) != dim:
        raise SizeError(f"{len(nm)} mode counts for a {dim}-d transform")
    return nm


def _grid_cap_check(total: int, cap: int) -> None:
    if total > cap:
        raise ResourceError(
            f"fine grids need {total} complex values, over the cap of {cap}; "
            "this regime is better served by direct summation")


def _coords_to_device(coords, dev, dim_expected=None):
    m = len(coords[0]) if not D.is_torch(coords[0]) else coords[0].numel()
    out = []
    for d, raw in enumerate(coords):
        shape = tuple(raw.shape) if hasattr(raw, "shape") else np.asarray(raw).shape
        if len(shape) != 1 or shape[0] != m:
            raise SizeError(f"coordinate array {d + 1} has shape {shape}, expected ({m},)")
        out.append(D.as_real_1d(raw, f"x{d + 1}", dev))
    if len({t.dtype for t in out}) > 1:
        out = [t.to(torch.float64) for t in out]
    return out, m


def _plan_for(ttype, dim, nm, isign, ntransf, params, opts: TransformOptions, dev):
    stream = torch.cuda.current_stream(dev).cuda_stream
    key = (ttype, dim, nm, isign, ntransf, params, opts.dtype, opts.sigma, opts.method,
           opts.bin_size, opts.max_subprob, opts.use_exact_kernel, opts.check_bounds,
           opts.max_grid_values, str(dev), stream)
    return PLANS.get(key, lambda: Plan(
        ttype, dim, nmodes=nm, isign=isign, ntransf=ntransf, tol=opts.tolerance, device=dev,
        sigma=opts.sigma, check_bounds=opts.check_bounds, use_exact_kernel=opts.use_exact_kernel,
        max_grid_values=opts.max_grid_values, dtype=opts.dtype, method=opts.method,
        bin_size=opts.bin_size, max_subprob=opts.max_subprob, timing=True, params=params))


def _flat_to_pos(flat: int, shape):
    idx = tuple(int(v) for v in np.unravel_index(flat, shape))
    return idx[0] if len(idx) == 1 else idx


def exec_type1(coords, strengths, num_modes, opts: TransformOptions):
    """Nonuniform-to-uniform transform; returns (modes, stage_seconds).

    strengths (M,) -> modes (N_d..N_1); strengths (T, M) -> (T, N_d..N_1)."""
    params = opts.kernel_params()
    dim = len(coords)
    nm = _as_mode_tuple(num_modes, dim)
    modes = ModeIndexSet(nm)
    sizes = fine_grid_sizes(nm, opts.sigma, params.w)
    _grid_cap_check(int(np.prod(sizes)), opts.max_grid_values)
    dev = D.device_of(opts.device)
    like_torch = D.is_torch(strengths)
    with torch.cuda.device(dev):
        xs, m = _coords_to_device(coords, dev)
        c = D.as_complex(strengths, dev, D.CPLX[opts.dtype])
        if c.dim() == 1:
            ntransf, batched = 1, False
        elif c.dim() == 2:
            ntransf, batched = c.shape[0], True
        else:
            ntransf, batched = -1, False
        if c.shape[-1:] != (m,) or ntransf < 1:
            raise SizeError(f"strengths shape {tuple(c.shape)} does not match M={m}")
        plan = _plan_for(1, dim, nm, opts.isign, ntransf, params, opts, dev)
        out = torch.empty(((ntransf,) if batched else ()) + modes.shape, dtype=plan.cplx, device=dev)
        with plan.lock:
            plan.setpts(xs)
            plan.execute(c, out)
            st, idx, d = plan.check_info()
            if st:
                raise_data_error(st, idx, d, xs, "strength")
            timings = plan.stage_times()
    return D.to_output(out, like_torch), timings


def spread_type1_grid(coords, strengths, num_modes, opts: TransformOptions):
    """First half of a type-1 transform: the fine grid of the spread
    (device tensor (T, n_d..n_1) / (n_d..n_1)) plus the plan that finishes it
    with ``finish_type1_grid``.  The grid of several point shards can be
    summed (e.g. an NCCL reduce) before finishing: spreading is linear."""
    params = opts.kernel_params()
    dim = len(coords)
    nm = _as_mode_tuple(num_modes, dim)
    ModeIndexSet(nm)
    sizes = fine_grid_sizes(nm, opts.sigma, params.w)
    _grid_cap_check(int(np.prod(sizes)), opts.max_grid_values)
    dev = D.device_of(opts.device)
    with torch.cuda.device(dev):
        xs, m = _coords_to_device(coords, dev)
        c = D.as_complex(strengths, dev, D.CPLX[opts.dtype])
        ntransf = 1 if c.dim() == 1 else c.shape[0]
        if c.shape[-1:] != (m,) or c.dim() > 2 or ntransf < 1:
            raise SizeError(f"strengths shape {tuple(c.shape)} does not match M={m}")
        plan = _plan_for(1, dim, nm, opts.isign, ntransf, params, opts, dev)
        grid = torch.empty(((ntransf,) if c.dim() == 2 else ()) + tuple(reversed(sizes)), dtype=plan.cplx,
                           device=dev)
        with plan.lock:
            plan.setpts(xs)
            plan.spread(c, grid)
            st, idx, d = plan.check_info()
            if st:
                raise_data_error(st, idx, d, xs, "strength")
    return grid, plan


def prepare_type1_spread(coords, strengths, num_modes, opts: TransformOptions):
    """Plan + sorted points of a type-1 spread whose grid lives elsewhere
    (``Plan.spread_add`` into a shared / peer-mapped fine grid): returns
    (plan, strengths on the device, fine-grid shape (T,) n_d..n_1)."""
    params = opts.kernel_params()
    dim = len(coords)
    nm = _as_mode_tuple(num_modes, dim)
    ModeIndexSet(nm)
    sizes = fine_grid_sizes(nm, opts.sigma, params.w)
    _grid_cap_check(int(np.prod(sizes)), opts.max_grid_values)
    dev = D.device_of(opts.device)
    with torch.cuda.device(dev):
        xs, m = _coords_to_device(coords, dev)
        c = D.as_complex(strengths, dev, D.CPLX[opts.dtype])
        ntransf = 1 if c.dim() == 1 else c.shape[0]
        if c.shape[-1:] != (m,) or c.dim() > 2 or ntransf < 1:
            raise SizeError(f"strengths shape {tuple(c.shape)} does not match M={m}")
        plan = _plan_for(1, dim, nm, opts.isign, ntransf, params, opts, dev)
        with plan.lock:
            plan.setpts(xs)
    shape = ((ntransf,) if c.dim() == 2 else ()) + tuple(reversed(sizes))
    return plan, c, xs, shape


def finish_type1_grid(plan: Plan, grid: torch.Tensor):
    """Second half: cuFFT (in place on ``grid``) and deconvolution
    (esn_plan_finish_type1); returns the modes (T, N_d..N_1) / (N_d..N_1)."""
    lead = tuple(grid.shape[:-plan.dim])
    out = torch.empty(lead + tuple(reversed(plan.nmodes)), dtype=plan.cplx, device=grid.device)
    with plan.lock:
        plan.finish_type1(grid, out)
        plan.check()
    return out


def exec_type2(coords, mode_coeffs, opts: TransformOptions):
    """Uniform-to-nonuniform transform; returns (strengths, stage_seconds).

    modes (N_d..N_1) -> (M,); modes (T, N_d..N_1) -> (T, M)."""
    params = opts.kernel_params()
    dim = len(coords)
    shape = tuple(mode_coeffs.shape) if hasattr(mode_coeffs, "shape") else np.asarray(mode_coeffs).shape
    if len(shape) == dim:
        ntransf, batched, mshape = 1, False, shape
    elif len(shape) == dim + 1 and shape[0] >= 1:
        ntransf, batched, mshape = shape[0], True, shape[1:]
    else:
        raise SizeError(f"mode array rank {len(shape)} for a {dim}-d transform")
    nm = tuple(reversed(mshape))
    ModeIndexSet(nm)
    sizes = fine_grid_sizes(nm, opts.sigma, params.w)
    _grid_cap_check(int(np.prod(sizes)), opts.max_grid_values)
    dev = D.device_of(opts.device)
    like_torch = D.is_torch(mode_coeffs)
    with torch.cuda.device(dev):
        f = D.as_complex(mode_coeffs, dev, D.CPLX[opts.dtype])
        xs, m = _coords_to_device(coords, dev)
        plan = _plan_for(2, dim, nm, opts.isign, ntransf, params, opts, dev)
        out = torch.empty(((ntransf,) if batched else ()) + (m,), dtype=plan.cplx, device=dev)
        with plan.lock:
            plan.setpts(xs)
            plan.execute(out, f)
            st, idx, d = plan.check_info()
            if st:
                if d == 0:
                    raise DataError(f"non-finite mode coefficient at index {_flat_to_pos(idx, shape)}")
                raise_data_error(st, idx, d, xs)
            timings = plan.stage_times()
    return D.to_output(out, like_torch), timings


# ---------------------------------------------------------------------------
# type 3 (transforms.py:221-351) composed from the GPU spreader and the GPU
# type-2 plan; the per-target phi-hat correction runs on device in float64.

@dataclass(frozen=True)
class Type3Geometry:
    x_shift: tuple
    s_shift: tuple
    x_half_width: tuple
    s_half_width: tuple
    sizes: tuple
    gamma: tuple


def _axis_shift(vmin: float, vmax: float) -> float:
    # transforms.py:233-242: recentre only when it halves the range
    mid = 0.5 * (vmin + vmax)
    if mid == 0.0:
        return 0.0
    before = max(abs(vmin), abs(vmax))
    after = 0.5 * (vmax - vmin)
    return mid if 2.0 * after < before else 0.0


def plan_type3_geometry(coords, targets, params: KernelParams, sigma: float) -> Type3Geometry:
    """transforms.py:245-264 (coords / targets may be numpy or torch)."""
    w = params.w
    x0, s0, xw, sw, sizes, gamma = [], [], [], [], [], []
    for x, s in zip(coords, targets):
        xt = x if D.is_torch(x) else torch.as_tensor(np.asarray(x, dtype=np.float64))
        st = s if D.is_torch(s) else torch.as_tensor(np.asarray(s, dtype=np.float64))
        xs = _axis_shift(float(xt.min()), float(xt.max())) if xt.numel() else 0.0
        ss = _axis_shift(float(st.min()), float(st.max())) if st.numel() else 0.0
        xh = float((xt - xs).abs().max()) if xt.numel() else 0.0
        sh = float((st - ss).abs().max()) if st.numel() else 0.0
        se = sh if sh > 0.0 else 1.0
        n = next_smooth(max(int(np.ceil((2.0 * sigma / np.pi) * xh * se)) + w, 2 * w))
        x0.append(xs)
        s0.append(ss)
        xw.append(xh)
        sw.append(sh)
        sizes.append(n)
        gamma.append(n / (2.0 * sigma * se))
    return Type3Geometry(tuple(x0), tuple(s0), tuple(xw), tuple(sw), tuple(sizes), tuple(gamma))


def exec_type3(coords, strengths, targets, opts: TransformOptions):
    """Nonuniform-to-nonuniform transform; returns (values, stage_seconds)."""
    params = opts.kernel_params()
    dim = len(coords)
    if dim not in (1, 2, 3):
        raise SizeError(f"dimension must be 1, 2, or 3, got {dim}")
    if len(targets) != dim:
        raise SizeError(f"{len(targets)} target arrays for a {dim}-d transform")
    dev = D.device_of(opts.device)
    like_torch = D.is_torch(strengths)
    timings = _new_timings()
    with torch.cuda.device(dev):
        xs = [D.as_real_1d(a, "x", dev).to(torch.float64) for a in coords]
        ss = [D.as_real_1d(a, "s", dev).to(torch.float64) for a in targets]
        m, nk = xs[0].numel(), ss[0].numel()
        for d in range(dim):
            if xs[d].dim() != 1 or xs[d].numel() != m:
                raise SizeError(f"coordinate array {d + 1} has shape {tuple(xs[d].shape)}")
            if ss[d].dim() != 1 or ss[d].numel() != nk:
                raise SizeError(f"target array {d + 1} has shape {tuple(ss[d].shape)}")
        c = D.as_complex(strengths, dev, torch.complex128)
        if tuple(c.shape) != (m,):
            raise SizeError(f"strengths shape {tuple(c.shape)} does not match M={m}")
        # every finiteness check in one device reduction (one host sync); the
        # reference's messages are rebuilt only when something is non-finite
        ok = torch.stack([torch.isfinite(t).all() for t in xs + ss] +
                         [(torch.isfinite(c.real) & torch.isfinite(c.imag)).all()])
        if not bool(ok.all()):
            for d in range(dim):
                if not bool(torch.isfinite(xs[d]).all()):
                    raise DataError(f"non-finite coordinate in dimension {d + 1}")
                if not bool(torch.isfinite(ss[d]).all()):
                    raise DataError(f"non-finite target in dimension {d + 1}")
            bad = ~(torch.isfinite(c.real) & torch.isfinite(c.imag))
            raise DataError(f"non-finite strength at index {int(torch.nonzero(bad)[0, 0])}")
        if nk == 0:
            out = torch.empty(0, dtype=torch.complex128, device=dev)
            return D.to_output(out, like_torch), timings
        geo = plan_type3_geometry(xs, ss, params, opts.sigma)
        inner_sizes = fine_grid_sizes(geo.sizes, opts.sigma, params.w)
        _grid_cap_check(int(np.prod(geo.sizes)) + int(np.prod(inner_sizes)), opts.max_grid_values)
        stream = torch.cuda.current_stream(dev).cuda_stream
        x0 = (ctypes.c_double * 3)(*geo.x_shift, *([0.0] * (3 - dim)))
        s0 = (ctypes.c_double * 3)(*geo.s_shift, *([0.0] * (3 - dim)))
        gam = (ctypes.c_double * 3)(*geo.gamma, *([1.0] * (3 - dim)))
        nf = _lib.i64_array(list(geo.sizes) + [1] * (3 - dim))
        p3 = lambda ts: [_ptr(t) for t in ts] + [None] * (3 - dim)  # noqa: E731
        # pre-phase (+ conjugation for isign < 0) and rescaled sources
        # (transforms.py:304-312), one kernel
        c = c.contiguous()
        cph = torch.empty_like(c)
        resc = [torch.empty_like(x) for x in xs]
        _lib.check(_lib.lib.esn_type3_prephase(dim, m, *p3([x.contiguous() for x in xs]), x0, s0, gam,
                                               int(opts.isign < 0), _ptr(c), _ptr(cph), *p3(resc), stream))
        # the spreader plan is cached like the type-1/2 plans (keyed by the
        # fine grid the geometry picked): repeated calls skip its allocations
        skey = (0, dim, tuple(geo.sizes), params, opts.sigma, opts.method, opts.use_exact_kernel,
                opts.max_grid_values, str(dev), stream)
        sp = PLANS.get(skey, lambda: Plan(0, dim, nfine=geo.sizes, device=dev, params=params, sigma=opts.sigma,
                                          use_exact_kernel=opts.use_exact_kernel, method=opts.method,
                                          dtype="float64", max_grid_values=opts.max_grid_values, timing=True))
        grid = torch.empty(tuple(reversed(geo.sizes)), dtype=torch.complex128, device=dev)
        sp.lock.acquire()  # (held until the stage times are read below)
        try:
            sp.setpts(resc)
            sp.spread(cph, grid)
        except BaseException:
            sp.lock.release()
            raise
        b = torch.empty_like(grid)
        _lib.check(_lib.lib.esn_fftshift(dim, nf, _ptr(grid), _ptr(b), stream))
        del grid
        inner = [torch.empty_like(s) for s in ss]
        _lib.check(_lib.lib.esn_type3_targets(dim, nk, *p3([s.contiguous() for s in ss]), s0, gam, nf,
                                              *p3(inner), stream))
        inner_opts = replace(opts, isign=1, check_bounds=False, params=params, dtype="float64")
        try:
            out, tin = exec_type2(inner, b, inner_opts)
            # (inputs were checked finite above, so the spreader plan's flags
            # need no read; its stage events are read once, after the type 2)
            t1 = sp.stage_times()
        finally:
            sp.lock.release()
        timings["sort"] += t1["sort"]
        timings["spread"] += t1["spread"]
        _merge_timings(timings, tin)
        # psi-hat correction, post-phase, final conjugation (transforms.py:333-351)
        kp = params.to_c()
        _lib.check(_lib.lib.esn_type3_correct(dim, nk, *p3([s.contiguous() for s in ss]), x0, s0, gam, nf,
                                              ctypes.byref(kp), int(opts.isign < 0), _ptr(out), stream))
    return D.to_output(out, like_torch), timings


# ---------------------------------------------------------------------------
# public wrappers (transforms.py:358-404)

def _opts(kw) -> TransformOptions:
    return TransformOptions(**kw)


def nufft1d1(x, c, n_modes, **kw):
    """Type 1 in 1d: f[k] = sum_j c[j] exp(isign i k x[j]), shape (N1,)."""
    return exec_type1((x,), c, _as_mode_tuple(n_modes, 1), _opts(kw))[0]


def nufft2d1(x, y, c, n_modes, **kw):
    """Type 1 in 2d; n_modes is (N1, N2) or a scalar, output shape (N2, N1)."""
    return exec_type1((x, y), c, _as_mode_tuple(n_modes, 2), _opts(kw))[0]


def nufft3d1(x, y, z, c, n_modes, **kw):
    """Type 1 in 3d; n_modes is (N1, N2, N3) or a scalar, output (N3, N2, N1)."""
    return exec_type1((x, y, z), c, _as_mode_tuple(n_modes, 3), _opts(kw))[0]


def nufft1d2(x, f, **kw):
    """Type 2 in 1d: c[j] = sum_k f[k] exp(isign i k x[j])."""
    return exec_type2((x,), f, _opts(kw))[0]


def nufft2d2(x, y, f, **kw):
    """Type 2 in 2d; f has shape (N2, N1)."""
    return exec_type2((x, y), f, _opts(kw))[0]


def nufft3d2(x, y, z, f, **kw):
    """Type 2 in 3d; f has shape (N3, N2, N1)."""
    return exec_type2((x, y, z), f, _opts(kw))[0]


def nufft1d3(x, c, s, **kw):
    """Type 3 in 1d: f[k] = sum_j c[j] exp(isign i s[k] x[j])."""
    return exec_type3((x,), c, (s,), _opts(kw))[0]


def nufft2d3(x, y, c, s, t, **kw):
    """Type 3 in 2d with target components (s[k], t[k])."""
    return exec_type3((x, y), c, (s, t), _opts(kw))[0]


def nufft3d3(x, y, z, c, s, t, u, **kw):
    """Type 3 in 3d with target components (s[k], t[k], u[k])."""
    return exec_type3((x, y, z), c, (s, t, u), _opts(kw))[0]


def clear_plan_cache() -> None:
    """Drop the cached transform plans and the cuFFT plans (fft.py:101-106)."""
    from . import fft
    PLANS.clear()
    fft.clear_plan_cache()
