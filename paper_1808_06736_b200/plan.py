"""Reusable GPU plans (the C ABI esn_plan_* wrapped for torch tensors).

A Plan amortises kernel parameters, the Horner table, phi-hat corrections,
the bin sort of a point set, the fine grid and the cuFFT plan across calls
(the reference re-does all of it per call,
transforms.py:136-218).  exec_type1/2 use a small cache of Plans.
"""

from __future__ import annotations

import ctypes
import threading
from collections import OrderedDict

import torch

from . import _lib
from .errors import DataError, BoundsViolationError, ErrorCode, SizeError
from .kernel import KernelParams

DTYPES = {"float64": _lib.ESN_F64, "float32": _lib.ESN_F32}
METHODS = {"auto": _lib.METHOD_AUTO, "global": _lib.METHOD_GLOBAL, "tile": _lib.METHOD_TILE}


def make_opts(*, sigma=2.0, check_bounds=False, use_exact_kernel=False,
              max_grid_values=2 ** 31, dtype="float64", method="auto", bin_size=None,
              max_subprob=0, timing=True, stream=None, params: KernelParams | None = None,
              coeffs=None, strength_dtype=None, coord_dtype=None):
    o = _lib.OptsC()
    _lib.lib.esn_default_opts(ctypes.byref(o))
    o.sigma = float(sigma)
    o.check_bounds = int(bool(check_bounds))
    o.use_exact_kernel = int(bool(use_exact_kernel))
    o.max_grid_values = int(max_grid_values)
    o.dtype = DTYPES[dtype]
    o.method = METHODS[method] if isinstance(method, str) else int(method)
    if bin_size:
        for d, b in enumerate(bin_size):
            o.bin_size[d] = int(b)
    o.max_subprob = int(max_subprob)
    o.timing = int(bool(timing))
    o.stream = ctypes.c_void_p(stream) if stream else None
    o.strength_dtype = DTYPES[strength_dtype] if strength_dtype else 0
    o.coord_dtype = DTYPES[coord_dtype] if coord_dtype else 0
    keep = []
    if params is not None:
        kp = params.to_c()
        keep.append(kp)
        o.params = ctypes.pointer(kp)
    if coeffs is not None:
        import numpy as np
        arr = np.ascontiguousarray(coeffs, dtype=np.float64)
        keep.append(arr)
        o.coeffs = arr.ctypes.data_as(_lib.P_dbl)
    return o, keep


def _ptr(t: torch.Tensor | None):
    return ctypes.c_void_p(t.data_ptr()) if t is not None and t.numel() else None


class Plan:
    """type 1 / 2 transform plan, or a spread/interp-only plan (type 0)."""

    def __init__(self, ttype: int, dim: int, *, nmodes=None, nfine=None, isign=1, ntransf=1,
                 tol=1e-6, device=None, **optkw):
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.dtype = optkw.get("dtype", "float64")
        self.real = torch.float64 if self.dtype == "float64" else torch.float32
        self.cplx = torch.complex128 if self.dtype == "float64" else torch.complex64
        self.ttype, self.dim, self.isign, self.ntransf = ttype, dim, isign, ntransf
        with torch.cuda.device(self.device):
            self.stream = torch.cuda.current_stream(self.device)
            optkw.setdefault("stream", self.stream.cuda_stream)
            o, keep = make_opts(**optkw)
            self._keep = keep
            h = ctypes.c_void_p()
            if ttype == 0:
                _lib.check(_lib.lib.esn_spreader_create(dim, _lib.i64_array(nfine), ntransf,
                                                        ctypes.byref(o), ctypes.byref(h)))
            else:
                _lib.check(_lib.lib.esn_plan_create(ttype, dim, _lib.i64_array(nmodes), isign,
                                                    ntransf, float(tol), ctypes.byref(o),
                                                    ctypes.byref(h)))
        self.h = h
        nf = (ctypes.c_int64 * 3)()
        kp = _lib.KernelParamsC()
        _lib.check(_lib.lib.esn_plan_info(self.h, nf, ctypes.byref(kp)))
        self.nfine = tuple(int(nf[d]) for d in range(dim))
        self.params = KernelParams(int(kp.w), float(kp.beta), float(kp.sigma), float(kp.gamma),
                                   int(kp.p_quad))
        self.nmodes = tuple(int(v) for v in nmodes) if nmodes is not None else None
        self.M = None
        self.lock = threading.Lock()
        self._coords = None

    # -- lifetime
    def close(self):
        if getattr(self, "h", None):
            _lib.lib.esn_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- operations (all stream ordered on self.stream)
    def setpts(self, coords, grid_units: bool = False):
        if len(coords) != self.dim:
            raise SizeError(f"{len(coords)} coordinate arrays for a {self.dim}-d plan")
        m = coords[0].numel()
        cd = _lib.ESN_F32 if coords[0].dtype == torch.float32 else _lib.ESN_F64
        for c in coords:
            if c.dtype != coords[0].dtype or c.device != self.device or not c.is_contiguous():
                raise SizeError("coordinate arrays must share dtype, device and be contiguous")
        if grid_units:
            cd |= 0x10
        ptrs = [_ptr(c) for c in coords] + [None] * (3 - self.dim)
        _lib.check(_lib.lib.esn_plan_setpts(self.h, m, cd, *ptrs))
        self.M = m
        self._coords = coords  # keep alive until the stream has consumed them
        return self

    def execute(self, c: torch.Tensor, f: torch.Tensor):
        _lib.check(_lib.lib.esn_plan_execute(self.h, _ptr(c), _ptr(f)))

    def spread(self, c: torch.Tensor, grid: torch.Tensor):
        _lib.check(_lib.lib.esn_plan_spread(self.h, _ptr(c), _ptr(grid)))

    def spread_add(self, c: torch.Tensor, grid):
        """Spread ADDING into ``grid`` (a tensor, or the integer device
        pointer of a peer-mapped grid: esn_plan_spread_add)."""
        g = _ptr(grid) if isinstance(grid, torch.Tensor) else ctypes.c_void_p(int(grid))
        _lib.check(_lib.lib.esn_plan_spread_add(self.h, _ptr(c), g))

    def finish_type1(self, grid: torch.Tensor, f: torch.Tensor):
        """cuFFT (in place on ``grid``) + deconvolution into ``f``."""
        _lib.check(_lib.lib.esn_plan_finish_type1(self.h, _ptr(grid), _ptr(f)))

    def interp(self, grid: torch.Tensor, c: torch.Tensor):
        _lib.check(_lib.lib.esn_plan_interp(self.h, _ptr(grid), _ptr(c)))

    def check(self):
        """Synchronise and raise the reference's exception for device-side
        data errors (non-finite input, bounds)."""
        info = (ctypes.c_int64 * 2)()
        st = _lib.lib.esn_plan_check(self.h, info)
        if st != ErrorCode.SUCCESS:
            _lib.check(st)

    def check_info(self):
        info = (ctypes.c_int64 * 2)()
        st = _lib.lib.esn_plan_check(self.h, info)
        return int(st), int(info[0]), int(info[1])

    def stage_times(self) -> dict:
        v = [ctypes.c_double() for _ in range(4)]
        _lib.check(_lib.lib.esn_plan_stage_times(self.h, *[ctypes.byref(x) for x in v]))
        return {"sort": v[0].value, "spread": v[1].value, "fft": v[2].value, "correct": v[3].value}

    def hot_kernel_seconds(self) -> float:
        v = ctypes.c_double()
        _lib.check(_lib.lib.esn_plan_hot_kernel_seconds(self.h, ctypes.byref(v)))
        return v.value

    def tasks(self) -> int:
        """Subproblems of the last sort (the kernels' scheduling units)."""
        v = ctypes.c_int64()
        _lib.check(_lib.lib.esn_plan_tasks(self.h, ctypes.byref(v)))
        return int(v.value)

    def bins(self):
        nb = ctypes.c_int()
        bs = (ctypes.c_int * 3)()
        nbd = (ctypes.c_int * 3)()
        _lib.check(_lib.lib.esn_plan_bins(self.h, ctypes.byref(nb), bs, nbd))
        return int(nb.value), tuple(bs[:self.dim]), tuple(nbd[:self.dim])

    def sort_view(self):
        """(perm, keys, bin_start) int32 device tensors of the current sort."""
        nb, _, _ = self.bins()
        perm = torch.empty(self.M, dtype=torch.int32, device=self.device)
        keys = torch.empty(self.M, dtype=torch.int32, device=self.device)
        start = torch.empty(nb + 1, dtype=torch.int32, device=self.device)
        _lib.check(_lib.lib.esn_plan_sort_view(self.h, _ptr(perm), _ptr(keys), _ptr(start)))
        return perm, keys, start

    def target_chunks(self) -> int:
        """Target chunks of a type-2 plan's sort order (1 = plain bin order)."""
        n = ctypes.c_int()
        _lib.check(_lib.lib.esn_plan_target_chunks(self.h, ctypes.byref(n)))
        return int(n.value)

    def device_bytes(self) -> int:
        return int(_lib.lib.esn_plan_device_bytes(self.h))


class PlanCache:
    """Small LRU of Plans keyed by everything that shapes device state
    (the fft.py:87-111 plan-cache idea applied to whole transforms)."""

    def __init__(self, capacity: int = 6):
        self.capacity = capacity
        self._d: OrderedDict = OrderedDict()
        self._lock = threading.Lock()

    def get(self, key, factory):
        with self._lock:
            p = self._d.get(key)
            if p is not None:
                self._d.move_to_end(key)
                return p
        p = factory()
        with self._lock:
            self._d[key] = p
            while len(self._d) > self.capacity:
                _, old = self._d.popitem(last=False)
                old.close()
        return p

    def clear(self):
        with self._lock:
            for p in self._d.values():
                p.close()
            self._d.clear()

    def __len__(self):
        return len(self._d)


PLANS = PlanCache()


def raise_data_error(status: int, index: int, dim: int, coords=None, what="strength"):
    """Reference-worded DataError / BoundsViolationError
    (spreadinterp.py:95-98, 201-204; grid.py:159-164; transforms.py:92-97)."""
    if status == ErrorCode.DATA_ERROR:
        if dim > 0:
            raise DataError(f"non-finite coordinate at index {index} in dimension {dim}")
        raise DataError(f"non-finite {what} at index {index}")
    if status == ErrorCode.BOUNDS_VIOLATION:
        val = ""
        if coords is not None and dim > 0:
            val = repr(float(coords[dim - 1][index].item()))
        raise BoundsViolationError(f"coordinate {val} at index {index} outside [-3 pi, 3 pi]")
    _lib.check(status)
