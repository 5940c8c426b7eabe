"""FFT seam on cuFFT (mirrors esnufft.fft, fft.py:1-124).

FORWARD applies e^{+2 pi i l k / n} with no scaling (cuFFT CUFFT_INVERSE);
BACKWARD the conjugate sign.  Plans are built once per key and cached
(fft.py:87-111): ``get_plan`` returns an ``_FftPlan`` owning one cuFFT
handle (esn_fft_plan_create), ``clear_plan_cache`` destroys them.  A plan
is per (key, batch, precision, device, stream): a cuFFT handle owns one
work area, so two streams never share one.
"""

from __future__ import annotations

import ctypes
import threading
import time
from dataclasses import dataclass, field

import torch

from . import _device as D
from . import _lib
from .errors import SizeError

FORWARD = "forward"
BACKWARD = "backward"


@dataclass(frozen=True)
class FftPlanKey:
    shape: tuple
    direction: str
    threads: int = 1

    def __post_init__(self):
        if self.direction not in (FORWARD, BACKWARD):
            raise SizeError(f"direction must be forward/backward, got {self.direction}")
        if len(self.shape) < 1 or any(n < 1 for n in self.shape):
            raise SizeError(f"invalid transform shape {self.shape}")


@dataclass
class _FftPlan:
    """fft.py:44-49: the key, the strategy that runs it and its build time;
    here the strategy is always cuFFT and ``handle`` its esn_fft_plan."""

    key: FftPlanKey
    strategy: str
    build_time: float
    handle: ctypes.c_void_p = field(repr=False, default=None)
    batch: int = 1
    precision: str = "complex128"
    device: int = 0
    stream: int = 0

    def execute(self, t: torch.Tensor) -> None:
        """In place on a CUDA tensor of this plan's shape, batch and precision."""
        _lib.check(_lib.lib.esn_fft_plan_exec(self.handle, ctypes.c_void_p(t.data_ptr()),
                                              1 if self.key.direction == FORWARD else -1,
                                              ctypes.c_void_p(self.stream)))

    def _destroy(self) -> None:
        if self.handle:
            _lib.lib.esn_fft_plan_destroy(self.handle)
            self.handle = None


_cache: dict = {}
_cache_lock = threading.Lock()


def _build_plan(key: FftPlanKey, batch: int, precision: str, device: int, stream: int) -> _FftPlan:
    """fft.py:79-84: make the cuFFT plan (its own work area) and time it."""
    if len(key.shape) > 3:
        raise SizeError("cuFFT seam supports 1..3 dimensions")
    t0 = time.perf_counter()
    h = ctypes.c_void_p()
    with torch.cuda.device(device):
        _lib.check(_lib.lib.esn_fft_plan_create(len(key.shape),
                                                _lib.ESN_F32 if precision == "complex64" else _lib.ESN_F64,
                                                batch, _lib.i64_array(list(reversed(key.shape))),
                                                ctypes.byref(h)))
    return _FftPlan(key=key, strategy="cufft", build_time=time.perf_counter() - t0, handle=h,
                    batch=batch, precision=precision, device=device, stream=stream)


def get_plan(key: FftPlanKey, batch: int = 1, precision: str = "complex128", stream=None) -> _FftPlan:
    """fft.py:87-96: the cached plan for ``key`` (built on first use) on the
    current device and stream."""
    dev = D.device_of(None)
    st = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    ck = (key, batch, precision, dev.index, st)
    with _cache_lock:
        plan = _cache.get(ck)
    if plan is not None:
        return plan
    plan = _build_plan(key, batch, precision, dev.index, st)
    with _cache_lock:
        kept = _cache.setdefault(ck, plan)
    if kept is not plan:
        plan._destroy()
    return kept


def clear_plan_cache(key: FftPlanKey | None = None) -> None:
    """fft.py:99-106: drop every cached plan, or those of ``key``; with no
    key the handles the plan-less esn_fft keeps are dropped too."""
    with _cache_lock:
        if key is None:
            gone = list(_cache.values())
            _cache.clear()
        else:
            gone = [p for ck, p in _cache.items() if ck[0] == key]
            for ck in [ck for ck in _cache if ck[0] == key]:
                del _cache[ck]
    if (gone or key is None) and torch.cuda.is_available() and torch.cuda.is_initialized():
        torch.cuda.synchronize()  # no FFT of a dropped plan may still be running
    for p in gone:
        p._destroy()
    if key is None:
        _lib.lib.esn_fft_cache_clear()


def plan_cache_size() -> int:
    """fft.py:109-111."""
    with _cache_lock:
        return len(_cache)


def fft_exec(key: FftPlanKey, data):
    """Unnormalised n-D FFT of ``data`` (shape == key.shape, or a leading
    batch axis); numpy in -> numpy out, CUDA tensor in -> new CUDA tensor."""
    shape = tuple(data.shape)
    if shape == key.shape:
        batch = 1
    elif len(shape) == len(key.shape) + 1 and shape[1:] == key.shape:
        batch = shape[0]
    else:
        raise SizeError(f"data shape {shape} does not match plan {key.shape}")
    if len(key.shape) > 3:
        raise SizeError("cuFFT seam supports 1..3 dimensions")
    dev = D.device_of(None)
    like_torch = D.is_torch(data)
    cd = torch.complex64 if (like_torch and data.dtype == torch.complex64) else torch.complex128
    t = D.as_complex(data, dev, cd).clone()
    plan = get_plan(key, batch, "complex64" if cd == torch.complex64 else "complex128")
    plan.execute(t)
    return D.to_output(t, like_torch)
