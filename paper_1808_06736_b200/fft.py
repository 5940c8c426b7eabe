"""FFT seam on cuFFT (mirrors esnufft.fft, fft.py:1-124).

FORWARD applies e^{+2 pi i l k / n} with no scaling (cuFFT CUFFT_INVERSE);
BACKWARD the conjugate sign.  Plans are cached inside libesnufft_b200.so
per (dim, sizes, dtype, batch, device) under a mutex (fft.py:87-111).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

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


def fft_exec(key: FftPlanKey, data):
    """Unnormalised n-D FFT of ``data`` (shape == key.shape, or a leading
    batch axis); numpy in -> numpy out, CUDA tensor in -> new CUDA tensor."""
    shape = tuple(data.shape)
    if shape == key.shape:
        batch, dims = 1, key.shape
    elif len(shape) == len(key.shape) + 1 and shape[1:] == key.shape:
        batch, dims = shape[0], key.shape
    else:
        raise SizeError(f"data shape {shape} does not match plan {key.shape}")
    if len(dims) > 3:
        raise SizeError("cuFFT seam supports 1..3 dimensions")
    dev = D.device_of(None)
    like_torch = D.is_torch(data)
    cd = torch.complex64 if (like_torch and data.dtype == torch.complex64) else torch.complex128
    t = D.as_complex(data, dev, cd).clone()
    nfine = list(reversed(dims))
    _lib.check(_lib.lib.esn_fft(len(dims), _lib.ESN_F32 if cd == torch.complex64 else _lib.ESN_F64,
                                batch, _lib.i64_array(nfine), ctypes.c_void_p(t.data_ptr()),
                                1 if key.direction == FORWARD else -1,
                                ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    return D.to_output(t, like_torch)


def get_plan(key: FftPlanKey):
    return key


def clear_plan_cache(key: FftPlanKey | None = None) -> None:
    """cuFFT plans live for the process (device memory is reclaimed with the
    context); kept for API compatibility."""
    return None
