"""Device-buffer plumbing: numpy / torch inputs -> contiguous CUDA tensors.

PyTorch is used only for device memory, streams and torch.distributed.
All arithmetic of the transform runs in libesnufft_b200.so kernels.
"""

from __future__ import annotations

import numpy as np
import torch

from .errors import InternalError, SizeError

REAL = {"float64": torch.float64, "float32": torch.float32}
CPLX = {"float64": torch.complex128, "float32": torch.complex64}


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise InternalError(
            "no CUDA device: esnufft-b200 runs only on the GPU (there is no CPU fallback)")


def device_of(opts_device) -> torch.device:
    require_cuda()
    if opts_device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(opts_device)
    if dev.type != "cuda":
        raise SizeError(f"device must be a CUDA device, got {dev}")
    return dev


def is_torch(a) -> bool:
    return isinstance(a, torch.Tensor)


def as_real_1d(a, name: str, dev: torch.device, dtype=torch.float64) -> torch.Tensor:
    """1-D coordinate array on dev; float32 inputs are kept (the kernels
    fold in float64 regardless)."""
    if is_torch(a):
        t = a
        if t.dtype not in (torch.float64, torch.float32):
            t = t.to(torch.float64)
    else:
        arr = np.asarray(a)
        if arr.dtype not in (np.float64, np.float32):
            arr = arr.astype(np.float64)
        t = torch.from_numpy(np.ascontiguousarray(arr))
    if t.dtype != dtype and dtype == torch.float64 and t.dtype != torch.float32:
        t = t.to(dtype)
    return t.to(dev, non_blocking=False).contiguous()


def as_complex(a, dev: torch.device, cdtype: torch.dtype) -> torch.Tensor:
    if is_torch(a):
        t = a
        if not t.is_complex():
            t = t.to(torch.float64)
    else:
        arr = np.asarray(a)
        if not np.iscomplexobj(arr):
            arr = arr.astype(np.float64)
        t = torch.from_numpy(np.ascontiguousarray(arr))
    return t.to(device=dev, dtype=cdtype).contiguous()


def to_output(t: torch.Tensor, like_torch: bool):
    if like_torch:
        return t
    return t.cpu().numpy()
