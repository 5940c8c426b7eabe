"""Peer-mappable device buffers (CUDA IPC behind the C ABI's esn_peer_*).

One process per GPU: the owner allocates a buffer and publishes its 64-byte
handle; every other rank maps it into its own address space and its kernels
then load / store / RED into the owner's HBM over NVLink (NVSwitch: full
bandwidth to every peer).  Used by distributed.exec_type1_peer_reduced, where
every rank's spreader flushes its tiles straight into the root's fine grid.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib


class _Raw:
    """__cuda_array_interface__ view of raw device bytes."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 2}


class PeerBuffer:
    """Device memory owned by this process that peers can map."""

    def __init__(self, nbytes: int, device: torch.device):
        self.device = torch.device(device)
        self.nbytes = int(nbytes)
        ptr = ctypes.c_void_p()
        handle = ctypes.create_string_buffer(64)
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib.esn_peer_alloc(self.nbytes, ctypes.byref(ptr), handle))
        self.ptr = int(ptr.value)
        self.handle = bytes(handle.raw)
        self._bytes = torch.as_tensor(_Raw(self.ptr, self.nbytes), device=self.device)

    def tensor(self, dtype: torch.dtype, shape) -> torch.Tensor:
        """Zero-copy tensor over the buffer's first bytes."""
        n = int(torch.empty((), dtype=dtype).element_size())
        count = 1
        for v in shape:
            count *= int(v)
        if count * n > self.nbytes:
            raise ValueError("peer buffer too small for the requested view")
        return self._bytes[: count * n].view(dtype).view(tuple(shape))

    def free(self):
        if self.ptr:
            self._bytes = None
            with torch.cuda.device(self.device):
                _lib.check(_lib.lib.esn_peer_free(ctypes.c_void_p(self.ptr)))
            self.ptr = 0


_OPENED: dict[bytes, int] = {}


def open_peer(handle: bytes, device: torch.device) -> int:
    """Device pointer (valid on ``device``) of the buffer behind ``handle``;
    mapped once per process and cached (a handle can be opened only once)."""
    handle = bytes(handle)
    ptr = _OPENED.get(handle)
    if ptr is None:
        out = ctypes.c_void_p()
        with torch.cuda.device(device):
            _lib.check(_lib.lib.esn_peer_open(handle, ctypes.byref(out)))
        ptr = _OPENED[handle] = int(out.value)
    return ptr


def close_all_peers():
    for h, ptr in list(_OPENED.items()):
        _lib.lib.esn_peer_close(ctypes.c_void_p(ptr))
        del _OPENED[h]
