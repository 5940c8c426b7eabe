"""C-style status bindings over the C ABI (the ``esnufftpy`` drop-in).

Mirrors the reference's status-code binding package
(``/root/reference/pkg/bindings/src/esnufftpy/__init__.py:1-215``): nine
routines ``nufft{1,2,3}d{1,2,3}`` with array-in / array-out semantics.  The
caller allocates the output array, the routine fills it in place and
returns an int status (0 on success, else the stable ``ErrorCode``).

Argument misuse detectable without running a transform (wrong dtype,
non-contiguous or read-only storage, shape or length mismatch, bad isign
or thread count) is rejected here with ``SIZE_ERROR`` before any core
machinery runs (reference ``:54-109``).  The core behind each routine is
the matching C-ABI host-buffer routine of ``libesnufft_b200.so``
(``esn_nufft{1,2,3}d{1,2,3}``, ``include/esnufft_b200.h``): it reads the
caller's host arrays, runs the GPU transform and writes the result straight
into the caller's output buffer -- the one marshaling copy, as in the
reference (``:14-17``).  Core failures (unsupported tolerance, non-finite
data, grid caps) surface as their own codes.

``threads`` is validated exactly as the reference does and otherwise has no
effect: the transform runs on the current CUDA device.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import ErrorCode, EsnufftError
from .transforms import TransformOptions

__version__ = "0.1.0"

__all__ = [
    "ErrorCode",
    "nufft1d1", "nufft1d2", "nufft1d3",
    "nufft2d1", "nufft2d2", "nufft2d3",
    "nufft3d1", "nufft3d2", "nufft3d3",
]


_SIZE = int(ErrorCode.SIZE_ERROR)


def _is_int(v) -> bool:
    return isinstance(v, (int, np.integer)) and not isinstance(v, bool)


def _ok(a, dtype, *, ndim=None, shape=None, writable=False) -> bool:
    """The binding's storage contract for one array: an ndarray of exactly
    ``dtype``, C-contiguous, of the given rank / shape, writable if it is
    an output.  No conversion is ever attempted."""
    if not isinstance(a, np.ndarray) or a.dtype != dtype or not a.flags.c_contiguous:
        return False
    if shape is not None and a.shape != tuple(shape):
        return False
    if ndim is not None and a.ndim != ndim:
        return False
    return not writable or a.flags.writeable


def _point_count(arrays):
    """Shared length of 1-D float64 component arrays, or None."""
    if not all(_ok(a, np.float64, ndim=1) for a in arrays):
        return None
    lens = {a.shape[0] for a in arrays}
    return lens.pop() if len(lens) == 1 else None


def _flags_ok(isign, threads) -> bool:
    return isign in (1, -1) and _is_int(threads) and threads >= 0


def _modes(n_modes, dim):
    """(N_1..N_dim) from an int or a length-dim sequence of ints, or None."""
    if _is_int(n_modes):
        nm = (int(n_modes),) * dim
    elif isinstance(n_modes, (tuple, list)) and len(n_modes) == dim and all(_is_int(v) for v in n_modes):
        nm = tuple(int(v) for v in n_modes)
    else:
        return None
    return nm if min(nm) >= 1 else None


def _p(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a.size else None


# -- the core: one C-ABI host routine per (type, dim).  Module attributes so
# the contract tests can replace them with sentinels (reference
# test_bindings.py:94-105 does the same to the core entry points).

def exec_type1(coords, c, nm, opts, f) -> int:
    dim, m = len(coords), coords[0].shape[0]
    fn = (_lib.lib.esn_nufft1d1, _lib.lib.esn_nufft2d1, _lib.lib.esn_nufft3d1)[dim - 1]
    return int(fn(m, *[_p(x) for x in coords], _p(c), opts.isign, opts.tolerance, *nm, _p(f), None))


def exec_type2(coords, f, opts, c) -> int:
    dim, m = len(coords), coords[0].shape[0]
    nm = tuple(reversed(f.shape))
    fn = (_lib.lib.esn_nufft1d2, _lib.lib.esn_nufft2d2, _lib.lib.esn_nufft3d2)[dim - 1]
    return int(fn(m, *[_p(x) for x in coords], _p(c), opts.isign, opts.tolerance, *nm, _p(f), None))


def exec_type3(coords, c, targets, opts, f) -> int:
    dim, m, k = len(coords), coords[0].shape[0], targets[0].shape[0]
    fn = (_lib.lib.esn_nufft1d3, _lib.lib.esn_nufft2d3, _lib.lib.esn_nufft3d3)[dim - 1]
    return int(fn(m, *[_p(x) for x in coords], _p(c), opts.isign, opts.tolerance, k,
                  *[_p(s) for s in targets], _p(f), None))


def _run(call, isign, tol, threads) -> int:
    """Validate the options the way the core does (TransformOptions,
    reference transforms.py:44-80), then run the C routine, which writes
    the caller's buffer in place."""
    try:
        opts = TransformOptions(tolerance=tol, isign=isign, threads=threads)
        return int(call(opts))
    except EsnufftError as exc:
        return int(exc.code)
    except Exception:
        return int(ErrorCode.INTERNAL_ERROR)


def _type1(coords, c, isign, tol, n_modes, f, threads) -> int:
    m = _point_count(coords)
    nm = _modes(n_modes, len(coords))
    if (m is None or not _ok(c, np.complex128, shape=(m,)) or not _flags_ok(isign, threads) or nm is None
            or not _ok(f, np.complex128, shape=tuple(reversed(nm)), writable=True)):
        return _SIZE
    return _run(lambda o: exec_type1(coords, c, nm, o, f), isign, tol, threads)


def _type2(coords, c, isign, tol, f, threads) -> int:
    m = _point_count(coords)
    if (m is None or not _ok(c, np.complex128, shape=(m,), writable=True) or not _flags_ok(isign, threads)
            or not _ok(f, np.complex128, ndim=len(coords)) or min(f.shape) < 1):
        return _SIZE
    return _run(lambda o: exec_type2(coords, f, o, c), isign, tol, threads)


def _type3(coords, c, isign, tol, targets, f, threads) -> int:
    m = _point_count(coords)
    k = _point_count(targets)
    if (m is None or k is None or not _ok(c, np.complex128, shape=(m,)) or not _flags_ok(isign, threads)
            or not _ok(f, np.complex128, shape=(k,), writable=True)):
        return _SIZE
    return _run(lambda o: exec_type3(coords, c, targets, o, f), isign, tol, threads)


def nufft1d1(x, c, isign, tol, n_modes, f, threads=1) -> int:
    """f[k] = sum_j c[j] exp(isign i k x[j]); fills f of shape (N1,)."""
    return _type1((x,), c, isign, tol, n_modes, f, threads)


def nufft2d1(x, y, c, isign, tol, n_modes, f, threads=1) -> int:
    """2D type 1; n_modes is (N1, N2) or an int, f has shape (N2, N1)."""
    return _type1((x, y), c, isign, tol, n_modes, f, threads)


def nufft3d1(x, y, z, c, isign, tol, n_modes, f, threads=1) -> int:
    """3D type 1; n_modes is (N1, N2, N3) or an int, f has shape (N3, N2, N1)."""
    return _type1((x, y, z), c, isign, tol, n_modes, f, threads)


def nufft1d2(x, c, isign, tol, f, threads=1) -> int:
    """c[j] = sum_k f[k] exp(isign i k x[j]); fills c of length len(x)."""
    return _type2((x,), c, isign, tol, f, threads)


def nufft2d2(x, y, c, isign, tol, f, threads=1) -> int:
    """2D type 2 reading modes f of shape (N2, N1); fills c."""
    return _type2((x, y), c, isign, tol, f, threads)


def nufft3d2(x, y, z, c, isign, tol, f, threads=1) -> int:
    """3D type 2 reading modes f of shape (N3, N2, N1); fills c."""
    return _type2((x, y, z), c, isign, tol, f, threads)


def nufft1d3(x, c, isign, tol, s, f, threads=1) -> int:
    """f[k] = sum_j c[j] exp(isign i s[k] x[j]); fills f of length len(s)."""
    return _type3((x,), c, isign, tol, (s,), f, threads)


def nufft2d3(x, y, c, isign, tol, s, t, f, threads=1) -> int:
    """2D type 3 with target components (s[k], t[k]); fills f."""
    return _type3((x, y), c, isign, tol, (s, t), f, threads)


def nufft3d3(x, y, z, c, isign, tol, s, t, u, f, threads=1) -> int:
    """3D type 3 with target components (s[k], t[k], u[k]); fills f."""
    return _type3((x, y, z), c, isign, tol, (s, t, u), f, threads)
