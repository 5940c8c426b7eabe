"""ctypes binding of libesnufft_b200.so (the C ABI in include/esnufft_b200.h).

The shared library is REQUIRED: there is no CPU fallback anywhere in this
package.  If it is missing, importing the package raises ImportError with
the build command; every transform then fails loudly instead of silently
running something else.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ErrorCode, raise_for_status

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_NAME = "libesnufft_b200.so"
LIB_PATH = os.path.join(HERE, LIB_NAME)

ESN_F64, ESN_F32 = 0, 1
METHOD_AUTO, METHOD_GLOBAL, METHOD_TILE = 0, 1, 2

i32, i64, dbl, vp = ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
P_i64 = ctypes.POINTER(ctypes.c_int64)
P_dbl = ctypes.POINTER(ctypes.c_double)


class KernelParamsC(ctypes.Structure):
    _fields_ = [("w", i32), ("beta", dbl), ("sigma", dbl), ("gamma", dbl), ("p_quad", i32)]


class OptsC(ctypes.Structure):
    _fields_ = [
        ("sigma", dbl), ("check_bounds", i32), ("use_exact_kernel", i32),
        ("max_grid_values", i64), ("dtype", i32), ("method", i32),
        ("bin_size", i32 * 3), ("max_subprob", i32), ("timing", i32),
        ("stream", vp), ("params", ctypes.POINTER(KernelParamsC)), ("coeffs", P_dbl),
        ("strength_dtype", i32), ("coord_dtype", i32),
    ]


# name -> (restype, argtypes); the exported surface of include/esnufft_b200.h
SIGNATURES = {
    "esn_version": (i32, []),
    "esn_last_error": (ctypes.c_char_p, []),
    "esn_select_params": (i32, [dbl, dbl, ctypes.POINTER(KernelParamsC)]),
    "esn_params_for_width": (i32, [i32, dbl, ctypes.POINTER(KernelParamsC)]),
    "esn_class_tolerance": (dbl, [i32, dbl]),
    "esn_next_smooth": (i32, [i64, P_i64]),
    "esn_fine_grid_sizes": (i32, [i32, P_i64, dbl, i32, P_i64]),
    "esn_gauss_legendre": (i32, [i32, P_dbl, P_dbl]),
    "esn_kernel_ft": (i32, [ctypes.POINTER(KernelParamsC), dbl, i64, P_dbl, P_dbl]),
    "esn_fseries_correction": (i32, [ctypes.POINTER(KernelParamsC), i64, i64, P_dbl]),
    "esn_piecewise_poly": (i32, [ctypes.POINTER(KernelParamsC), P_dbl, P_dbl]),
    "esn_default_opts": (None, [ctypes.POINTER(OptsC)]),
    "esn_plan_create": (i32, [i32, i32, P_i64, i32, i32, dbl, ctypes.POINTER(OptsC), ctypes.POINTER(vp)]),
    "esn_spreader_create": (i32, [i32, P_i64, i32, ctypes.POINTER(OptsC), ctypes.POINTER(vp)]),
    "esn_plan_setpts": (i32, [vp, i64, i32, vp, vp, vp]),
    "esn_plan_execute": (i32, [vp, vp, vp]),
    "esn_plan_spread": (i32, [vp, vp, vp]),
    "esn_plan_interp": (i32, [vp, vp, vp]),
    "esn_plan_check": (i32, [vp, P_i64]),
    "esn_plan_stage_times": (i32, [vp, P_dbl, P_dbl, P_dbl, P_dbl]),
    "esn_plan_hot_kernel_seconds": (i32, [vp, P_dbl]),
    "esn_plan_info": (i32, [vp, P_i64, ctypes.POINTER(KernelParamsC)]),
    "esn_plan_device_bytes": (i64, [vp]),
    "esn_plan_destroy": (i32, [vp]),
    "esn_plan_sort_view": (i32, [vp, vp, vp, vp]),
    "esn_plan_finish_type1": (i32, [vp, vp, vp]),
    "esn_plan_spread_add": (i32, [vp, vp, vp]),
    "esn_peer_alloc": (i32, [i64, ctypes.POINTER(vp), ctypes.c_char_p]),
    "esn_peer_open": (i32, [ctypes.c_char_p, ctypes.POINTER(vp)]),
    "esn_peer_close": (i32, [vp]),
    "esn_peer_free": (i32, [vp]),
    "esn_plan_target_chunks": (i32, [vp, vp]),
    "esn_plan_bins": (i32, [vp, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i32)]),
    "esn_plan_tasks": (i32, [vp, P_i64]),
    "esn_fold_coords": (i32, [i64, i32, vp, i64, vp, vp]),
    "esn_fft": (i32, [i32, i32, i32, P_i64, vp, i32, vp]),
    "esn_fft_plan_create": (i32, [i32, i32, i32, P_i64, ctypes.POINTER(vp)]),
    "esn_fft_plan_exec": (i32, [vp, vp, i32, vp]),
    "esn_fft_plan_work_bytes": (i64, [vp]),
    "esn_fft_plan_destroy": (i32, [vp]),
    "esn_fft_cache_clear": (i32, []),
    "esn_type3_prephase": (i32, [i32, i64, vp, vp, vp, P_dbl, P_dbl, P_dbl, i32, vp, vp, vp, vp, vp, vp]),
    "esn_type3_targets": (i32, [i32, i64, vp, vp, vp, P_dbl, P_dbl, P_i64, vp, vp, vp, vp]),
    "esn_type3_correct": (i32, [i32, i64, vp, vp, vp, P_dbl, P_dbl, P_dbl, P_i64,
                                ctypes.POINTER(KernelParamsC), i32, vp, vp]),
    "esn_fftshift": (i32, [i32, P_i64, vp, vp, vp]),
    "esn_direct": (i32, [i32, i64, vp, vp, vp, vp, i64, vp, vp, vp, i32, vp, vp]),
    "esn_nufft1d3": (i32, [i64, vp, vp, i32, dbl, i64, vp, vp, ctypes.POINTER(OptsC)]),
    "esn_nufft2d3": (i32, [i64, vp, vp, vp, i32, dbl, i64, vp, vp, vp, ctypes.POINTER(OptsC)]),
    "esn_nufft3d3": (i32, [i64, vp, vp, vp, vp, i32, dbl, i64, vp, vp, vp, vp, ctypes.POINTER(OptsC)]),
    "esn_nufft1d1": (i32, [i64, vp, vp, i32, dbl, i64, vp, ctypes.POINTER(OptsC)]),
    "esn_nufft2d1": (i32, [i64, vp, vp, vp, i32, dbl, i64, i64, vp, ctypes.POINTER(OptsC)]),
    "esn_nufft3d1": (i32, [i64, vp, vp, vp, vp, i32, dbl, i64, i64, i64, vp, ctypes.POINTER(OptsC)]),
    "esn_nufft1d2": (i32, [i64, vp, vp, i32, dbl, i64, vp, ctypes.POINTER(OptsC)]),
    "esn_nufft2d2": (i32, [i64, vp, vp, vp, i32, dbl, i64, i64, vp, ctypes.POINTER(OptsC)]),
    "esn_nufft3d2": (i32, [i64, vp, vp, vp, vp, i32, dbl, i64, i64, i64, vp, ctypes.POINTER(OptsC)]),
    "esn_nufft_host": (i32, [i32, i32, i64, vp, vp, vp, i32, vp, i32, dbl, P_i64, vp,
                             ctypes.POINTER(OptsC)]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_NAME} not found at {LIB_PATH}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (make -C "
            "paper_1808_06736_b200/csrc).  There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def last_error() -> str:
    msg = lib.esn_last_error()
    return msg.decode() if msg else ""


def check(status: int) -> None:
    """Map a C status int to the reference exception classes."""
    if status != ErrorCode.SUCCESS:
        raise_for_status(int(status), last_error())


def i64_array(vals):
    arr = (ctypes.c_int64 * max(1, len(vals)))()
    for i, v in enumerate(vals):
        arr[i] = int(v)
    return arr
