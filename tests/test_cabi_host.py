"""CPU-side checks of the product (no GPU compute): the C ABI library loads
and exports every symbol include/esnufft_b200.h declares, the status table
matches the reference, and the host kernel math of libesnufft_b200.so
(esn_math.cpp) agrees with the reference's golden vectors."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "esnufft_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(esn_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_1808_06736_b200", "libesnufft_b200.so"))
    syms = header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    from paper_1808_06736_b200 import _lib
    assert set(syms) <= set(_lib.SIGNATURES), set(syms) - set(_lib.SIGNATURES)


def test_status_table_matches_reference():
    from paper_1808_06736_b200.errors import ErrorCode
    assert [int(c) for c in ErrorCode] == [0, 1, 2, 3, 4, 5, 6]
    assert [c.name for c in ErrorCode] == ["SUCCESS", "BAD_TOLERANCE", "BOUNDS_VIOLATION",
                                           "SIZE_ERROR", "RESOURCE_ERROR", "DATA_ERROR",
                                           "INTERNAL_ERROR"]
    hdr = open(os.path.join(ROOT, "include", "esnufft_b200.h")).read()
    for c in ErrorCode:
        assert re.search(rf"ESN_{c.name}\s*=\s*{int(c)}\b", hdr)


def test_host_params_exact(golden):
    import paper_1808_06736_b200 as E
    from paper_1808_06736_b200 import grid as G
    k = golden("kernel")
    for tol, sigma, w, beta, gamma, pq in k["params"]:
        p = E.select_params(tol, sigma)
        assert (p.w, p.beta, p.gamma, p.p_quad) == (w, beta, gamma, pq)
    for n, s in zip(k["smooth_in"], k["smooth"]):
        assert G.next_smooth(int(n)) == s
    for row in k["fine_sizes"]:
        nm = tuple(int(v) for v in row[:3] if v > 0)
        assert G.fine_grid_sizes(nm, row[3], int(row[4])) == tuple(int(v) for v in row[5:5 + len(nm)])


def test_host_quadrature_and_poly(golden):
    import paper_1808_06736_b200 as E
    from paper_1808_06736_b200 import kernel as K
    from cases import FSERIES_CASES
    k = golden("kernel")
    for n in (1, 2, 3, 5, 8, 16, 26, 37, 64):
        x, w = K.gauss_legendre(n)
        np.testing.assert_allclose(x, k[f"gl_x_{n}"], atol=1e-15)
        np.testing.assert_allclose(w, k[f"gl_w_{n}"], atol=1e-15)
    for i, (w, sigma, n, N) in enumerate(FSERIES_CASES):
        got = K.fseries_correction(E.params_for_width(w, sigma), n, N)
        np.testing.assert_allclose(got, k[f"fs_{i}"], rtol=5e-12)
    for w in range(2, 17):
        poly = K.build_piecewise_poly(E.params_for_width(w))
        assert poly.coeffs.shape == (w, w + 4)
        # Householder QR vs LAPACK gelsd: same least-squares minimiser
        np.testing.assert_allclose(poly.coeffs, k[f"poly_{w}"], atol=5e-15)
    np.testing.assert_allclose(K.kernel_ft(E.params_for_width(9), 0.05, k["kft_k"]), k["kft"],
                               rtol=1e-13, atol=1e-14 * np.abs(k["kft"]).max())


def test_host_errors_mirror_reference():
    import paper_1808_06736_b200 as E
    for bad in (1e-16, 0.5, 0.0, -1.0):
        with pytest.raises(E.BadToleranceError):
            E.select_params(bad)
    with pytest.raises(E.BadToleranceError):
        E.select_params(1e-6, 3.0)
    with pytest.raises(E.BadToleranceError):
        E.params_for_width(17)
    with pytest.raises(E.BadToleranceError):
        E.TransformOptions(tolerance=1e-20)
    with pytest.raises(E.SizeError):
        E.TransformOptions(isign=0)
    with pytest.raises(E.SizeError):
        E.TransformOptions(threads=-1)
    with pytest.raises(E.SizeError):
        E.TransformOptions(max_grid_values=0)
    assert E.__version__ == "0.1.0"
    for name in ["nufft1d1", "nufft2d1", "nufft3d1", "nufft1d2", "nufft2d2", "nufft3d2",
                 "nufft1d3", "nufft2d3", "nufft3d3", "exec_type1", "exec_type2", "exec_type3",
                 "direct_type1", "direct_type2", "direct_type3", "rel_l2", "aliasing_probe",
                 "ErrorReport", "KernelParams", "class_tolerance", "params_for_width",
                 "select_params", "TransformOptions", "ErrorCode", "EsnufftError"]:
        assert hasattr(E, name), name


def test_plan_without_gpu_fails_loudly():
    import torch
    import paper_1808_06736_b200 as E
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(E.InternalError):
        E.nufft1d1(np.zeros(3), np.ones(3, complex), 8)


def test_fft_plan_cache_api_without_gpu():
    """fft.py:99-111 surface: the cache starts empty, clear_plan_cache (all
    or one key) and plan_cache_size work on a host without a GPU; plans
    themselves are built on first use on the device (test_gpu_properties)."""
    from paper_1808_06736_b200 import fft
    from paper_1808_06736_b200.errors import SizeError
    fft.clear_plan_cache()
    assert fft.plan_cache_size() == 0
    fft.clear_plan_cache(fft.FftPlanKey((8, 8), fft.FORWARD))
    assert fft.plan_cache_size() == 0
    with pytest.raises(SizeError):
        fft.FftPlanKey((8,), "sideways")
