"""The C ABI one-shot routines on HOST buffers (the esnufftpy convention):
pipelined (pinned buffers, >= 2 Mi points: chunked H2D / compute / D2H on
two streams) and plain paths against the CPU oracle and the device API."""

import ctypes

import numpy as np
import pytest
import torch

import cases

pytestmark = pytest.mark.gpu


def _call_host(ttype, coords, data, nm, tol, isign, dtype="float64", ntransf=1, pinned=True):
    from paper_1808_06736_b200 import _lib
    from paper_1808_06736_b200.plan import make_opts
    cplx = torch.complex128 if dtype == "float64" else torch.complex64
    M = len(coords[0])
    hx = [torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)) for x in coords]
    hd = torch.from_numpy(np.ascontiguousarray(data)).to(cplx)
    if ttype == 1:
        hout = torch.empty(((ntransf,) if ntransf > 1 else ()) + tuple(reversed(nm)), dtype=cplx)
    else:
        hout = torch.empty((ntransf, M) if ntransf > 1 else (M,), dtype=cplx)
    if pinned:
        hx = [x.pin_memory() for x in hx]
        hd = hd.pin_memory()
        hout = hout.pin_memory()
    cptr, fptr = (hd, hout) if ttype == 1 else (hout, hd)
    o, keep = make_opts(dtype=dtype, timing=False)
    xp = [ctypes.c_void_p(x.data_ptr()) for x in hx] + [None] * (3 - len(hx))
    st = _lib.lib.esn_nufft_host(ttype, len(coords), M, xp[0], xp[1], xp[2], ntransf,
                                 ctypes.c_void_p(cptr.data_ptr()), isign, tol, _lib.i64_array(nm),
                                 ctypes.c_void_p(fptr.data_ptr()), ctypes.byref(o))
    return st, hout.numpy()


@pytest.mark.parametrize("pinned", [True, False])
def test_host_type2_pipelined_matches_device(esn, pinned):
    coords, f, cfg = cases.make_inputs("c2", M=3_000_000)
    st, out = _call_host(2, coords, f, cfg["nm"], cfg["tol"], cfg["isign"], pinned=pinned)
    assert st == 0
    ref, _ = esn.exec_type2(coords, f, esn.TransformOptions(tolerance=cfg["tol"], isign=cfg["isign"]))
    assert np.linalg.norm(out - ref) <= 1e-13 * np.linalg.norm(ref)


def test_host_type1_pipelined_matches_device(esn):
    coords, c, cfg = cases.make_inputs("c3", M=2_500_000)
    st, out = _call_host(1, coords, c, cfg["nm"], cfg["tol"], cfg["isign"])
    assert st == 0
    ref, _ = esn.exec_type1(coords, c, cfg["nm"], esn.TransformOptions(tolerance=cfg["tol"], isign=cfg["isign"]))
    assert np.linalg.norm(out - ref) <= 1e-12 * np.linalg.norm(ref)


def test_host_batched_pipelined_matches_device(esn):
    coords, c, cfg = cases.make_inputs("c5", M=2_200_000, ntransf=5)
    st, out = _call_host(1, coords, c, cfg["nm"], cfg["tol"], cfg["isign"], dtype="float32", ntransf=5)
    assert st == 0
    ref, _ = esn.exec_type1([x.astype(np.float32) for x in coords], c.astype(np.complex64), cfg["nm"],
                            esn.TransformOptions(tolerance=cfg["tol"], isign=cfg["isign"], dtype="float32"))
    assert np.linalg.norm(out - ref) <= 1e-5 * np.linalg.norm(ref)


def test_host_status_codes(esn):
    from paper_1808_06736_b200 import _lib
    # argument misuse -> SIZE_ERROR (3) before any work (esnufftpy __init__.py:54-122)
    st = _lib.lib.esn_nufft_host(3, 1, 10, None, None, None, 1, None, 1, 1e-6, None, None, None)
    assert st == 3
    x = np.array([0.5, np.nan])
    st, _ = _call_host(1, [x], np.ones(2, complex), (8,), 1e-6, 1, pinned=False)
    assert st == 5  # DATA_ERROR
    st, _ = _call_host(1, [np.array([0.5])], np.ones(1, complex), (8,), 1e-20, 1, pinned=False)
    assert st == 1  # BAD_TOLERANCE
    assert "tolerance" in _lib.last_error()


@pytest.mark.parametrize("dim", [1, 2, 3])
@pytest.mark.parametrize("isign", [1, -1])
def test_host_type3_matches_device_and_oracle(esn, oracle, dim, isign):
    """esn_nufft{1,2,3}d3 (host buffers, C++ composition) against the
    Python device composition (same kernels) and the oracle's type 3."""
    from paper_1808_06736_b200 import _lib
    from paper_1808_06736_b200.plan import make_opts
    rng = np.random.default_rng(40 + dim)
    M, K, tol = 3000, 2500, 1e-6
    xs = [np.ascontiguousarray(rng.uniform(-2.0, 3.5, M)) for _ in range(dim)]
    ss = [np.ascontiguousarray(rng.uniform(-40.0, 25.0, K)) for _ in range(dim)]
    c = np.ascontiguousarray(rng.standard_normal(M) + 1j * rng.standard_normal(M))
    f = np.zeros(K, dtype=np.complex128)
    o, keep = make_opts(timing=False)
    P = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    fn = {1: _lib.lib.esn_nufft1d3, 2: _lib.lib.esn_nufft2d3, 3: _lib.lib.esn_nufft3d3}[dim]
    st = fn(M, *[P(x) for x in xs], P(c), isign, tol, K, *[P(s) for s in ss], P(f), ctypes.byref(o))
    assert st == 0, _lib.last_error()
    dev, _ = esn.exec_type3(xs, c, ss, esn.TransformOptions(tolerance=tol, isign=isign))
    assert np.linalg.norm(f - dev) <= 1e-13 * np.linalg.norm(dev)
    ref = oracle.exec_type3(xs, c, ss, tol=tol, isign=isign)
    assert np.linalg.norm(f - ref) <= 1e-3 * tol * np.linalg.norm(ref)


def test_host_type3_status_codes(esn):
    from paper_1808_06736_b200 import _lib
    x = np.array([0.5, 1.0])
    c = np.ones(2, complex)
    s = np.array([1.0, np.inf])
    f = np.zeros(2, complex)
    P = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    assert _lib.lib.esn_nufft1d3(2, P(x), P(c), 2, 1e-6, 2, P(s), P(f), None) == 3  # isign
    assert _lib.lib.esn_nufft1d3(2, P(x), P(c), 1, 1e-6, 2, P(s), P(f), None) == 5  # non-finite target
    assert "target" in _lib.last_error()
    assert _lib.lib.esn_nufft1d3(2, P(x), P(c), 1, 1e-6, 0, P(s), P(f), None) == 0  # no targets


def test_host_batched_transform_pipeline(esn):
    """ntransf > 32 with M below the point-chunk threshold runs the
    transform-group pipeline (groups of 32 transforms: strengths up, spread +
    FFT + deconvolution, modes down, overlapped): same result as the device
    API, and a non-finite strength in the FIRST group is still reported."""
    coords, c, cfg = cases.make_inputs("c5", M=300_000, ntransf=70)
    st, out = _call_host(1, coords, c, cfg["nm"], cfg["tol"], cfg["isign"], dtype="float32", ntransf=70)
    assert st == 0
    ref, _ = esn.exec_type1([x.astype(np.float32) for x in coords], c.astype(np.complex64), cfg["nm"],
                            esn.TransformOptions(tolerance=cfg["tol"], isign=cfg["isign"], dtype="float32"))
    assert np.linalg.norm(out - ref) <= 1e-5 * np.linalg.norm(ref)
    bad = c.copy()
    bad[3, 1234] = np.nan
    st, _ = _call_host(1, coords, bad, cfg["nm"], cfg["tol"], cfg["isign"], dtype="float32", ntransf=70)
    assert st == 5  # DATA_ERROR (errors.py:13-20)


@pytest.mark.parametrize("M,T", [(2_300_000, 1), (50_000, 1), (40_000, 40)])
def test_host_complex64_strengths_for_float64(esn, M, T):
    """esn_opts.strength_dtype = float32: complex64 host strengths for a
    float64 type-1 transform (c3's inputs) are upcast exactly on the device,
    through the point-chunk pipeline, the plain path and the transform-group
    pipeline: the same modes as complex128 strengths of the same values."""
    from paper_1808_06736_b200 import _lib
    from paper_1808_06736_b200.plan import make_opts
    rng = np.random.default_rng(41)
    coords = [rng.uniform(-np.pi, np.pi, M) for _ in range(3)]
    c = (rng.standard_normal((T, M)) + 1j * rng.standard_normal((T, M))).astype(np.complex64)
    if T == 1:
        c = c[0]
    nm = (24, 20, 18)
    ref_st, ref = _call_host(1, coords, c.astype(np.complex128), nm, 1e-6, 1, ntransf=T)
    assert ref_st == 0
    hx = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in coords]
    hc = torch.from_numpy(np.ascontiguousarray(c)).pin_memory()
    hout = torch.empty(((T,) if T > 1 else ()) + tuple(reversed(nm)), dtype=torch.complex128).pin_memory()
    o, keep = make_opts(dtype="float64", timing=False, strength_dtype="float32")
    st = _lib.lib.esn_nufft_host(1, 3, M, *[ctypes.c_void_p(x.data_ptr()) for x in hx], T,
                                 ctypes.c_void_p(hc.data_ptr()), 1, 1e-6, _lib.i64_array(nm),
                                 ctypes.c_void_p(hout.data_ptr()), ctypes.byref(o))
    assert st == 0
    out = hout.numpy()
    assert np.linalg.norm(out - ref) <= 1e-13 * np.linalg.norm(ref)


@pytest.mark.parametrize("M,T", [(2_300_000, 1), (60_000, 1), (40_000, 40)])
def test_host_float32_coordinates(esn, M, T):
    """esn_opts.coord_dtype = float32: a float32 plan's host coordinates go
    over as float32 (the device sort reads them directly) -- identical modes
    to float64 copies of the same values, in every host path."""
    from paper_1808_06736_b200 import _lib
    from paper_1808_06736_b200.plan import make_opts
    rng = np.random.default_rng(43)
    coords = [rng.uniform(-np.pi, np.pi, M).astype(np.float32) for _ in range(2)]
    c = (rng.standard_normal((T, M)) + 1j * rng.standard_normal((T, M))).astype(np.complex64)
    if T == 1:
        c = c[0]
    nm = (48, 40)
    ref_st, ref = _call_host(1, [x.astype(np.float64) for x in coords], c, nm, 1e-4, 1, dtype="float32", ntransf=T)
    assert ref_st == 0
    hx = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in coords]
    hc = torch.from_numpy(np.ascontiguousarray(c)).pin_memory()
    hout = torch.empty(((T,) if T > 1 else ()) + tuple(reversed(nm)), dtype=torch.complex64).pin_memory()
    o, keep = make_opts(dtype="float32", timing=False, coord_dtype="float32")
    st = _lib.lib.esn_nufft_host(1, 2, M, *[ctypes.c_void_p(x.data_ptr()) for x in hx], None, T,
                                 ctypes.c_void_p(hc.data_ptr()), 1, 1e-4, _lib.i64_array(nm),
                                 ctypes.c_void_p(hout.data_ptr()), ctypes.byref(o))
    assert st == 0
    assert np.linalg.norm(hout.numpy() - ref) <= 1e-6 * np.linalg.norm(ref)
