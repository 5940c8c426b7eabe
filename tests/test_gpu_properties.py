"""The reference's hot-path properties re-asserted on the GPU path
(pkg/tests/test_spreadinterp.py, test_transforms.py, test_acceptance.py):
single-point kernel, linearity, adjointness, periodic alias / h-shift,
run-to-run invariance (atomics: to rounding), closed forms,
direct-sum accuracy (<= 10 eps), isign, float32 and batched paths, options,
and the error classes / messages."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TWO_PI = 2 * np.pi


def _periodized(x, n, w, beta):
    # test_spreadinterp.py:18-26: psi~(l h - x) summed over periodic images
    h = TWO_PI / n
    alpha = 0.5 * w * h
    l = np.arange(n) * h
    out = np.zeros(n)
    for shift in (-TWO_PI, 0.0, TWO_PI):
        z = (l - x + shift) / alpha
        ins = np.abs(z) <= 1
        out[ins] += np.exp(beta * (np.sqrt(1 - z[ins] ** 2) - 1))
    return out


@pytest.mark.parametrize("method", ["tile", "global"])
def test_single_point_spread_is_kernel(esn, method):
    from paper_1808_06736_b200 import spreadinterp as SI
    p = esn.params_for_width(7)
    n = 64
    for x in [0.0, 0.1, np.pi, TWO_PI - 1e-3, 2.5]:
        g = SI.spread(SI.build_point_set([np.array([x])], (n,)), np.array([1.5 - 0.5j]), p,
                      use_exact=True, method=method)
        np.testing.assert_allclose(g, (1.5 - 0.5j) * _periodized(x, n, 7, p.beta), atol=1e-14)
    n2 = (16, 20, 18)
    xs = (2.2, 0.4, 5.9)
    g = SI.spread(SI.build_point_set([np.array([v]) for v in xs], n2), np.array([1.0 + 0j]), p,
                  use_exact=True, method=method)
    ks = [_periodized(xs[d], n2[d], 7, p.beta) for d in range(3)]
    np.testing.assert_allclose(g.real, np.einsum("c,b,a->cba", ks[2], ks[1], ks[0]), atol=1e-14)


@pytest.mark.parametrize("dim", [1, 2, 3])
def test_adjointness_and_linearity(esn, dim):
    from paper_1808_06736_b200 import spreadinterp as SI
    rng = np.random.default_rng(dim)
    sizes = {1: (48,), 2: (40, 36), 3: (24, 20, 18)}[dim]
    m = 3000
    p = esn.params_for_width(7)
    pts = SI.build_point_set([rng.uniform(0, TWO_PI, m) for _ in range(dim)], sizes)
    c = rng.standard_normal(m) + 1j * rng.standard_normal(m)
    c2 = rng.standard_normal(m) + 1j * rng.standard_normal(m)
    b = rng.standard_normal(tuple(reversed(sizes))) + 1j * rng.standard_normal(tuple(reversed(sizes)))
    lhs = np.vdot(b, SI.spread(pts, c, p))
    rhs = np.vdot(SI.interp(pts, b, p), c)
    assert abs(lhs - rhs) <= 1e-13 * abs(lhs)
    g1, g2 = SI.spread(pts, c, p), SI.spread(pts, c2, p)
    g12 = SI.spread(pts, 2.0 * c - 1j * c2, p)
    np.testing.assert_allclose(g12, 2.0 * g1 - 1j * g2, atol=1e-13 * np.abs(c).max())
    assert not np.any(SI.spread(pts, np.zeros(m, complex), p))


def test_alias_and_shift(esn):
    from paper_1808_06736_b200 import spreadinterp as SI
    rng = np.random.default_rng(8)
    p = esn.params_for_width(7)
    x = rng.uniform(np.pi, TWO_PI, 500)
    c = rng.standard_normal(500) + 1j * rng.standard_normal(500)
    g1 = SI.spread(SI.build_point_set([x], (128,)), c, p)
    g2 = SI.spread(SI.build_point_set([x - TWO_PI], (128,)), c, p)
    # folds are bit-identical; spread sums differ only by atomic order
    np.testing.assert_allclose(g1, g2, atol=1e-14 * np.abs(c).sum())
    n = 90
    h = TWO_PI / n
    x = rng.uniform(0, TWO_PI - h, 400)
    g = SI.spread(SI.build_point_set([x], (n,)), c[:400], p)
    gs = SI.spread(SI.build_point_set([x + h], (n,)), c[:400], p)
    np.testing.assert_allclose(gs, np.roll(g, 1), atol=1e-13 * np.abs(c[:400]).sum())


@pytest.mark.parametrize("ttype", [1, 2])
def test_run_to_run_invariance(esn, ttype):
    rng = np.random.default_rng(12)
    m = 200_000
    coords = [rng.uniform(-np.pi, np.pi, m) for _ in range(3)]
    o = esn.TransformOptions(tolerance=1e-9)
    if ttype == 1:
        c = rng.standard_normal(m) + 1j * rng.standard_normal(m)
        a = esn.exec_type1(coords, c, (32, 30, 28), o)[0]
        b = esn.exec_type1(coords, c, (32, 30, 28), o)[0]
        assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(a)
    else:
        f = rng.standard_normal((28, 30, 32)) + 1j * rng.standard_normal((28, 30, 32))
        a = esn.exec_type2(coords, f, o)[0]
        b = esn.exec_type2(coords, f, o)[0]
        np.testing.assert_array_equal(a, b)  # interp is a pure gather: bitwise


def test_closed_forms(esn):
    f = esn.nufft1d1(np.array([0.0]), np.array([1.0 + 0j]), 8, tolerance=1e-9)
    np.testing.assert_allclose(f, np.ones(8), atol=1e-9)
    modes = np.zeros(9, complex)
    modes[4] = 1.0
    x = np.random.default_rng(0).uniform(-np.pi, np.pi, 25)
    np.testing.assert_allclose(esn.nufft1d2(x, modes, tolerance=1e-9), np.ones(25), atol=1e-9)
    out = esn.nufft1d3(np.array([0.7]), np.array([1.0 + 0j]), np.array([1.3]), tolerance=1e-9)
    np.testing.assert_allclose(out, [np.exp(0.91j)], atol=1e-9)


@pytest.mark.parametrize("dim", [1, 2, 3])
@pytest.mark.parametrize("isign", [1, -1])
def test_vs_direct_sum(esn, oracle, dim, isign):
    """<= 10 eps vs the exact direct sum (test_transforms.py:49-84), and the
    GPU direct sum equals the CPU one."""
    rng = np.random.default_rng(dim * 10 + isign)
    coords = [rng.uniform(-np.pi, np.pi, 400) for _ in range(dim)]
    c = rng.standard_normal(400) + 1j * rng.standard_normal(400)
    nm = {1: (50,), 2: (14, 10), 3: (8, 6, 7)}[dim]
    for tol in (1e-3, 1e-6, 1e-9, 1e-12):
        fast, _ = esn.exec_type1(coords, c, nm, esn.TransformOptions(tolerance=tol, isign=isign))
        exact = oracle.direct_type1(coords, c, nm, isign=isign)
        assert esn.rel_l2(fast, exact).rel_l2 <= 10 * tol
        f = rng.standard_normal(tuple(reversed(nm))) + 1j * rng.standard_normal(tuple(reversed(nm)))
        fast2, _ = esn.exec_type2(coords, f, esn.TransformOptions(tolerance=tol, isign=isign))
        assert esn.rel_l2(fast2, oracle.direct_type2(coords, f, isign=isign)).rel_l2 <= 10 * tol
    gpu_direct = esn.direct_type1(coords, c, nm, isign=isign)
    np.testing.assert_allclose(gpu_direct, oracle.direct_type1(coords, c, nm, isign=isign), rtol=1e-11,
                               atol=1e-11 * np.abs(gpu_direct).max())


def test_float32_and_batched_paths(esn, oracle):
    rng = np.random.default_rng(3)
    m, T, nm = 50_000, 5, (64, 48)
    coords = [rng.uniform(-np.pi, np.pi, m).astype(np.float32) for _ in range(2)]
    c = (rng.standard_normal((T, m)) + 1j * rng.standard_normal((T, m))).astype(np.complex64)
    o = esn.TransformOptions(tolerance=1e-4, dtype="float32")
    batched, _ = esn.exec_type1(coords, c, nm, o)
    assert batched.shape == (T, 48, 64) and batched.dtype == np.complex64
    c64 = [x.astype(np.float64) for x in coords]
    for t in range(T):
        single, _ = esn.exec_type1(coords, c[t], nm, o)
        assert np.linalg.norm(single - batched[t]) <= 1e-5 * np.linalg.norm(single)
        ref = oracle.exec_type1(c64, c[t].astype(np.complex128), nm, tol=1e-4)
        assert np.linalg.norm(batched[t] - ref) <= 10 * 1e-4 * np.linalg.norm(ref)
    f = (rng.standard_normal((T, 48, 64)) + 1j * rng.standard_normal((T, 48, 64))).astype(np.complex64)
    outb, _ = esn.exec_type2(coords, f, o)
    assert outb.shape == (T, m)
    for t in range(T):
        ref = oracle.exec_type2(c64, f[t].astype(np.complex128), tol=1e-4)
        assert np.linalg.norm(outb[t] - ref) <= 10 * 1e-4 * np.linalg.norm(ref)


def test_torch_in_torch_out(esn):
    dev = torch.device("cuda")
    x = torch.rand(1000, dtype=torch.float64, device=dev) * 6 - 3
    y = torch.rand(1000, dtype=torch.float64, device=dev) * 6 - 3
    c = torch.randn(1000, dtype=torch.complex128, device=dev)
    f = esn.nufft2d1(x, y, c, (16, 12), tolerance=1e-8)
    assert isinstance(f, torch.Tensor) and f.is_cuda and f.shape == (12, 16)
    ref = esn.nufft2d1(x.cpu().numpy(), y.cpu().numpy(), c.cpu().numpy(), (16, 12), tolerance=1e-8)
    np.testing.assert_allclose(f.cpu().numpy(), ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


def test_options_exact_sigma_bounds(esn, oracle):
    rng = np.random.default_rng(15)
    coords = [rng.uniform(-np.pi, np.pi, 300) for _ in range(2)]
    c = rng.standard_normal(300) + 1j * rng.standard_normal(300)
    poly, _ = esn.exec_type1(coords, c, (20, 16), esn.TransformOptions(tolerance=1e-8))
    exact, _ = esn.exec_type1(coords, c, (20, 16), esn.TransformOptions(tolerance=1e-8, use_exact_kernel=True))
    assert esn.rel_l2(poly, exact).rel_l2 <= 1e-8
    fast, _ = esn.exec_type1(coords, c, (18, 12), esn.TransformOptions(tolerance=1e-7, sigma=1.25))
    assert esn.rel_l2(fast, oracle.direct_type1(coords, c, (18, 12))).rel_l2 <= 1e-6
    x = np.array([0.5, 20.0])
    with pytest.raises(esn.BoundsViolationError) as e:
        esn.exec_type1((x,), np.ones(2, complex), (8,), esn.TransformOptions(check_bounds=True))
    assert "index 1" in str(e.value)
    out, _ = esn.exec_type1((x,), np.ones(2, complex), (8,), esn.TransformOptions())
    assert np.all(np.isfinite(out))


def test_errors_mirror_reference(esn):
    x = np.array([0.5, 1.0])
    c = np.ones(2, dtype=complex)
    with pytest.raises(esn.SizeError):
        esn.exec_type1((x,), np.ones(3, dtype=complex), (8,), esn.TransformOptions())
    with pytest.raises(esn.SizeError):
        esn.exec_type1((x, x), c, (8,), esn.TransformOptions())
    with pytest.raises(esn.DataError) as e:
        esn.exec_type1((np.array([0.5, np.nan]),), c, (8,), esn.TransformOptions())
    assert "index 1" in str(e.value)
    with pytest.raises(esn.DataError) as e:
        esn.exec_type1((x,), np.array([1.0, np.nan + 0j]), (8,), esn.TransformOptions())
    assert "index 1" in str(e.value)
    with pytest.raises(esn.DataError) as e:
        esn.exec_type2((x,), np.array([1.0, np.inf, 0j]), esn.TransformOptions())
    assert "index 1" in str(e.value)
    with pytest.raises(esn.SizeError):
        esn.exec_type2((x, x), np.zeros(8, dtype=complex), esn.TransformOptions())
    with pytest.raises(esn.SizeError):
        esn.exec_type3((x,), c, (np.zeros(3), np.zeros(3)), esn.TransformOptions())
    with pytest.raises(esn.DataError):
        esn.exec_type3((x,), c, (np.array([0.0, np.inf]),), esn.TransformOptions())
    with pytest.raises(esn.ResourceError) as e:
        esn.exec_type1((x,), c, (64,), esn.TransformOptions(max_grid_values=100))
    assert "direct summation" in str(e.value)


def test_wrappers_cover_all_nine(esn):
    rng = np.random.default_rng(18)
    m = 40
    x, y, z = (rng.uniform(-np.pi, np.pi, m) for _ in range(3))
    c = rng.standard_normal(m) + 1j * rng.standard_normal(m)
    s, t, u = (rng.uniform(-10, 10, 12) for _ in range(3))
    kw = dict(tolerance=1e-8)
    assert esn.nufft1d1(x, c, 10, **kw).shape == (10,)
    assert esn.nufft2d1(x, y, c, (10, 6), **kw).shape == (6, 10)
    assert esn.nufft3d1(x, y, z, c, 4, **kw).shape == (4, 4, 4)
    assert esn.nufft1d2(x, np.ones(10, dtype=complex), **kw).shape == (m,)
    assert esn.nufft2d2(x, y, np.ones((6, 10), dtype=complex), **kw).shape == (m,)
    assert esn.nufft3d2(x, y, z, np.ones((4, 4, 4), dtype=complex), **kw).shape == (m,)
    assert esn.nufft1d3(x, c, s, **kw).shape == (12,)
    assert esn.nufft2d3(x, y, c, s, t, **kw).shape == (12,)
    assert esn.nufft3d3(x, y, z, c, s, t, u, **kw).shape == (12,)
    f2 = esn.nufft2d1(x, y, c, (10, 6), **kw)
    np.testing.assert_allclose(f2, esn.direct_type1([x, y], c, (10, 6)), atol=1e-6 * np.abs(c).sum())


def test_fft_seam_sign_and_roundtrip(esn):
    from paper_1808_06736_b200.fft import BACKWARD, FORWARD, FftPlanKey, fft_exec
    d = np.zeros(4, complex)
    d[0] = 1
    np.testing.assert_allclose(fft_exec(FftPlanKey((4,), FORWARD), d), np.ones(4), atol=1e-15)
    rng = np.random.default_rng(1)
    a = rng.standard_normal((12, 10)) + 1j * rng.standard_normal((12, 10))
    k = np.arange(10)
    naive = np.exp(2j * np.pi * np.outer(k, k) / 10)  # e^{+2 pi i lk/n} (fft.py:3-6)
    got = fft_exec(FftPlanKey((12, 10), FORWARD), a)
    ref = np.exp(2j * np.pi * np.outer(np.arange(12), np.arange(12)) / 12) @ a @ naive.T
    np.testing.assert_allclose(got, ref, atol=1e-11)
    back = fft_exec(FftPlanKey((12, 10), BACKWARD), got)
    np.testing.assert_allclose(back, 120 * a, atol=1e-10)


@pytest.mark.gpu
def test_fft_plan_cache(esn):
    """fft.py:87-111: get_plan builds once per key and caches; plan_cache_size
    counts; clear_plan_cache(key) / () drop; a cached plan executes like the
    plan-less path (reference test: esnufft tests/test_fft.py plan cache)."""
    import torch
    from paper_1808_06736_b200 import fft as F
    F.clear_plan_cache()
    assert F.plan_cache_size() == 0
    k1, k2 = F.FftPlanKey((16, 12), F.FORWARD), F.FftPlanKey((9,), F.BACKWARD)
    p1 = F.get_plan(k1)
    assert F.get_plan(k1) is p1 and p1.strategy == "cufft" and p1.build_time >= 0
    F.get_plan(k2)
    assert F.plan_cache_size() == 2
    rng = np.random.default_rng(5)
    a = rng.standard_normal((16, 12)) + 1j * rng.standard_normal((16, 12))
    t = torch.tensor(a, device="cuda")
    p1.execute(t)
    np.testing.assert_allclose(t.cpu().numpy(), np.fft.ifftn(a) * a.size, atol=1e-11)
    np.testing.assert_allclose(F.fft_exec(k1, a), np.fft.ifftn(a) * a.size, atol=1e-11)
    F.clear_plan_cache(k2)
    assert F.plan_cache_size() == 1 and F.get_plan(k1) is p1
    F.clear_plan_cache()
    assert F.plan_cache_size() == 0
    np.testing.assert_allclose(F.fft_exec(k1, a), np.fft.ifftn(a) * a.size, atol=1e-11)


@pytest.mark.gpu
def test_spread_interp_stats(esn):
    """spreadinterp.py:165-184: stats gets busy_per_thread and tasks (plus the
    GPU stage times)."""
    from paper_1808_06736_b200 import spreadinterp as S
    from paper_1808_06736_b200.kernel import select_params
    rng = np.random.default_rng(6)
    m = 20_000
    xs = [rng.uniform(-np.pi, np.pi, m) for _ in range(2)]
    c = rng.standard_normal(m) + 1j * rng.standard_normal(m)
    kp = select_params(1e-6)
    pts = S.build_point_set(xs, (64, 48))
    st = {}
    g = S.spread(pts, c, kp, stats=st)
    assert st["tasks"] >= 1 and set(st["busy_per_thread"]) == {0} and st["busy_per_thread"][0] > 0
    st2 = {}
    S.interp(pts, g, kp, stats=st2)
    assert st2["tasks"] >= 1 and st2["busy_per_thread"][0] > 0


@pytest.mark.gpu
def test_error_tracks_tolerance(esn, oracle):
    """Reference tests/test_transforms.py error_tracks_tolerance_slope: the
    achieved error against the exact sum falls with the requested tolerance,
    log-log slope close to 1, and stays within 10 tol."""
    rng = np.random.default_rng(6)
    m, nm = 400, (60,)
    x = [rng.uniform(-np.pi, np.pi, m)]
    c = rng.standard_normal(m) + 1j * rng.standard_normal(m)
    exact = oracle.direct_type1(x, c, nm)
    tols = [1e-3, 1e-5, 1e-7, 1e-9, 1e-11]
    errs = []
    for tol in tols:
        got, _ = esn.exec_type1(x, c, nm, esn.TransformOptions(tolerance=tol))
        errs.append(max(float(np.linalg.norm(got - exact) / np.linalg.norm(exact)), 1e-16))
    slope = np.polyfit(np.log10(tols), np.log10(errs), 1)[0]
    assert 0.7 <= slope <= 1.2, (slope, errs)
    assert all(e <= 10 * t for e, t in zip(errs, tols)), errs


@pytest.mark.gpu
def test_timings_reported(esn):
    """exec_type1/2 return the reference's stage keys with device seconds."""
    rng = np.random.default_rng(9)
    x = [rng.uniform(-np.pi, np.pi, 2000) for _ in range(2)]
    c = rng.standard_normal(2000) + 1j * rng.standard_normal(2000)
    _, t1 = esn.exec_type1(x, c, (32, 24), esn.TransformOptions(tolerance=1e-6))
    f = rng.standard_normal((24, 32)) + 1j * rng.standard_normal((24, 32))
    _, t2 = esn.exec_type2(x, f, esn.TransformOptions(tolerance=1e-6))
    for t in (t1, t2):
        assert set(t) == {"sort", "spread", "fft", "correct"}
        assert all(v >= 0.0 for v in t.values()) and t["spread"] > 0.0


@pytest.mark.gpu
def test_type2_worst_case_bounded_by_l1_norm(esn, oracle):
    """Reference test_transforms.py type2_worst_case_bounded_by_l1_norm: the
    aliasing probe (type 1 of every unit strength against the exact sum,
    oracle.py aliasing_probe -- here one batched call with the identity as
    strengths) bounds the type-2 error for any modes: max |c~ - c| <=
    2 max|E| ||f||_1 (linearity; the type-2 map is the transpose)."""
    from paper_1808_06736_b200.kernel import params_for_width
    rng = np.random.default_rng(7)
    m, n = 32, 32
    x = rng.uniform(-np.pi, np.pi, m)
    p = params_for_width(7, 2.0)
    o = esn.TransformOptions(params=p)
    unit = np.eye(m, dtype=np.complex128)
    fast1, _ = esn.exec_type1((x,), unit, (n,), o)
    exact1 = np.stack([oracle.direct_type1([x], unit[j], (n,)) for j in range(m)])
    eps = float(np.abs(fast1 - exact1).max())
    f = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    fast2, _ = esn.exec_type2((x,), f, o)
    exact2 = oracle.direct_type2([x], f)
    assert np.abs(fast2 - exact2).max() <= 2.0 * eps * np.abs(f).sum()
