"""Pins the CPU oracle (oracle/esn_oracle.*) to the REAL reference: every
golden vector in tests/golden/ref_*.npz was produced by running esnufft
itself (tests/golden/make_golden.py).  The oracle is bit-identical on all
of them (same operation order, no FMA contraction, same pocketfft)."""

import numpy as np
import pytest

import cases
from cases import FSERIES_CASES, SPREAD_CASES, XFORM_CASES


def test_params_and_sizes(oracle, golden):
    k = golden("kernel")
    for tol, sigma, w, beta, gamma, pq in k["params"]:
        p = oracle.select_params(tol, sigma)
        assert (p.w, p.beta, p.gamma, p.p_quad) == (w, beta, gamma, pq)
    for n, s in zip(k["smooth_in"], k["smooth"]):
        assert oracle.next_smooth(int(n)) == s
    for row in k["fine_sizes"]:
        nm = tuple(int(v) for v in row[:3] if v > 0)
        sigma, w = row[3], int(row[4])
        assert oracle.fine_grid_sizes(nm, sigma, w) == tuple(int(v) for v in row[5:5 + len(nm)])


def test_quadrature_corrections_poly(oracle, golden):
    k = golden("kernel")
    for n in (1, 2, 3, 5, 8, 16, 26, 37, 64):
        x, w = oracle.gauss_legendre(n)
        np.testing.assert_array_equal(x, k[f"gl_x_{n}"])
        np.testing.assert_array_equal(w, k[f"gl_w_{n}"])
    for i, (w, sigma, n, N) in enumerate(FSERIES_CASES):
        np.testing.assert_array_equal(oracle.fseries_correction(oracle.params_for_width(w, sigma), n, N),
                                      k[f"fs_{i}"])
    for w in range(2, 17):
        p = oracle.params_for_width(w)
        np.testing.assert_array_equal(oracle.piecewise_poly(p.w, p.beta), k[f"poly_{w}"])
    np.testing.assert_allclose(oracle.kernel_ft(oracle.params_for_width(9), 0.05, k["kft_k"]),
                               k["kft"], rtol=1e-14)


def test_fold_base_and_sort(oracle, golden):
    g = golden("grid")
    xs = g["fold_x"]
    for n in (20, 256, 2000, 20000, 1):
        gg, bad, oob = oracle.grid_coords(xs, n)
        np.testing.assert_array_equal(gg, g[f"g_{n}"])
        assert bad == -1 and oob >= 0
        for w in (2, 5, 6, 7, 10, 16):
            np.testing.assert_array_equal(oracle.base_indices(gg, w), g[f"base_{n}_{w}"])
    specs = [((64,), 1000, 1), ((100,), 5000, 2), ((128, 64), 20000, 3), ((50, 37), 3000, 4),
             ((64, 32, 32), 5000, 5), ((30, 22, 17), 4000, 6), ((64,), 100, 7)]
    for i, (sizes, m, seed) in enumerate(specs):
        r = np.random.default_rng(seed)
        coords = tuple(r.uniform(0, s, m) for s in sizes)
        if i == 6:
            coords = (np.full(m, 2.5),)
        perm, boxes = oracle.bin_sort(coords, sizes)
        np.testing.assert_array_equal(perm, g[f"bs_perm_{i}"])
        np.testing.assert_array_equal(boxes, g[f"bs_boxes_{i}"])


@pytest.mark.parametrize("i", range(len(SPREAD_CASES)))
def test_spread_interp_bitwise(oracle, golden, i):
    s = golden("spread")
    dim, sizes, m, w, exact, seed = SPREAD_CASES[i]
    r = np.random.default_rng(seed)
    coords = [r.uniform(-np.pi, np.pi, m) for _ in range(dim)]
    c = r.standard_normal(m) + 1j * r.standard_normal(m)
    b = r.standard_normal(tuple(reversed(sizes))) + 1j * r.standard_normal(tuple(reversed(sizes)))
    p = oracle.params_for_width(w)
    gs = [oracle.grid_coords(x, n)[0] for x, n in zip(coords, sizes)]
    perm, _ = oracle.bin_sort(gs, sizes)
    np.testing.assert_array_equal(oracle.spread(gs, perm, c, sizes, p, exact, threads=4), s[f"sp_grid_{i}"])
    np.testing.assert_array_equal(oracle.interp(gs, perm, b, sizes, p, exact, threads=4), s[f"sp_interp_{i}"])


@pytest.mark.parametrize("i", range(len(XFORM_CASES)))
def test_transforms_bitwise(oracle, golden, i):
    t = golden("transforms")
    tt, dim, nm, m, tol, isign, sigma, exact, seed = XFORM_CASES[i]
    r = np.random.default_rng(seed)
    coords = [r.uniform(-np.pi, np.pi, m) for _ in range(dim)]
    if tt == 1:
        c = r.standard_normal(m) + 1j * r.standard_normal(m)
        out = oracle.exec_type1(coords, c, nm, tol, isign, sigma, use_exact=exact)
    elif tt == 2:
        f = r.standard_normal(tuple(reversed(nm))) + 1j * r.standard_normal(tuple(reversed(nm)))
        out = oracle.exec_type2(coords, f, tol, isign, sigma, use_exact=exact)
    else:
        c = r.standard_normal(m) + 1j * r.standard_normal(m)
        targets = [r.uniform(-30, 30, 180) for _ in range(dim)]
        out = oracle.exec_type3(coords, c, targets, tol, isign, sigma, use_exact=exact)
    np.testing.assert_array_equal(out, t[f"x_{i}"])


@pytest.mark.parametrize("name", ["c1", "c5"])
def test_north_star_small_configs(oracle, golden, name):
    g = golden("northstar")
    cfg = cases.CONFIGS[name]
    T = cfg.get("ntransf_golden", 1)
    coords, data, cfg = cases.make_inputs(name, M=cfg["M_golden"], ntransf=T)
    cs = data if T > 1 else data[None]
    out = np.stack([oracle.exec_type1(coords, c, cfg["nm"], cfg["tol"], cfg["isign"]) for c in cs])
    flat = out.reshape(T, -1)
    if f"{name}_full" in g.files:
        np.testing.assert_allclose(flat, g[f"{name}_full"].reshape(T, -1), rtol=0, atol=1e-9)
    else:
        np.testing.assert_allclose(flat[:, g[f"{name}_idx"]], g[f"{name}_sample"], rtol=1e-12, atol=1e-9)


def test_direct_sums_closed_forms(oracle):
    # oracle.py:101-151 closed forms: point at the origin -> all-ones modes
    f = oracle.direct_type1([np.array([0.0])], np.array([1.0 + 0j]), (8,))
    np.testing.assert_allclose(f, np.ones(8), atol=1e-15)
    x = np.random.default_rng(0).uniform(-np.pi, np.pi, 25)
    modes = np.zeros(9, complex)
    modes[4] = 1.0
    np.testing.assert_allclose(oracle.direct_type2([x], modes), np.ones(25), atol=1e-15)


@pytest.mark.parametrize("tt", (1, 2, 3))
@pytest.mark.parametrize("dim", (1, 2, 3))
def test_binding_fixtures_bitwise(oracle, golden, tt, dim):
    """The esnufftpy binding fixtures (reference make_fixtures.py recipe,
    regenerated from the reference core by make_golden.gen_bindings)."""
    b = cases.binding_case(tt, dim)
    if tt == 1:
        out = oracle.exec_type1(b["coords"], b["c"], b["nm"], b["tol"], b["isign"])
    elif tt == 2:
        out = oracle.exec_type2(b["coords"], b["f"], b["tol"], b["isign"])
    else:
        out = oracle.exec_type3(b["coords"], b["c"], b["targets"], b["tol"], b["isign"])
    np.testing.assert_array_equal(out, golden("bindings")[f"t{tt}d{dim}"])
