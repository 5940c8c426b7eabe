"""Generate the golden vectors by running the REAL reference (esnufft from
/root/reference/pkg/src) on seeded inputs.  Run in the build container only:

    python tests/golden/make_golden.py

Outputs ``tests/golden/ref_*.npz``.  Inputs are regenerated from seeds by
``cases.py`` so only outputs (or sampled outputs plus checksums) are stored.
Nothing at test / bench time reads /root/reference.
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
REF_SRC = "/root/reference/pkg/src"
os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "esn_numba_cache"))
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
sys.path.insert(0, REF_SRC)

import cases  # noqa: E402
import esnufft  # noqa: E402
from esnufft import grid as rgrid  # noqa: E402
from esnufft import kernel as rkernel  # noqa: E402
from esnufft import spreadinterp as rsi  # noqa: E402
from esnufft.transforms import (TransformOptions, exec_type1, exec_type2,  # noqa: E402
                                exec_type3)

from cases import FSERIES_CASES, SPREAD_CASES, TOLS, XFORM_CASES  # noqa: E402

SAMPLE = 4096


def gen_params():
    rows = []
    for sigma in (2.0, 1.25):
        for tol in TOLS:
            p = rkernel.select_params(tol, sigma)
            rows.append((tol, sigma, p.w, p.beta, p.gamma, p.p_quad))
    arr = np.array(rows, dtype=np.float64)
    ns = np.arange(1, 3001)
    big = np.array([10**6 + 1, 2**20 + 1, 3**13 + 7, 123456789, 1999999, 4096 * 5 + 1])
    smooth = np.array([rgrid.next_smooth(int(n)) for n in np.concatenate([ns, big])])
    fg = []
    for nm, sigma, w in [((100,), 2.0, 7), ((5,), 2.0, 7), ((128,), 1.25, 7),
                         ((1000, 1000), 2.0, 6), ((128, 128, 128), 2.0, 7),
                         ((128, 128, 128), 2.0, 10), ((512, 512), 2.0, 5),
                         ((10000,), 2.0, 7), ((1, 3, 7), 2.0, 16), ((33, 65, 129), 1.25, 11)]:
        s = rgrid.fine_grid_sizes(nm, sigma, w)
        fg.append(list(nm) + [0] * (3 - len(nm)) + [sigma, w] + list(s) + [0] * (3 - len(s)))
    gl = {}
    for n in (1, 2, 3, 5, 8, 16, 26, 37, 64):
        x, wts = rkernel.gauss_legendre(n)
        gl[f"gl_x_{n}"] = np.asarray(x)
        gl[f"gl_w_{n}"] = np.asarray(wts)
    fs = {}
    for i, (w, sigma, n, N) in enumerate(FSERIES_CASES):
        p = rkernel.params_for_width(w, sigma)
        fs[f"fs_{i}"] = rkernel.fseries_correction(p, n, N)
    polys = {}
    for w in range(2, 17):
        p = rkernel.params_for_width(w, 2.0)
        polys[f"poly_{w}"] = np.asarray(rkernel.build_piecewise_poly(p).coeffs)
    p = rkernel.params_for_width(11, 1.25)
    polys["poly_11_s125"] = np.asarray(rkernel.build_piecewise_poly(p).coeffs)
    kft_p = rkernel.params_for_width(9, 2.0)
    ks = np.linspace(-300.0, 300.0, 257)
    kft = rkernel.kernel_ft(kft_p, 0.05, ks)
    np.savez_compressed(os.path.join(HERE, "ref_kernel.npz"), params=arr, smooth_in=np.concatenate([ns, big]),
                        smooth=smooth, fine_sizes=np.array(fg, dtype=np.float64),
                        fs_cases=np.array(FSERIES_CASES, dtype=np.float64), kft_k=ks, kft=kft,
                        **gl, **fs, **polys)


def gen_grid():
    out = {}
    rng = np.random.default_rng(77)
    xs = np.concatenate([cases.EDGE_COORDS, rng.uniform(-3 * np.pi, 3 * np.pi, 500)])
    out["fold_x"] = xs
    for n in (20, 256, 2000, 20000, 1):
        pts = rsi.build_point_set([xs], (n,))
        out[f"g_{n}"] = pts.grid_coords[0]
        for w in (2, 5, 6, 7, 10, 16):
            out[f"base_{n}_{w}"] = rsi._base_indices(pts, w)[0]
    # bin sort
    for i, (sizes, m, seed) in enumerate([((64,), 1000, 1), ((100,), 5000, 2), ((128, 64), 20000, 3),
                                           ((50, 37), 3000, 4), ((64, 32, 32), 5000, 5),
                                           ((30, 22, 17), 4000, 6), ((64,), 100, 7)]):
        r = np.random.default_rng(seed)
        coords = tuple(r.uniform(0, s, m) for s in sizes)
        if i == 6:
            coords = (np.full(m, 2.5),)
        res = rgrid.bin_sort(coords, sizes)
        out[f"bs_perm_{i}"] = res.perm
        out[f"bs_boxes_{i}"] = res.boxes
    np.savez_compressed(os.path.join(HERE, "ref_grid.npz"), **out)


def gen_spread():
    out = {}
    for i, (dim, sizes, m, w, exact, seed) in enumerate(SPREAD_CASES):
        r = np.random.default_rng(seed)
        coords = [r.uniform(-np.pi, np.pi, m) for _ in range(dim)]
        c = r.standard_normal(m) + 1j * r.standard_normal(m)
        shape = tuple(reversed(sizes))
        b = r.standard_normal(shape) + 1j * r.standard_normal(shape)
        p = rkernel.params_for_width(w, 2.0)
        pts = rsi.ensure_sorted(rsi.build_point_set(coords, sizes))
        out[f"sp_grid_{i}"] = rsi.spread(pts, c, p, threads=1, use_exact=exact)
        out[f"sp_interp_{i}"] = rsi.interp(pts, b, p, threads=1, use_exact=exact)
    np.savez_compressed(os.path.join(HERE, "ref_spread.npz"),
                        cases=np.array([(d, m, w, int(e), s) for d, _, m, w, e, s in SPREAD_CASES]), **out)


def gen_transforms():
    out = {}
    for i, (tt, dim, nm, m, tol, isign, sigma, exact, seed) in enumerate(XFORM_CASES):
        r = np.random.default_rng(seed)
        coords = [r.uniform(-np.pi, np.pi, m) for _ in range(dim)]
        opts = TransformOptions(tolerance=tol, isign=isign, sigma=sigma, use_exact_kernel=exact)
        if tt == 1:
            c = r.standard_normal(m) + 1j * r.standard_normal(m)
            out[f"x_{i}"] = exec_type1(coords, c, nm, opts)[0]
        elif tt == 2:
            shape = tuple(reversed(nm))
            f = r.standard_normal(shape) + 1j * r.standard_normal(shape)
            out[f"x_{i}"] = exec_type2(coords, f, opts)[0]
        else:
            c = r.standard_normal(m) + 1j * r.standard_normal(m)
            targets = [r.uniform(-30, 30, 180) for _ in range(dim)]
            out[f"x_{i}"] = exec_type3(coords, c, targets, opts)[0]
    # edge cases: M = 0 and a single point
    o = TransformOptions(tolerance=1e-6)
    out["empty_t1"] = exec_type1((np.zeros(0), np.zeros(0)), np.zeros(0, complex), (6, 4), o)[0]
    out["empty_t2"] = exec_type2((np.zeros(0),), np.ones(8, complex), o)[0]
    out["origin_t1"] = exec_type1((np.array([0.0]),), np.array([1.0 + 0j]), (8,),
                                  TransformOptions(tolerance=1e-9))[0]
    np.savez_compressed(os.path.join(HERE, "ref_transforms.npz"), **out)


def gen_north_star():
    """The BASELINE configs at golden-size M (full N), run by the reference
    with threads = all cores."""
    out = {}
    th = os.cpu_count()
    for name, cfg in cases.CONFIGS.items():
        T = cfg.get("ntransf_golden", 1)
        coords, data, cfg = cases.make_inputs(name, M=cfg["M_golden"], ntransf=T)
        opts = TransformOptions(tolerance=cfg["tol"], isign=cfg["isign"], threads=th)
        if cfg["ttype"] == 1:
            cs = data if T > 1 else data[None]
            res = np.stack([exec_type1(coords, cc, cfg["nm"], opts)[0] for cc in cs])
        else:
            res = exec_type2(coords, data, opts)[0][None]
        flat = res.reshape(res.shape[0], -1)
        if flat.shape[1] <= 100_000:
            out[f"{name}_full"] = res
        else:
            idx = cases.sample_flat(flat.shape[1], SAMPLE, cfg["seed"] + 7)
            out[f"{name}_idx"] = idx
            out[f"{name}_sample"] = flat[:, idx]
        out[f"{name}_norm"] = np.linalg.norm(flat, axis=1)
        out[f"{name}_sum"] = flat.sum(axis=1)
        print(name, "done", flush=True)
    np.savez_compressed(os.path.join(HERE, "ref_northstar.npz"), **out)


def gen_bindings():
    """The reference binding fixtures (bindings/tests/make_fixtures.py
    recipe, core output at one thread) for the nine esnufftpy routines."""
    out = {}
    for tt in (1, 2, 3):
        for dim in (1, 2, 3):
            b = cases.binding_case(tt, dim)
            opts = TransformOptions(tolerance=b["tol"], isign=b["isign"], threads=1)
            if tt == 1:
                r = exec_type1(b["coords"], b["c"], b["nm"], opts)[0]
            elif tt == 2:
                r = exec_type2(b["coords"], b["f"], opts)[0]
            else:
                r = exec_type3(b["coords"], b["c"], b["targets"], opts)[0]
            out[f"t{tt}d{dim}"] = r
    np.savez_compressed(os.path.join(HERE, "ref_bindings.npz"), **out)


def gen_bench():
    """The reference's benchmark clouds (esnufft.bench.gen_points): small
    cases in full, the north-star-sized quadrature clouds as count + sums."""
    from esnufft.bench import gen_points
    out = {}
    for i, (dist, m, dim, seed) in enumerate(cases.BENCH_POINT_CASES):
        pts = gen_points(dist, m, dim, seed)
        for d, x in enumerate(pts):
            out[f"p{i}_{d}"] = np.asarray(x)
    for i, (dist, m, dim) in enumerate(cases.BENCH_POINT_BIG):
        pts = gen_points(dist, m, dim, 0)
        out[f"big{i}_n"] = np.int64(len(pts[0]))
        out[f"big{i}_sum"] = np.array([np.sum(x) for x in pts])
        out[f"big{i}_sumsq"] = np.array([np.sum(x * x) for x in pts])
        out[f"big{i}_sample"] = np.stack([np.asarray(x)[:: max(1, len(x) // 4096)] for x in pts])
    np.savez_compressed(os.path.join(HERE, "ref_bench.npz"), **out)


if __name__ == "__main__":
    print("reference esnufft", esnufft.__version__)
    gen_params()
    gen_grid()
    gen_spread()
    gen_transforms()
    gen_north_star()
    gen_bindings()
    gen_bench()
    print("ok")
