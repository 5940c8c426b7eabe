"""Seeded input generators shared by the golden-vector script, the parity
tests and bench.py.

Follows the reference's generation idiom (bench.py:117, 215-216 and
BASELINE.md section 3.4): ``rng = np.random.default_rng(seed)``; coordinates
``rng.uniform(lo, hi, M)`` for dims 1..d in order; strengths / modes
``standard_normal + 1j * standard_normal`` (real drawn before imag).  For
complex64 configs the values are drawn in float64 and cast; the CPU side is
fed the cast values upcast back to float64 so both sides see bit-identical
inputs.
"""

from __future__ import annotations

import math

import numpy as np

PI = math.pi

# The BASELINE.json configs.  "M_full" is the north-star size; the golden
# fixtures use "M_golden" so the reference finishes in seconds.
CONFIGS = {
    "c1": dict(ttype=1, dim=1, nm=(10000,), M_full=100_000, M_golden=100_000,
               tol=1e-6, isign=1, dtype="float64", lo=-PI, hi=PI, ntransf=1, seed=1001),
    "c2": dict(ttype=2, dim=2, nm=(1000, 1000), M_full=10_000_000, M_golden=20_000,
               tol=1e-5, isign=-1, dtype="float64", lo=-PI, hi=PI, ntransf=1, seed=1002),
    "c3": dict(ttype=1, dim=3, nm=(128, 128, 128), M_full=10_000_000, M_golden=20_000,
               tol=1e-6, isign=1, dtype="float64", lo=-PI, hi=PI, ntransf=1, seed=1003,
               cdtype="complex64"),
    "c3f": dict(ttype=1, dim=3, nm=(128, 128, 128), M_full=10_000_000, M_golden=20_000,
                tol=1e-4, isign=1, dtype="float32", lo=-PI, hi=PI, ntransf=1, seed=1003,
                cdtype="complex64"),
    "c4": dict(ttype=1, dim=3, nm=(128, 128, 128), M_full=10_000_000, M_golden=20_000,
               tol=1e-9, isign=1, dtype="float64", lo=-PI, hi=-PI + 2 * PI / 8,
               ntransf=1, seed=1004),
    "c5": dict(ttype=1, dim=2, nm=(512, 512), M_full=1_000_000, M_golden=10_000,
               tol=1e-4, isign=1, dtype="float32", lo=-PI, hi=PI, ntransf=64, seed=1005,
               ntransf_golden=3, cdtype="complex64"),
}


DISTRIBUTIONS = ("uniform", "disc-quad", "sph-quad")


def quad_points(dist: str, m: int, dim: int):
    """Clustered quadrature point clouds of the paper's benchmark section:
    the reference's gen_points (esnufft bench.py:100-139) as restated by
    the product's benchrows.gen_points, bit-identical to the reference
    (pinned by tests/test_benchrows.py against ref_bench.npz).  disc-quad
    (2D) / sph-quad (3D); the returned count is close to, not equal to, m."""
    from paper_1808_06736_b200.benchrows import gen_points
    if dist not in ("disc-quad", "sph-quad"):
        raise ValueError(f"unknown distribution {dist!r}")
    if (dist == "disc-quad") != (dim == 2):
        raise ValueError(f"{dist} is {'2D' if dist == 'disc-quad' else '3D'}")
    return list(gen_points(dist, m, dim, 0))


# esnufftpy binding fixtures: the reference's make_fixtures.py recipe
# (bindings/tests/make_fixtures.py:19-60) -- seeds 8800 + 10 type + dim
BIND_M, BIND_K, BIND_TOL = 300, 200, 1e-9
BIND_NM = {1: (50,), 2: (12, 10), 3: (6, 5, 4)}
BIND_ISIGN = {1: 1, 2: -1, 3: 1}


def binding_case(ttype: int, dim: int):
    """Seeded inputs of one binding fixture: dict with coords, isign, tol and
    c / f / targets / n_modes as the (type, dim) needs."""
    rng = np.random.default_rng(8800 + 10 * ttype + dim)
    nm = BIND_NM[dim]
    out = dict(isign=BIND_ISIGN[dim], tol=BIND_TOL, nm=nm)
    out["coords"] = [rng.uniform(-np.pi, np.pi, BIND_M) for _ in range(dim)]
    if ttype == 1:
        out["c"] = rng.standard_normal(BIND_M) + 1j * rng.standard_normal(BIND_M)
    elif ttype == 2:
        n = int(np.prod(nm))
        out["f"] = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).reshape(tuple(reversed(nm)))
    else:
        out["c"] = rng.standard_normal(BIND_M) + 1j * rng.standard_normal(BIND_M)
        out["targets"] = [rng.uniform(-20.0, 20.0, BIND_K) for _ in range(dim)]
    return out


# reference gen_points pins: (dist, m, dim, seed)
BENCH_POINT_CASES = [("rand-uniform", 1000, 2, 3), ("rand-uniform", 500, 3, 9), ("disc-quad", 1000, 2, 0),
                     ("disc-quad", 20000, 2, 5), ("sph-quad", 1000, 3, 0), ("sph-quad", 30000, 3, 1)]
BENCH_POINT_BIG = [("disc-quad", 10_000_000, 2), ("sph-quad", 10_000_000, 3)]


def make_inputs(name: str, M: int | None = None, ntransf: int | None = None, dist: str = "uniform"):
    """Return (coords list float64, data complex128, cfg) for a config.

    data is strengths (ntransf, M) / (M,) for type 1, or the mode array
    (N_d..N_1) for type 2.  For float32 configs coordinates are rounded to
    float32 (then upcast) and complex data to complex64 (then upcast).
    dist != "uniform" replaces the coordinates by a quadrature cloud
    (quad_points; cfg["M_actual"] holds its size)."""
    cfg = dict(CONFIGS[name])
    M = cfg["M_full"] if M is None else M
    T = cfg["ntransf"] if ntransf is None else ntransf
    rng = np.random.default_rng(cfg["seed"])
    coords = [rng.uniform(cfg["lo"], cfg["hi"], M) for _ in range(cfg["dim"])]
    if dist != "uniform":
        coords = quad_points(dist, M, cfg["dim"])
        M = len(coords[0])
    cfg["M_actual"] = M
    cfg["dist"] = dist
    if cfg["ttype"] == 1:
        shape = (T, M) if T > 1 else (M,)
    else:
        shape = tuple(reversed(cfg["nm"]))
        if T > 1:
            shape = (T,) + shape
    data = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    if cfg["dtype"] == "float32":
        coords = [x.astype(np.float32).astype(np.float64) for x in coords]
    cd = cfg.get("cdtype", "complex128")
    if cd == "complex64" or cfg["dtype"] == "float32":
        data = data.astype(np.complex64).astype(np.complex128)
    return coords, data, cfg


def rand_problem(dim: int, m: int, seed: int, lo=-PI, hi=PI):
    """test_transforms.py:23-27 style random problem."""
    rng = np.random.default_rng(seed)
    coords = [rng.uniform(lo, hi, m) for _ in range(dim)]
    c = rng.standard_normal(m) + 1j * rng.standard_normal(m)
    return coords, c


def rand_modes(nm, seed: int):
    rng = np.random.default_rng(seed)
    shape = tuple(reversed(nm))
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def sample_flat(total: int, count: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(total, size=min(count, total), replace=False))


# Special coordinates that exercise the fold edge cases (grid.py:152-168).
EDGE_COORDS = np.array([
    0.0, -0.0, 2 * PI, -2 * PI, PI, -PI, 3 * PI, -3 * PI, 1e-300, -1e-300,
    -1e-17, 2 * PI - 1e-15, np.nextafter(2 * PI, 0.0), np.nextafter(-2 * PI, 0.0),
    1e6, -1e6, 12.345, -12.345, 0.5, np.nextafter(0.0, -1.0), 6.283185307179586,
])


# Golden-vector case tables (make_golden.py runs the reference on these).
TOLS = [1e-1, 9e-2, 3e-2, 1e-2, 1e-3, 2e-4, 1e-4, 1e-5, 1e-6, 1e-7, 1e-8,
        1e-9, 1e-10, 1e-11, 1e-12, 1e-13, 1e-14, 1e-15]
FSERIES_CASES = [  # (w, sigma, n, N)
    (7, 2.0, 20000, 10000), (6, 2.0, 2000, 1000), (7, 2.0, 256, 128),
    (5, 2.0, 256, 128), (10, 2.0, 256, 128), (5, 2.0, 1024, 512),
    (2, 2.0, 4, 1), (16, 2.0, 64, 31), (13, 2.0, 3000, 1499), (11, 1.25, 160, 128),
    (3, 2.0, 6, 3), (8, 2.0, 2500, 2500),
]
SPREAD_CASES = [  # (dim, sizes, M, w, use_exact, seed)
    (1, (48,), 200, 7, False, 1), (1, (600,), 3000, 7, True, 2),
    (1, (20,), 50, 16, False, 3), (1, (8,), 40, 2, False, 4),
    (2, (24, 20), 200, 7, False, 5), (2, (80, 64), 5000, 6, False, 6),
    (2, (36, 30), 700, 13, True, 7), (2, (40, 50), 1500, 5, False, 8),
    (3, (12, 16, 10), 200, 7, False, 9), (3, (32, 24, 20), 4000, 5, False, 10),
    (3, (24, 24, 24), 3000, 10, False, 11), (3, (20, 18, 22), 500, 3, True, 12),
    (3, (40, 40, 40), 25_000, 7, False, 13),
]
XFORM_CASES = [  # (ttype, dim, nm, M, tol, isign, sigma, exact, seed)
    (1, 1, (50,), 300, 1e-9, 1, 2.0, False, 21), (1, 1, (64,), 500, 1e-6, -1, 2.0, False, 22),
    (1, 2, (14, 10), 300, 1e-9, 1, 2.0, False, 23), (1, 2, (32, 24), 1000, 1e-5, -1, 2.0, False, 24),
    (1, 3, (8, 6, 7), 300, 1e-9, -1, 2.0, False, 25), (1, 3, (16, 16, 16), 2000, 1e-4, 1, 2.0, False, 26),
    (1, 2, (18, 12), 250, 1e-7, 1, 1.25, False, 27), (1, 2, (20, 16), 300, 1e-8, 1, 2.0, True, 28),
    (1, 1, (1,), 30, 1e-3, 1, 2.0, False, 29), (1, 3, (9, 5, 4), 150, 1e-12, 1, 2.0, False, 30),
    (2, 1, (40,), 200, 1e-9, 1, 2.0, False, 31), (2, 1, (129,), 800, 1e-6, -1, 2.0, False, 32),
    (2, 2, (12, 9), 200, 1e-9, -1, 2.0, False, 33), (2, 2, (50, 40), 3000, 1e-5, 1, 2.0, False, 34),
    (2, 3, (6, 5, 8), 200, 1e-9, 1, 2.0, False, 35), (2, 3, (16, 12, 10), 1500, 1e-3, -1, 2.0, False, 36),
    (2, 2, (17, 11), 300, 1e-7, -1, 1.25, False, 37), (2, 3, (7, 7, 7), 100, 1e-14, 1, 2.0, False, 38),
    (3, 1, None, 250, 1e-9, 1, 2.0, False, 41), (3, 2, None, 250, 1e-9, -1, 2.0, False, 42),
    (3, 3, None, 250, 1e-6, 1, 2.0, False, 43), (3, 1, None, 400, 1e-4, -1, 2.0, False, 44),
]
