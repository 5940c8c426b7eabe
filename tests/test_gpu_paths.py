"""Cross-checks between the device code paths that must agree.

* fp64 batched transforms (ntransf > 1) against one transform at a time:
  type 2 bit-identical (each output is computed by one thread with the
  same operations, esn_device.cuh k_interp_bulk), type 1 to rounding (the
  global-memory reductions of the row spreader are unordered).
* the pipelined bulk-copy interpolator against the synchronous tile
  interpolator (ESN_INTERP=tile, read once per process -> child process):
  bit-identical outputs.
"""
import os
import subprocess
import sys
import textwrap

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("dim,nm,tol", [(2, (40, 36), 1e-6), (3, (12, 10, 14), 1e-5)])
def test_fp64_batched_matches_single(esn, dim, nm, tol):
    rng = np.random.default_rng(11 + dim)
    m, T = 20_000, 3
    coords = [rng.uniform(-np.pi, np.pi, m) for _ in range(dim)]
    o = esn.TransformOptions(tolerance=tol, isign=-1)
    f = rng.standard_normal((T,) + nm[::-1]) + 1j * rng.standard_normal((T,) + nm[::-1])
    outb, _ = esn.exec_type2(coords, f, o)
    assert outb.shape == (T, m)
    for t in range(T):
        single, _ = esn.exec_type2(coords, f[t], o)
        assert np.array_equal(single, outb[t]), f"type 2 transform {t}"
    c = rng.standard_normal((T, m)) + 1j * rng.standard_normal((T, m))
    fb, _ = esn.exec_type1(coords, c, nm, o)
    assert fb.shape == (T,) + nm[::-1]
    for t in range(T):
        single, _ = esn.exec_type1(coords, c[t], nm, o)
        assert np.linalg.norm(single - fb[t]) <= 1e-13 * np.linalg.norm(single), f"type 1 transform {t}"


SCRIPT = textwrap.dedent(r"""
    import sys, numpy as np
    sys.path.insert(0, sys.argv[1])
    import paper_1808_06736_b200 as nu
    rng = np.random.default_rng(5)
    for dim, nm, M, tol, T, lo, hi in [(2, (64, 50), 40_000, 1e-5, 1, -np.pi, np.pi),
                                       (2, (30, 30), 10_000, 1e-9, 2, -np.pi, np.pi),
                                       (3, (16, 14, 12), 30_000, 1e-6, 1, -np.pi, np.pi),
                                       (1, (300,), 5_000, 1e-7, 1, -np.pi, np.pi),
                                       (2, (100, 80), 60_000, 1e-6, 2, -np.pi, np.pi),
                                       (2, (48, 40), 30_000, 1e-5, 1, -np.pi, -np.pi + 0.2)]:
        xs = [rng.uniform(lo, hi, M) for _ in range(dim)]
        shape = ((T,) if T > 1 else ()) + nm[::-1]
        f = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        c, _ = nu.exec_type2(tuple(xs), f, nu.TransformOptions(tolerance=tol, isign=1))
        np.save(sys.argv[2] + f"/t2_{dim}_{T}_{nm[0]}.npy", c)
""")


def _run(tmp, env_extra):
    env = dict(os.environ)
    env.pop("ESN_INTERP", None)
    env.update(env_extra)
    os.makedirs(tmp, exist_ok=True)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, tmp], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]


@pytest.mark.gpu
def test_bulk_and_tile_interpolators_bit_identical(tmp_path, esn):
    """bulk-copy pipelined kernel vs the synchronous tile kernel over the same
    records: every target computes the same operations, so the outputs are
    bitwise equal (including a clustered 2D cloud, many points per cell)."""
    _run(str(tmp_path / "bulk"), {})
    _run(str(tmp_path / "tile"), {"ESN_INTERP": "tile"})
    names = sorted(os.listdir(tmp_path / "bulk"))
    assert len(names) == 6
    for n in names:
        a = np.load(tmp_path / "bulk" / n)
        b = np.load(tmp_path / "tile" / n)
        assert np.array_equal(a, b), n


@pytest.mark.gpu
@pytest.mark.parametrize("dist,dim,ttype", [("disc-quad", 2, 1), ("disc-quad", 2, 2), ("sph-quad", 3, 1),
                                            ("sph-quad", 3, 2)])
def test_clustered_quadrature_clouds(esn, oracle, dist, dim, ttype):
    """The paper's clustered benchmark clouds (dense near the origin / along
    the axis: a few bins hold most points, so subproblems split and the
    spreaders see their worst-case load) against the oracle."""
    import cases
    coords = cases.quad_points(dist, 20_000 if dim == 2 else 30_000, dim)
    m = len(coords[0])
    rng = np.random.default_rng(17)
    nm = (48, 40) if dim == 2 else (20, 16, 18)
    tol = 1e-6
    o = esn.TransformOptions(tolerance=tol, isign=1)
    if ttype == 1:
        c = rng.standard_normal(m) + 1j * rng.standard_normal(m)
        got, _ = esn.exec_type1(coords, c, nm, o)
        ref = oracle.exec_type1(coords, c, nm, tol=tol, isign=1)
    else:
        f = rng.standard_normal(nm[::-1]) + 1j * rng.standard_normal(nm[::-1])
        got, _ = esn.exec_type2(coords, f, o)
        ref = oracle.exec_type2(coords, f, tol=tol, isign=1)
    assert np.linalg.norm(got - ref) <= 1e-3 * tol * np.linalg.norm(ref)


@pytest.mark.gpu
@pytest.mark.parametrize("dim,nm,T", [(2, (40, 30), 1), (3, (16, 12, 10), 1), (3, (10, 10, 10), 3)])
def test_spread_then_finish_equals_type1(esn, dim, nm, T):
    """spread_type1_grid + finish_type1_grid (the fine-grid-reduce multi-GPU
    variant's two halves, esn_plan_spread + esn_plan_finish_type1) equal the
    one-call type 1; a sum of two shards' grids equals the unsplit result."""
    import torch
    from paper_1808_06736_b200.transforms import finish_type1_grid, spread_type1_grid
    rng = np.random.default_rng(23)
    m = 12_000
    coords = [rng.uniform(-np.pi, np.pi, m) for _ in range(dim)]
    c = rng.standard_normal((T, m) if T > 1 else m) + 1j * rng.standard_normal((T, m) if T > 1 else m)
    o = esn.TransformOptions(tolerance=1e-6, isign=-1)
    ref, _ = esn.exec_type1(coords, c, nm, o)
    g, plan = spread_type1_grid(coords, c, nm, o)
    got = finish_type1_grid(plan, g).cpu().numpy()
    assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)
    h = m // 2
    g1, p1 = spread_type1_grid([x[:h] for x in coords], c[..., :h], nm, o)
    g1 = g1.clone()
    g2, _ = spread_type1_grid([x[h:] for x in coords], c[..., h:], nm, o)
    both = finish_type1_grid(p1, g1 + g2).cpu().numpy()
    assert np.linalg.norm(both - ref) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.gpu
@pytest.mark.parametrize("nm,T,m,clustered", [
    ((13, 9), 3, 4000, False),      # fine grid narrower than one 16 x 16 block: wrapped halo cells
    ((37, 21), 33, 20_000, False),  # partial last blocks in x and y, a partial second transform group
    ((64, 48), 4, 60_000, True),    # clustered: hundreds of points per cell, many pieces per source row
    ((96, 80), 40, 600_000, True),  # clustered, above the graph threshold: the device-side imbalance flag
                                    # hands the spread to the RED-flush kernel (k_zero_if + k_spread_batch2d)
    ((200, 150), 64, 80_000, False),  # two full transform groups, many strips / segments
])
def test_batched_owner_spreader(esn, oracle, nm, T, m, clustered):
    """float32 batched 2D type 1 goes through an owner-computes spreader
    (every fine cell written once by its owner warp: k_spread_b2roll, the
    y-rolling strip kernel, when the fine grid is at least 8 + w - 1 by
    32 + w - 1 cells and w <= 6, else k_spread_b2own -- the (13, 9) case);
    the single transforms go through the row spreader, an independent kernel."""
    rng = np.random.default_rng(11)
    lo, hi = (-np.pi, -np.pi + 0.3) if clustered else (-np.pi, np.pi)
    coords = [rng.uniform(lo, hi, m).astype(np.float32) for _ in range(2)]
    c = (rng.standard_normal((T, m)) + 1j * rng.standard_normal((T, m))).astype(np.complex64)
    o = esn.TransformOptions(tolerance=1e-4, dtype="float32")
    batched, _ = esn.exec_type1(coords, c, nm, o)
    c64 = [x.astype(np.float64) for x in coords]
    for t in sorted({0, T // 2, T - 1}):
        single, _ = esn.exec_type1(coords, c[t], nm, o)
        assert np.linalg.norm(single - batched[t]) <= 2e-5 * np.linalg.norm(single), t
        ref = oracle.exec_type1(c64, c[t].astype(np.complex128), nm, tol=1e-4)
        assert np.linalg.norm(batched[t] - ref) <= 10 * 1e-4 * np.linalg.norm(ref), t


ROLL_SCRIPT = textwrap.dedent(r"""
    import sys, numpy as np
    sys.path.insert(0, sys.argv[1])
    import paper_1808_06736_b200 as nu
    rng = np.random.default_rng(17)
    # uniform (rolled segments), clustered (split bins: second queue), a z size
    # that is not a multiple of the bin depth (wrapped last bin), float32
    for tag, nm, M, tol, lo, hi, dt in [("u", (40, 36, 30), 60_000, 1e-6, -np.pi, np.pi, "float64"),
                                        ("c", (32, 32, 32), 80_000, 1e-6, -np.pi, -np.pi + 0.4, "float64"),
                                        ("w", (20, 18, 13), 20_000, 1e-7, -np.pi, np.pi, "float64"),
                                        ("f", (40, 36, 30), 60_000, 1e-4, -np.pi, np.pi, "float32")]:
        xs = [rng.uniform(lo, hi, M) for _ in range(3)]
        c = rng.standard_normal(M) + 1j * rng.standard_normal(M)
        if dt == "float32":
            xs = [x.astype(np.float32) for x in xs]
            c = c.astype(np.complex64)
        f, _ = nu.exec_type1(tuple(xs), c, nm, nu.TransformOptions(tolerance=tol, dtype=dt))
        np.save(sys.argv[2] + f"/t1_{tag}.npy", f)
""")


@pytest.mark.gpu
def test_3d_z_rolling_matches_plain(tmp_path, esn):
    """The 3D row spreader's z-rolling segments (ESN_ROLL3=1: partial flushes
    of the completed planes, a second queue for split bins) against the
    plain per-subproblem kernel (ESN_ROLL3=0, itself checked against the
    oracle elsewhere): the same result to rounding (the flush order differs)."""
    out = {}
    for mode in ("0", "1"):
        d = tmp_path / f"roll{mode}"
        os.makedirs(d)
        env = dict(os.environ, ESN_ROLL3=mode)
        r = subprocess.run([sys.executable, "-c", ROLL_SCRIPT, ROOT, str(d)], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        out[mode] = {n: np.load(d / n) for n in sorted(os.listdir(d))}
    assert len(out["1"]) == 4
    for n, a in out["1"].items():
        b = out["0"][n]
        bound = 1e-5 if n == "t1_f.npy" else 1e-13
        assert np.linalg.norm(a - b) <= bound * np.linalg.norm(b), n
