"""Bench row schema and clouds (reference esnufft/bench.py).

CPU: the clouds are bit-identical to the reference's gen_points (fixture
ref_bench.npz from make_golden.gen_bench), the tables round-trip exactly
through CSV and JSON lines, spec validation mirrors the reference.  GPU:
run_sweep measures real rows on the device transforms."""

import io
import math

import numpy as np
import pytest

import cases
from paper_1808_06736_b200 import benchrows as B
from paper_1808_06736_b200.errors import SizeError

REF_COLUMNS = ("transform_type", "dim", "dist", "m", "n", "tol", "threads", "reps", "seed", "status",
               "t_total", "t_sort", "t_spread", "t_fft", "t_correct", "rel_err", "err_ref", "pts_per_sec")


@pytest.mark.parametrize("i", range(len(cases.BENCH_POINT_CASES)))
def test_gen_points_bit_identical_to_reference(golden, i):
    g = golden("bench")
    dist, m, dim, seed = cases.BENCH_POINT_CASES[i]
    pts = B.gen_points(dist, m, dim, seed)
    assert len(pts) == dim
    for d, x in enumerate(pts):
        np.testing.assert_array_equal(x, g[f"p{i}_{d}"])


@pytest.mark.parametrize("i", range(len(cases.BENCH_POINT_BIG)))
def test_gen_points_full_size_checksums(golden, i):
    g = golden("bench")
    dist, m, dim = cases.BENCH_POINT_BIG[i]
    pts = B.gen_points(dist, m, dim, 0)
    assert len(pts[0]) == int(g[f"big{i}_n"])
    np.testing.assert_array_equal(np.array([np.sum(x) for x in pts]), g[f"big{i}_sum"])
    np.testing.assert_array_equal(np.array([np.sum(x * x) for x in pts]), g[f"big{i}_sumsq"])
    step = max(1, len(pts[0]) // 4096)
    np.testing.assert_array_equal(np.stack([x[::step] for x in pts]), g[f"big{i}_sample"])


def test_cases_quad_points_are_the_reference_clouds(golden):
    g = golden("bench")
    for i, (dist, m, dim, seed) in enumerate(cases.BENCH_POINT_CASES):
        if dist == "rand-uniform":
            continue
        for d, x in enumerate(cases.quad_points(dist, m, dim)):
            np.testing.assert_array_equal(x, g[f"p{i}_{d}"])


def test_columns_match_reference_order():
    assert B.COLUMNS == REF_COLUMNS
    assert B.SCHEMA == "esnufft-bench-v1"


def _rows():
    spec = B.BenchSpec(transform_type=2, dim=2, dist="disc-quad", m=400, n=64, tolerances=(1e-6, 1e-9))
    return [
        B._row(spec, 1e-6, 1, 400, 64, "ok", 0.1 / 3, {"sort": 1e-3, "spread": math.pi * 1e-3,
                                                       "fft": 2.5e-4, "correct": 1 / 7e4},
               1.234567890123e-7, "direct", 400 / (0.1 / 3)),
        B._row(spec, 1e-9, 4, 400, 64, "error: BadToleranceError: tolerance 1e-20 out of range"),
    ]


@pytest.mark.parametrize("fmt", ("csv", "jsonl"))
def test_tables_round_trip_exactly(fmt):
    rows = _rows()
    buf = io.StringIO()
    B.write_rows(rows, buf, fmt)
    text = buf.getvalue()
    assert "esnufft-bench-v1" in text.splitlines()[0]
    back = B.read_rows(io.StringIO(text), fmt)
    assert back == rows  # dataclass equality: float bits and None cells included


def test_table_errors():
    with pytest.raises(SizeError):
        B.write_rows(_rows(), io.StringIO(), "xml")
    with pytest.raises(SizeError):
        B.read_rows(io.StringIO('{"schema": "other"}\n'), "jsonl")
    with pytest.raises(SizeError):
        B.read_rows(io.StringIO("a,b\n1,2\n"), "csv")


def test_spec_validation():
    for kw in (dict(transform_type=4), dict(dim=0), dict(dist="gauss"), dict(reps=2), dict(m=0)):
        with pytest.raises(SizeError):
            B.BenchSpec(**kw)
    with pytest.raises(SizeError):
        B.gen_points("disc-quad", 100, 3, 0)
    with pytest.raises(SizeError):
        B.gen_points("sph-quad", 100, 2, 0)
    with pytest.raises(SizeError):
        B.gen_points("rand-uniform", 0, 2, 0)
    assert B.mode_counts(1000, 3) == (10, 10, 10)


@pytest.mark.gpu
@pytest.mark.parametrize("tt,dim,dist", [(1, 2, "disc-quad"), (2, 3, "sph-quad"), (3, 1, "rand-uniform"),
                                         (1, 3, "rand-uniform")])
def test_run_sweep_on_gpu(esn, tt, dim, dist):
    spec = B.BenchSpec(transform_type=tt, dim=dim, dist=dist, m=3000, n=1000, tolerances=(1e-4, 1e-8),
                       threads=(1,), reps=3, seed=2)
    rows = B.run_sweep(spec)
    assert len(rows) == 2
    for r in rows:
        assert r.status == "ok", r.status
        assert r.err_ref == "direct"
        assert r.rel_err <= 10 * r.tol
        assert r.t_total > 0 and r.pts_per_sec > 0
        assert set(k for k in ("t_sort", "t_spread", "t_fft", "t_correct") if getattr(r, k) is None) == set()
    bad = B.run_sweep(B.BenchSpec(transform_type=1, dim=1, m=100, n=16, tolerances=(1e-20,)))
    assert bad[0].status.startswith("error: BadToleranceError")
