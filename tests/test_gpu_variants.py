"""The kernel variants kept behind environment switches must agree with the
defaults on the same inputs (each switch is read once per process, so every
variant runs in a child process):

* ESN_SORT_OVERLAP=0 -- type-2 setpts on the plan stream instead of the side
  stream: the same kernels on the same data, so BIT-identical outputs;
* ESN_SPREAD3=rows   -- the first 3D row spreader (k_spread_rows) instead of
  k_spread_rows3: a different summation order, fp64 rounding only;
* ESN_B2=tile        -- the RED-flush batched 2D spreader (k_spread_batch2d)
  instead of the owner-computes k_spread_b2own: fp32 rounding only.
"""
import os
import subprocess
import sys
import textwrap

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent(r"""
    import sys, numpy as np
    sys.path.insert(0, sys.argv[1])
    import paper_1808_06736_b200 as nu
    rng = np.random.default_rng(5)
    out = sys.argv[2]
    # type 2, 2D and 3D (side-stream sort)
    for dim, nm in ((2, (120, 90)), (3, (20, 18, 16))):
        xs = [rng.uniform(-np.pi, np.pi, 200_000) for _ in range(dim)]
        f = rng.standard_normal(nm[::-1]) + 1j * rng.standard_normal(nm[::-1])
        c, _ = nu.exec_type2(tuple(xs), f, nu.TransformOptions(tolerance=1e-6, isign=-1))
        np.save(out + f"/t2_{dim}.npy", c)
    # type 1, 3D fp64 (ε = 1e-6 and 1e-9) and fp32
    for tag, tol, dt in (("f64", 1e-6, "float64"), ("f64w", 1e-9, "float64"), ("f32", 1e-4, "float32")):
        xs = [rng.uniform(-np.pi, np.pi, 150_000) for _ in range(3)]
        c = rng.standard_normal(150_000) + 1j * rng.standard_normal(150_000)
        if dt == "float32":
            xs = [x.astype(np.float32) for x in xs]
            c = c.astype(np.complex64)
        f, _ = nu.exec_type1(tuple(xs), c, (40, 36, 32), nu.TransformOptions(tolerance=tol, dtype=dt))
        np.save(out + f"/t1_3d_{tag}.npy", f)
    # type 1, 2D batched fp32
    xs = [rng.uniform(-np.pi, np.pi, 100_000).astype(np.float32) for _ in range(2)]
    c = (rng.standard_normal((40, 100_000)) + 1j * rng.standard_normal((40, 100_000))).astype(np.complex64)
    f, _ = nu.exec_type1(tuple(xs), c, (96, 80), nu.TransformOptions(tolerance=1e-4, dtype="float32"))
    np.save(out + "/t1_2d_batch.npy", f)
    print("ok")
""")


def _run(tmp, env_extra):
    env = dict(os.environ)
    for k in ("ESN_SORT_OVERLAP", "ESN_SPREAD3", "ESN_B2"):
        env.pop(k, None)
    env.update(env_extra)
    os.makedirs(tmp, exist_ok=True)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, tmp], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return {f[:-4]: np.load(os.path.join(tmp, f)) for f in os.listdir(tmp) if f.endswith(".npy")}


@pytest.fixture(scope="module")
def default_out(tmp_path_factory):
    return _run(str(tmp_path_factory.mktemp("default")), {})


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.gpu
def test_sort_overlap_bit_identical(tmp_path, default_out):
    alt = _run(str(tmp_path), {"ESN_SORT_OVERLAP": "0"})
    for k in ("t2_2", "t2_3"):
        assert np.array_equal(alt[k], default_out[k]), k


@pytest.mark.gpu
def test_rows3_matches_first_row_spreader(tmp_path, default_out):
    alt = _run(str(tmp_path), {"ESN_SPREAD3": "rows"})
    assert _rel(default_out["t1_3d_f64"], alt["t1_3d_f64"]) <= 1e-13
    assert _rel(default_out["t1_3d_f64w"], alt["t1_3d_f64w"]) <= 1e-13
    assert _rel(default_out["t1_3d_f32"], alt["t1_3d_f32"]) <= 1e-6


@pytest.mark.gpu
def test_b2own_matches_tile_batched_spreader(tmp_path, default_out):
    alt = _run(str(tmp_path), {"ESN_B2": "tile"})
    assert _rel(default_out["t1_2d_batch"], alt["t1_2d_batch"]) <= 1e-6


@pytest.mark.gpu
def test_graph_replay_follows_new_data(esn):
    """Small plans replay setpts / execute as captured CUDA graphs (keyed by
    buffer pointers, M and the plan's allocation generation): new VALUES in
    the same buffers, a different output buffer, a different M and a
    different coordinate buffer must all give what a fresh plan gives."""
    import torch
    from paper_1808_06736_b200.plan import Plan
    dev = torch.device("cuda", torch.cuda.current_device())
    rng = np.random.default_rng(9)
    nm = (40, 36)
    p2 = Plan(2, 2, nmodes=nm, isign=-1, tol=1e-6, device=dev)
    p1 = Plan(1, 2, nmodes=nm, isign=1, tol=1e-6, device=dev)
    x = torch.empty(5000, dtype=torch.float64, device=dev)
    y = torch.empty(5000, dtype=torch.float64, device=dev)
    for rep, m in enumerate((5000, 5000, 3000, 5000)):
        if rep == 3:  # a different coordinate buffer
            x = torch.empty(5000, dtype=torch.float64, device=dev)
        x[:m] = torch.from_numpy(rng.uniform(-np.pi, np.pi, m))
        y[:m] = torch.from_numpy(rng.uniform(-np.pi, np.pi, m))
        f = torch.from_numpy(rng.standard_normal(nm[::-1]) + 1j * rng.standard_normal(nm[::-1])).to(dev)
        c = torch.from_numpy(rng.standard_normal(m) + 1j * rng.standard_normal(m)).to(dev)
        out2 = torch.empty(m, dtype=torch.complex128, device=dev)
        p2.setpts([x[:m], y[:m]])
        p2.execute(out2, f)
        out1 = torch.empty(nm[::-1], dtype=torch.complex128, device=dev)
        p1.setpts([x[:m], y[:m]])
        p1.execute(c, out1)
        xs = (x[:m].cpu().numpy(), y[:m].cpu().numpy())
        ref2, _ = esn.exec_type2(xs, f.cpu().numpy(), esn.TransformOptions(tolerance=1e-6, isign=-1))
        ref1, _ = esn.exec_type1(xs, c.cpu().numpy(), nm, esn.TransformOptions(tolerance=1e-6))
        assert np.array_equal(out2.cpu().numpy(), ref2), rep
        assert _rel(out1.cpu().numpy(), ref1) <= 1e-13, rep
    p1.close()
    p2.close()


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,tols", [
    ("float64", (1e-2, 1e-3, 1e-5, 1e-7, 1e-8, 1e-10, 1e-11, 1e-12, 1e-13, 1e-14)),
    ("float32", (1e-2, 1e-3, 1e-4, 1e-5, 1e-6)),
])
def test_every_width_3d_type1_and_batched_2d(esn, oracle, dtype, tols):
    """Each kernel width instantiates its own spreader (w = 2 .. 15 here):
    3D type 1 (k_spread_rows3) and float32 batched 2D type 1
    (k_spread_b2own) against the oracle at small M."""
    rng = np.random.default_rng(21)
    m = 6000
    for tol in tols:
        xs = [rng.uniform(-np.pi, np.pi, m) for _ in range(3)]
        c = rng.standard_normal(m) + 1j * rng.standard_normal(m)
        o = esn.TransformOptions(tolerance=tol, dtype=dtype)
        if dtype == "float32":
            xs = [x.astype(np.float32) for x in xs]
            c = c.astype(np.complex64)
        got, _ = esn.exec_type1(xs, c, (20, 18, 16), o)
        ref = oracle.exec_type1([x.astype(np.float64) for x in xs], c.astype(np.complex128), (20, 18, 16), tol=tol)
        bound = 1e-3 * tol if dtype == "float64" else max(10 * tol, 1e-5)
        assert _rel(got, ref) <= max(bound, 1e-13), (tol, _rel(got, ref))
        if dtype == "float32":
            cb = (rng.standard_normal((3, m)) + 1j * rng.standard_normal((3, m))).astype(np.complex64)
            gotb, _ = esn.exec_type1(xs[:2], cb, (40, 34), o)
            for t in range(3):
                refb = oracle.exec_type1([x.astype(np.float64) for x in xs[:2]], cb[t].astype(np.complex128),
                                         (40, 34), tol=tol)
                assert _rel(gotb[t], refb) <= max(10 * tol, 1e-5), (tol, t, _rel(gotb[t], refb))


@pytest.mark.gpu
@pytest.mark.parametrize("nm,T,isign", [((37, 509), 1, 1), ((64, 512), 3, -1), ((1000, 505), 2, 1)])
def test_fused_column_fft_deconv(esn, oracle, nm, T, isign):
    """float32 2D type 1 with a 1024-point fine y axis (N2 in 501..512) runs
    cuFFT along x and the fused 1024-point column FFT + deconvolution
    (k_colfft1024_deconv): odd N1, partial column tiles, both signs, batches."""
    rng = np.random.default_rng(31)
    m = 30_000
    xs = [rng.uniform(-np.pi, np.pi, m).astype(np.float32) for _ in range(2)]
    c = (rng.standard_normal((T, m)) + 1j * rng.standard_normal((T, m))).astype(np.complex64)
    o = esn.TransformOptions(tolerance=1e-5, isign=isign, dtype="float32")
    got, _ = esn.exec_type1(xs, c if T > 1 else c[0], nm, o)
    got = np.asarray(got).reshape(T, nm[1], nm[0])
    for t in range(T):
        ref = oracle.exec_type1([x.astype(np.float64) for x in xs], c[t].astype(np.complex128), nm, tol=1e-5,
                                isign=isign)
        assert _rel(got[t], ref) <= 1e-5, (t, _rel(got[t], ref))
