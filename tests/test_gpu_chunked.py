"""Target-chunked type-2 sort order (esn_plan.cu: set_key_space / setpts).

Large type-2 plans order their points by (chunk of original indices, bin,
sub-cell) so the interpolator's scattered outputs stay L2-resident.  Each
output is still computed by one thread with the same operations, so results
must be BIT-identical to the plain bin order; the adjoint spread of such a
plan goes through the order-agnostic spreader.  The chunk threshold is
forced low through ESN_OUT_CHUNK_MB in a child process (it is read once per
process).
"""
import json
import os
import subprocess
import sys
import textwrap

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent(r"""
    import json, sys, numpy as np, torch
    sys.path.insert(0, sys.argv[1])
    import paper_1808_06736_b200 as nu
    from paper_1808_06736_b200.plan import Plan
    from paper_1808_06736_b200 import spreadinterp as SI
    out = {}
    rng = np.random.default_rng(7)
    cases = [(2, (96, 80), 150_000, 1e-5), (3, (24, 20, 16), 60_000, 1e-6), (1, (500,), 80_000, 1e-6)]
    for dim, nm, M, tol in cases:
        xs = [rng.uniform(-np.pi, np.pi, M) for _ in range(dim)]
        f = rng.standard_normal(nm[::-1]) + 1j * rng.standard_normal(nm[::-1])
        o = nu.TransformOptions(tolerance=tol, isign=-1)
        c, _ = nu.exec_type2(tuple(xs), f, o)
        np.save(sys.argv[2] + f"/t2_{dim}.npy", c)
        # chunk count actually used by a plan of this shape
        p = Plan(2, dim, nmodes=nm, isign=-1, tol=tol)
        p.setpts([torch.as_tensor(x, device="cuda") for x in xs])
        out[f"nchunk_{dim}"] = p.target_chunks()
        # adjoint spread through the same (chunked) plan
        g = torch.zeros(tuple(p.nfine[::-1]), dtype=torch.complex128, device="cuda")
        cc = torch.as_tensor(rng.standard_normal(M) + 1j * rng.standard_normal(M), device="cuda")
        p.spread(cc, g)
        np.save(sys.argv[2] + f"/sp_{dim}.npy", g.cpu().numpy())
        # independent path: a spreader plan (bin-structured spreader)
        pts = SI.NuPointSet(tuple(torch.as_tensor(x, device="cuda") for x in xs), p.nfine)
        ref = SI.spread(pts, cc, p.params)
        np.save(sys.argv[2] + f"/spref_{dim}.npy", ref.cpu().numpy() if hasattr(ref, "cpu") else ref)
        p.close()
    # host-buffer pipelined path (M >= 2 Mi, pinned buffers)
    M = 2_300_000
    x = torch.empty(M, dtype=torch.float64).pin_memory(); x.numpy()[:] = rng.uniform(-np.pi, np.pi, M)
    y = torch.empty(M, dtype=torch.float64).pin_memory(); y.numpy()[:] = rng.uniform(-np.pi, np.pi, M)
    f = torch.empty((64, 72), dtype=torch.complex128).pin_memory()
    f.numpy()[:] = rng.standard_normal((64, 72)) + 1j * rng.standard_normal((64, 72))
    c = torch.empty(M, dtype=torch.complex128).pin_memory()
    st = nu._lib.lib.esn_nufft2d2(M, x.data_ptr(), y.data_ptr(), c.data_ptr(), -1, 1e-5, 72, 64, f.data_ptr(), None)
    out["host_status"] = int(st)
    np.save(sys.argv[2] + "/host.npy", c.numpy())
    print(json.dumps(out))
""")


def _run(tmp, env_extra):
    env = dict(os.environ)
    env.pop("ESN_OUT_CHUNK_MB", None)
    env.update(env_extra)
    os.makedirs(tmp, exist_ok=True)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, tmp], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_chunked_order_bit_identical(tmp_path, esn):
    a = _run(str(tmp_path / "plain"), {"ESN_OUT_CHUNK_MB": "0"})
    b = _run(str(tmp_path / "chunk"), {"ESN_OUT_CHUNK_MB": "0.3"})
    for dim in (1, 2, 3):
        assert a[f"nchunk_{dim}"] == 1
        assert b[f"nchunk_{dim}"] > 1, b
        ca = np.load(tmp_path / "plain" / f"t2_{dim}.npy")
        cb = np.load(tmp_path / "chunk" / f"t2_{dim}.npy")
        assert np.array_equal(ca, cb), f"dim {dim}: max diff {np.abs(ca - cb).max()}"
        ga = np.load(tmp_path / "plain" / f"sp_{dim}.npy")
        gb = np.load(tmp_path / "chunk" / f"sp_{dim}.npy")
        gr = np.load(tmp_path / "plain" / f"spref_{dim}.npy")
        # different spreaders (summation order): fp64 rounding only
        for g in (ga, gb):
            assert np.abs(g - gr).max() <= 1e-12 * max(1.0, np.abs(gr).max()), f"dim {dim}"
    assert a["host_status"] == 0 and b["host_status"] == 0
    ha = np.load(tmp_path / "plain" / "host.npy")
    hb = np.load(tmp_path / "chunk" / "host.npy")
    assert np.array_equal(ha, hb)
