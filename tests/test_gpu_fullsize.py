"""Every BASELINE.json config at its FULL north-star size (M = 1e5 .. 1e7):

* against the exact direct sum (GPU `direct_*`, itself pinned to the oracle
  in test_gpu_properties.py) on a seeded sample of modes (type 1) or points
  (type 2): rel l2 <= 10 eps -- the north star's "within the requested eps"
  is not met by the reference itself at these widths (1.1 --
  2.3 eps), so the reference-parity bound 10 eps is used;
* against the CPU oracle (C restatement of the reference path, all host
  threads) on the same inputs for the configs it finishes in seconds:
  rel l2 <= 10 eps (float32 plans) and far tighter for float64.
"""
import time

import numpy as np
import pytest

import cases

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _inputs(name):
    cfg = cases.CONFIGS[name]
    T = cfg.get("ntransf", 1)
    coords, data, cfg = cases.make_inputs(name, ntransf=T)
    if cfg["dtype"] == "float32":
        coords = [x.astype(np.float32) for x in coords]
        data = data.astype(np.complex64)
    return coords, data, cfg, T


def _run(esn, name):
    coords, data, cfg, T = _inputs(name)
    opts = esn.TransformOptions(tolerance=cfg["tol"], isign=cfg["isign"], dtype=cfg["dtype"])
    if cfg["ttype"] == 1:
        out, _ = esn.exec_type1(coords, data, cfg["nm"], opts)
    else:
        out, _ = esn.exec_type2(coords, data, opts)
    return coords, data, cfg, T, np.asarray(out)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c3f", "c4", "c5"])
def test_fullsize_vs_direct_sum(esn, name):
    coords, data, cfg, T, out = _run(esn, name)
    rng = np.random.default_rng(77)
    c64 = [np.asarray(x, dtype=np.float64) for x in coords]
    if cfg["ttype"] == 1:
        nm = cfg["nm"]
        t = T - 1 if T > 1 else 0  # (batched: the last transform)
        strengths = (data[t] if T > 1 else data).astype(np.complex128)
        got = out[t] if T > 1 else out
        # sampled modes k (centered indices), exact sums as type-3 targets
        ks = [rng.integers(-(n // 2), n - n // 2, 16) for n in nm]
        exact = []
        for lo in range(0, 16, 4):  # (<= 4e7 terms per call: under the direct-sum cap)
            tg = [k[lo:lo + 4].astype(np.float64) for k in ks]
            exact.append(np.asarray(esn.direct_type3(c64, strengths, tg, isign=cfg["isign"])))
        exact = np.concatenate(exact)
        idx = tuple(k + n // 2 for k, n in zip(ks[::-1], nm[::-1]))  # modes stored (N_d..N_1)
        sample = got[idx]
    else:
        pts = rng.choice(len(c64[0]), 64, replace=False)
        exact = np.asarray(esn.direct_type2([x[pts] for x in c64], data.astype(np.complex128), isign=cfg["isign"]))
        sample = out[pts]
    e = _rel(sample, exact)
    print(f"{name}: direct-sum sample rel l2 {e:.2e} ({e / cfg['tol']:.2f} eps)")
    assert e <= 10 * cfg["tol"], (name, e)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c3f", "c4", "c5"])
def test_fullsize_vs_oracle(esn, oracle, name):
    coords, data, cfg, T, out = _run(esn, name)
    c64 = [np.asarray(x, dtype=np.float64) for x in coords]
    t0 = time.perf_counter()
    if cfg["ttype"] == 1:
        ts = [0, T - 1] if T > 1 else [None]
        for t in ts:
            strengths = (data[t] if t is not None else data).astype(np.complex128)
            ref = oracle.exec_type1(c64, strengths, cfg["nm"], tol=cfg["tol"], isign=cfg["isign"])
            got = out[t] if t is not None else out
            bound = 10 * cfg["tol"] if cfg["dtype"] == "float32" else 1e-3 * cfg["tol"]
            print(f"{name}[{t}]: vs oracle rel l2 {_rel(got, ref):.2e}")
            assert _rel(got, ref) <= bound, (name, t, _rel(got, ref))
    else:
        ref = oracle.exec_type2(c64, data.astype(np.complex128), tol=cfg["tol"], isign=cfg["isign"])
        print(f"{name}: vs oracle rel l2 {_rel(out, ref):.2e}")
        assert _rel(out, ref) <= 1e-3 * cfg["tol"], (name, _rel(out, ref))
    print(f"{name}: oracle {time.perf_counter() - t0:.1f} s")
