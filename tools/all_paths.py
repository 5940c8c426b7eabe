"""Small runs of every kernel path in one process (a smoke test of the
whole dispatch table; compute-sanitizer is not available on the GPU pool):
1D/2D/3D type 1 and 2 (fp64, fp32), batched 2D (owner-computes
spreader), the fused column FFT (n2 = 1024), type 3, a reused plan (graph
replay) and the host routines (plain, transform-group pipeline)."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1808_06736_b200 as nu  # noqa: E402
from paper_1808_06736_b200 import _lib  # noqa: E402
from paper_1808_06736_b200.plan import make_opts  # noqa: E402

rng = np.random.default_rng(1)
m = 3000
for dim, nm in ((1, (64,)), (2, (40, 30)), (3, (20, 16, 12))):
    for dt, tol in (("float64", 1e-6), ("float32", 1e-4)):
        xs = [rng.uniform(-np.pi, np.pi, m) for _ in range(dim)]
        c = rng.standard_normal(m) + 1j * rng.standard_normal(m)
        if dt == "float32":
            xs = [x.astype(np.float32) for x in xs]
            c = c.astype(np.complex64)
        o = nu.TransformOptions(tolerance=tol, dtype=dt)
        nu.exec_type1(xs, c, nm, o)
        f = rng.standard_normal(nm[::-1]) + 1j * rng.standard_normal(nm[::-1])
        nu.exec_type2(xs, f.astype(np.complex64) if dt == "float32" else f, o)
# batched 2D (b2own) and the fused column FFT (N2 = 509 -> n2 = 1024)
xs = [rng.uniform(-np.pi, np.pi, m).astype(np.float32) for _ in range(2)]
cb = (rng.standard_normal((35, m)) + 1j * rng.standard_normal((35, m))).astype(np.complex64)
nu.exec_type1(xs, cb, (24, 509), nu.TransformOptions(tolerance=1e-4, dtype="float32"))
# type 3
s = [rng.uniform(-20, 20, 50) for _ in range(2)]
nu.nufft2d3(*[x.astype(np.float64) for x in xs], cb[0].astype(np.complex128), *s, tolerance=1e-6)
# host routine, transform-group pipeline (T > 32)
import torch  # noqa: E402
hx = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in xs]
hc = torch.from_numpy(np.ascontiguousarray(cb)).pin_memory()
hout = torch.empty((35, 30, 40), dtype=torch.complex64).pin_memory()
opt, keep = make_opts(dtype="float32", timing=False, coord_dtype="float32")
st = _lib.lib.esn_nufft_host(1, 2, m, ctypes.c_void_p(hx[0].data_ptr()), ctypes.c_void_p(hx[1].data_ptr()), None,
                             35, ctypes.c_void_p(hc.data_ptr()), 1, 1e-4, _lib.i64_array((40, 30)),
                             ctypes.c_void_p(hout.data_ptr()), ctypes.byref(opt))
assert st == 0, st
print("all paths ok")
