"""Type 3 measured like the BASELINE configs: 2D, M = 1e6
sources iid uniform on [-pi, pi)^2, K = 1e6 targets iid uniform on
[-500, 500)^2 (the inner type-2 grid is c2-sized), complex128 N(0,1)
strengths, eps = 1e-6, float64; seeded.  Our exec_type3 on device-resident
tensors (CUDA events, W warm-up, K timed calls, synchronised) beside the CPU
oracle (C + OpenMP restatement of transforms.py:267-351, all host threads) on
a bounded sample; the two agree on a small case first.
usage: python tools/bench_type3.py [steps]"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_1808_06736_b200 as nu  # noqa: E402
import esn_oracle as O  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
M = K = 1_000_000
tol = 1e-6
rng = np.random.default_rng(1301)
xs = [rng.uniform(-np.pi, np.pi, M) for _ in range(2)]
ss = [rng.uniform(-500, 500, K) for _ in range(2)]
c = rng.standard_normal(M) + 1j * rng.standard_normal(M)
o = nu.TransformOptions(tolerance=tol)
O.build()

# parity on a small case
m = 20_000
got, _ = nu.exec_type3([x[:m] for x in xs], c[:m], [s[:m] for s in ss], o)
ref = O.exec_type3([x[:m] for x in xs], c[:m], [s[:m] for s in ss], tol=tol)
rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))

dev = torch.device("cuda", 0)
dx = [torch.from_numpy(x).to(dev) for x in xs]
ds = [torch.from_numpy(s).to(dev) for s in ss]
dc = torch.from_numpy(c).to(dev)
for _ in range(3):
    nu.exec_type3(dx, dc, ds, o)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    nu.exec_type3(dx, dc, ds, o)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps

ms_cpu = 0.0
Mc = 200_000
cores = O.num_procs()
O.exec_type3([x[:2000] for x in xs], c[:2000], [s[:2000] for s in ss], tol=tol, threads=cores)
t0 = time.perf_counter()
O.exec_type3([x[:Mc] for x in xs], c[:Mc], [s[:Mc] for s in ss], tol=tol, threads=cores)
ms_cpu = (time.perf_counter() - t0) * 1e3
print(json.dumps({
    "metric": "NU points/sec (type 3, sources + targets)", "unit": "NU points/s",
    "value": (M + K) / (ms * 1e-3), "ms_per_step": ms, "steps": steps, "warmup": 3, "dtype": "f64",
    "config": {"workload": "t3: 2D type-3, M=1e6 sources on [-pi,pi)^2, K=1e6 targets on [-500,500)^2, "
                           "eps=1e-6, isign=+1", "data": "synthetic, seeded"},
    "parity_rel_l2_vs_oracle_m2e4": rel,
    "cpu_baseline": {"value": 2 * Mc / (ms_cpu * 1e-3), "unit": "NU points/s", "cores": cores, "kind": "port",
                     "sample": f"M = K = {Mc:.0e} (oracle C+OpenMP restatement)"},
}))
