"""Device timeline of the bench step of one config (torch profiler / CUPTI):
kernel and memset start, duration and stream over a few back-to-back steps.

python tools/timeline.py c2 [steps] [timing 0|1]  ->  gpurun_out/timeline_<cfg>.txt
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests", "golden"))
import cases  # noqa: E402
from paper_1808_06736_b200.plan import Plan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
timing = bool(int(sys.argv[3])) if len(sys.argv) > 3 else True
dev = torch.device("cuda", 0)
cfg = cases.CONFIGS[name]
M, T = cfg["M_full"], cfg["ntransf"]
coords, data, cfg = cases.make_inputs(name, M=M, ntransf=T)
real = torch.float64 if cfg["dtype"] == "float64" else torch.float32
cplx = torch.complex128 if cfg["dtype"] == "float64" else torch.complex64
xs = [torch.from_numpy(x).to(dev, real).contiguous() for x in coords]
d = torch.from_numpy(np.ascontiguousarray(data)).to(dev, cplx).contiguous()
plan = Plan(cfg["ttype"], cfg["dim"], nmodes=cfg["nm"], isign=cfg["isign"], ntransf=T, tol=cfg["tol"], device=dev,
            dtype=cfg["dtype"], timing=timing)
if cfg["ttype"] == 1:
    out = torch.empty(((T,) if T > 1 else ()) + tuple(reversed(cfg["nm"])), dtype=cplx, device=dev)
    cin, fout = d, out
else:
    out = torch.empty((T, M) if T > 1 else (M,), dtype=cplx, device=dev)
    cin, fout = out, d


only = os.environ.get("TL_ONLY", "")


def step():
    if only != "execute":
        plan.setpts(xs)
    if only != "setpts":
        plan.execute(cin, fout)


if only == "execute":
    plan.setpts(xs)
for _ in range(3):
    step()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
os.makedirs("gpurun_out", exist_ok=True)
with open(f"gpurun_out/timeline_{name}.txt", "w") as f:
    prev_end = 0.0
    for e in ev:
        s = e.time_range.start - t0
        dur = e.time_range.end - e.time_range.start
        f.write(f"{s:10.1f} us  +{dur:8.1f}  gap {s - prev_end:7.1f}  {e.name[:70]}\n")
        prev_end = max(prev_end, s + dur)
    f.write(f"total {prev_end:.1f} us over {steps} steps = {prev_end / steps:.1f} us/step\n")
print(open(f"gpurun_out/timeline_{name}.txt").read()[-6000:])
