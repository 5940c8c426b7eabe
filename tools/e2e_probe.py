"""Time the host-buffer C-ABI path (esn_nufft_host) for a config, plus a
copy-only PCIe floor with the same bytes.  usage: python tools/e2e_probe.py c2 [reps]"""
import ctypes, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import numpy as np
import torch
from cases import CONFIGS, make_inputs
from paper_1808_06736_b200 import _lib
from paper_1808_06736_b200.plan import make_opts

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = CONFIGS[name]
coords, data, _ = make_inputs(name, M=cfg["M_full"], ntransf=cfg.get("ntransf", 1))
M, T = cfg["M_full"], cfg.get("ntransf", 1)
cplx = torch.complex128 if cfg["dtype"] == "float64" else torch.complex64
hx = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in coords]
hd = torch.from_numpy(np.ascontiguousarray(data)).to(cplx).pin_memory()
if cfg["ttype"] == 1:
    hout = torch.empty((T,) + tuple(reversed(cfg["nm"])), dtype=cplx).pin_memory()
    cptr, fptr = hd.data_ptr(), hout.data_ptr()
else:
    hout = torch.empty((T, M) if T > 1 else (M,), dtype=cplx).pin_memory()
    cptr, fptr = hout.data_ptr(), hd.data_ptr()
o, keep = make_opts(dtype=cfg["dtype"], timing=False)
nm = _lib.i64_array(cfg["nm"])
xp = [ctypes.c_void_p(x.data_ptr()) for x in hx] + [None] * (3 - len(hx))


def call():
    _lib.check(_lib.lib.esn_nufft_host(cfg["ttype"], cfg["dim"], M, xp[0], xp[1], xp[2], T, ctypes.c_void_p(cptr),
                                       cfg["isign"], cfg["tol"], nm, ctypes.c_void_p(fptr), ctypes.byref(o)))


for _ in range(3):
    call()
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    t0 = time.perf_counter(); call(); ts.append(time.perf_counter() - t0)
print(f"{name} e2e: median {1e3 * np.median(ts):.3f} ms  min {1e3 * min(ts):.3f} ms  "
      f"(streams={os.environ.get('ESN_PIPE_STREAMS', '4')} chunks={os.environ.get('ESN_PIPE_CHUNKS', '16')})")
# copy-only floor: same H2D / D2H bytes, chunked over 4 streams
h2d_src = [x for x in hx] + ([hd] if True else [])
dev_in = [torch.empty_like(x, device="cuda") for x in h2d_src]
dev_out = torch.empty_like(hout, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
K = 16


def copies():
    for k in range(K):
        s = streams[k % 4]
        with torch.cuda.stream(s):
            for src, dst in zip(h2d_src, dev_in):
                n = src.numel(); lo = k * n // K; hi = (k + 1) * n // K
                dst.view(-1)[lo:hi].copy_(src.view(-1)[lo:hi], non_blocking=True)
            n = hout.numel(); lo = k * n // K; hi = (k + 1) * n // K
            hout.view(-1)[lo:hi].copy_(dev_out.view(-1)[lo:hi], non_blocking=True)
    torch.cuda.synchronize()


copies()
ts = []
for _ in range(reps):
    t0 = time.perf_counter(); copies(); ts.append(time.perf_counter() - t0)
nb_in = sum(x.numel() * x.element_size() for x in h2d_src)
nb_out = hout.numel() * hout.element_size()
print(f"copy-only floor: median {1e3 * np.median(ts):.3f} ms for {nb_in / 1e6:.0f} MB in + {nb_out / 1e6:.0f} MB out")
