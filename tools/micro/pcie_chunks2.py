"""Variants of the chunked H2D/D2H pattern to find what slows the pipeline."""
import time
import torch

MB = 2**20
M = 10_000_000
hx = torch.empty(M, dtype=torch.float64).pin_memory()
hy = torch.empty(M, dtype=torch.float64).pin_memory()
hf = torch.empty(2 * MB, dtype=torch.complex128).pin_memory()  # 32 MB... use 16 MB below
hout = torch.empty(M, dtype=torch.complex128).pin_memory()
dx = torch.empty(M, dtype=torch.float64, device="cuda")
dy = torch.empty(M, dtype=torch.float64, device="cuda")
df = torch.empty(1 * MB, dtype=torch.complex128, device="cuda")
dout = torch.empty(M, dtype=torch.complex128, device="cuda")
up, down = torch.cuda.Stream(), torch.cuda.Stream()
hs = [torch.cuda.Stream() for _ in range(4)]


def tm(f, reps=5):
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


def run(K, modes_first, two, via_hs):
    bounds = [M * k // K for k in range(K + 1)]
    eu = [torch.cuda.Event() for _ in range(K)]
    ec = [torch.cuda.Event() for _ in range(K)]
    def f():
        with torch.cuda.stream(up):
            if modes_first:
                df.copy_(hf[:MB], non_blocking=True)
            for k in range(K):
                lo, hi = bounds[k], bounds[k + 1]
                dx[lo:hi].copy_(hx[lo:hi], non_blocking=True)
                if two:
                    dy[lo:hi].copy_(hy[lo:hi], non_blocking=True)
                eu[k].record(up)
        for k in range(K):
            lo, hi = bounds[k], bounds[k + 1]
            if via_hs:
                s = hs[k % 4]
                s.wait_event(eu[k]); ec[k].record(s)
                down.wait_event(ec[k])
            else:
                down.wait_event(eu[k])
            with torch.cuda.stream(down):
                hout[lo:hi].copy_(dout[lo:hi], non_blocking=True)
    return tm(f)


for K in (8, 12):
    print(f"K={K}: x only {run(K, False, False, False):.3f}  x+y {run(K, False, True, False):.3f}  "
          f"+modes {run(K, True, True, False):.3f}  +hs events {run(K, True, True, True):.3f} ms")
