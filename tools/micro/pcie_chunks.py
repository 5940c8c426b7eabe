"""Chunked pinned H2D / D2H rates: sequential, concurrent, and dependent
(D2H of chunk k waits for H2D of chunk k), as the host-buffer pipeline does."""
import time
import torch

MB = 2**20
nin, nout = 176 * MB, 160 * MB
hin = torch.empty(nin, dtype=torch.uint8).pin_memory()
hout = torch.empty(nout, dtype=torch.uint8).pin_memory()
din = torch.empty(nin, dtype=torch.uint8, device="cuda")
dout = torch.empty(nout, dtype=torch.uint8, device="cuda")
up, down = torch.cuda.Stream(), torch.cuda.Stream()


def tm(f, reps=5):
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


def run(K, mode):
    ci, co = nin // K, nout // K
    evs = [torch.cuda.Event() for _ in range(K)]
    def f():
        for k in range(K):
            if mode in ("h2d", "both", "dep"):
                with torch.cuda.stream(up):
                    din[k * ci:(k + 1) * ci].copy_(hin[k * ci:(k + 1) * ci], non_blocking=True)
                    evs[k].record(up)
            if mode in ("d2h", "both", "dep"):
                with torch.cuda.stream(down):
                    if mode == "dep":
                        down.wait_event(evs[k])
                    hout[k * co:(k + 1) * co].copy_(dout[k * co:(k + 1) * co], non_blocking=True)
    return tm(f)


for K in (1, 4, 8, 16, 32):
    print(f"K={K:2d}  h2d {run(K, 'h2d'):.3f} ms  d2h {run(K, 'd2h'):.3f} ms  both {run(K, 'both'):.3f} ms  "
          f"dep {run(K, 'dep'):.3f} ms")
