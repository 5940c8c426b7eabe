"""Pinned host<->device bandwidth on the box: H2D, D2H, and both at once."""
import time
import torch
n = 160 * 2**20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    d1.copy_(h1, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
def tm(f, reps=5):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / reps
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
print("H2D GB/s %.1f" % (n / tm(lambda: d1.copy_(h1, non_blocking=True)) / 1e9))
print("D2H GB/s %.1f" % (n / tm(lambda: h2.copy_(d2, non_blocking=True)) / 1e9))
t = tm(both); print("both: %.2f ms (each %.1f GB/s)" % (t * 1e3, n / t / 1e9))
