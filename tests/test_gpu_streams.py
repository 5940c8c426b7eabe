"""Stream topology of the plans under concurrency: two type-2 plans (each
with its sort, count and aux streams) and a type-1 plan on three caller
streams, interleaved setpts / execute calls with new points every round and
sizes above the CUDA-graph threshold (so the side streams are used).  Every
result must equal the one a fresh plan computes alone on the default stream
(type 2: bit-identical, the interpolation is deterministic; type 1: up to the
order of the atomic adds)."""

import numpy as np
import pytest


@pytest.mark.gpu
def test_interleaved_plans_on_three_streams(esn):
    import torch
    from paper_1808_06736_b200.plan import Plan
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(77)
    nm2, nm1 = (96, 80), (40, 36, 32)
    streams = [torch.cuda.Stream(dev) for _ in range(3)]
    plans = []
    for k, s in enumerate(streams):
        with torch.cuda.stream(s):
            plans.append(Plan(2, 2, nmodes=nm2, isign=-1, tol=1e-7, device=dev) if k < 2 else
                         Plan(1, 3, nmodes=nm1, tol=1e-6, device=dev))
    rounds, outs, inputs = 4, [], []
    torch.cuda.synchronize(dev)
    for it in range(rounds):
        for k, (s, p) in enumerate(zip(streams, plans)):
            M = 560000 + 30000 * it + 7000 * k  # > 2^19: no graph replay, side streams in use
            d = 2 if k < 2 else 3
            xs = [torch.from_numpy(rng.uniform(-np.pi, np.pi, M)).to(dev) for _ in range(d)]
            if k < 2:
                f = torch.from_numpy(rng.standard_normal(tuple(reversed(nm2))) +
                                     1j * rng.standard_normal(tuple(reversed(nm2)))).to(dev)
                out = torch.empty(M, dtype=torch.complex128, device=dev)
            else:
                f = torch.from_numpy(rng.standard_normal(M) + 1j * rng.standard_normal(M)).to(dev)
                out = torch.empty(tuple(reversed(nm1)), dtype=torch.complex128, device=dev)
            torch.cuda.current_stream(dev).synchronize()  # inputs ready before the side streams read them
            with torch.cuda.stream(s):
                p.setpts(xs)
                if k < 2:
                    p.execute(out, f)
                else:
                    p.execute(f, out)
            inputs.append((k, xs, f))
            outs.append(out)
    for p in plans:
        p.check()
    torch.cuda.synchronize(dev)
    ref2 = Plan(2, 2, nmodes=nm2, isign=-1, tol=1e-7, device=dev)
    ref1 = Plan(1, 3, nmodes=nm1, tol=1e-6, device=dev)
    for (k, xs, f), out in zip(inputs, outs):
        if k < 2:
            want = torch.empty_like(out)
            ref2.setpts(xs)
            ref2.execute(want, f)
            ref2.check()
            assert torch.equal(out, want)
        else:
            want = torch.empty_like(out)
            ref1.setpts(xs)
            ref1.execute(f, want)
            ref1.check()
            assert torch.linalg.norm(out - want) <= 1e-13 * torch.linalg.norm(want)
