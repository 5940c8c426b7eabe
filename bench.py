"""bench.py -- NU points/sec of the full type-1/2 transform on B200.

python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                [--config c2] [--no-e2e] [--no-cpu]

Workload (BASELINE.json configs[1], the metric's config at N = 1):
  c2: 2D type 2, modes 1000x1000 complex128 N(0,1), M = 1e7 targets iid
      uniform on [-pi, pi)^2, eps = 1e-5, isign = -1, float64.
Other configs (--config c1/c3/c3f/c4/c5) exist for parity-shape timing.

A "step" is one full transform (setpts sort + amplify/spread + cuFFT +
interp/deconv) over one batch of synthetic seeded input already resident in
HBM.  `--gpus N` with N > 1 re-launches itself under torch.distributed.run
(N ranks, NCCL, 127.0.0.1) unless already under torchrun; it exits 2 when
fewer than N GPUs are visible or WORLD_SIZE != N.  At N > 1 every rank runs
its own independent shard of c2 (weak scaling, no data-path collective:
type-2 targets are independent outputs), and the line carries
`sharded_configs`: c3 with its points split across the ranks and the
fine grids NCCL-reduced to rank 0 (north_star; plus the mode-array reduce
variant) and c5 with its 64 transforms split (strong scaling).  Times are
CUDA events on the launching stream, max over ranks.  e2e = the same metric
end to end with pinned HOST buffers, H2D + D2H inside the timed region:
through the C ABI one-shot routine (esn_nufft_host) for replicas, through
the package's distributed API for the sharded paths.  --impl reference
times the CPU restatement of the reference (oracle/, "port") with all host
threads on the same config.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import cases  # noqa: E402

METRIC = "NU points/sec (spread+interp, full type-1/2) at 1/2/4/8 B200; % HBM roofline"
UNIT = "NU points/s"
K_E2E = 20  # end-to-end calls timed (a few ms each: enough to average out PCIe jitter)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def hot_kernel_name(cfg):
    """The kernel the plan dispatches for this config's hot stage
    (esn_inst.cuh: SpreadGlobalOp / SpreadRowsOp / SpreadBatchOp / InterpOp)."""
    f32 = cfg.get("dtype", "float64") == "float32"
    if cfg["ttype"] == 2:
        return "k_interp_tile" if f32 else "k_interp_bulk"
    if cfg["dim"] == 1:
        return "k_spread_global"
    if cfg["dim"] == 2 and f32 and cfg.get("ntransf", 1) > 1:
        b2 = os.environ.get("ESN_B2")
        return {"tile": "k_spread_batch2d", "own": "k_spread_b2own"}.get(b2, "k_spread_b2roll")
    if cfg["dim"] == 3:
        return "k_spread_rows" if os.environ.get("ESN_SPREAD3") == "rows" else "k_spread_rows3"
    return "k_spread_rows"


# what actually bounds each config's hot kernel (ncu
# pipe / shared-memory utilisation); roofline.frac stays the HBM fraction
BINDING = {
    "c1": "launch / latency (1e5 points; CUDA-graph replay)",
    "c2": "shared-memory wavefronts (59.7 M: ~73 % of the LSU pipe over the kernel) + FP64 pipe (~32 %), not HBM",
    "c3": "shared-memory wavefronts (14 per point-warp pass around 16 FP64 instructions; ~58 % of the LSU pipe) "
          "+ FP64 pipe ~31 % at 16 warps per SM, not HBM",
    "c3f": "shared-memory wavefronts (~53 % of the LSU pipe) / issue 55 % (two-point step: 32 instructions around "
           "12 FFMA2 / FMUL2), not HBM",
    "c4": "FP64 pipe 46 % + shared-memory wavefronts (~62 % of the LSU pipe; 1000 cells per point at ~56 % lane "
          "coverage), not HBM",
    "c5": "latency (12 warps per SM: short scoreboard 34 %, wait 26 %; issue 35 %), DRAM ~ algorithmic bytes",
}


def algorithmic_bytes(cfg, M, T):
    """B = M d s_r + T M s_c + T G s_c for the spread/interp."""
    sr = 8 if cfg["dtype"] == "float64" else 4
    sc = 2 * sr
    w = select_w(cfg)
    G = 1
    for n in cfg["nm"]:
        G *= next_smooth(max(math.ceil(2.0 * n), 2 * w))
    return M * cfg["dim"] * sr + T * M * sc + T * G * sc, G


# measured FMA peaks of the box (tools/micro/fma_peak.cu; profiles/r01/fma_peak.txt)
FMA_PEAK = {"float64": 1.7e13, "float32": 3.57e13}


def algorithmic_fma(cfg, M, T):
    """FMAs the spread / interp kernel must issue: the ES rows by Horner
    (d w (w + 3) per point, shared by the transforms) plus the separable
    complex accumulation 2 (w + w^2 + ... + w^d) per point and transform."""
    w, d = select_w(cfg), cfg["dim"]
    rows = d * w * (w + 3)
    acc = 2 * sum(w ** k for k in range(1, d + 1))
    return M * rows + M * T * acc


def select_w(cfg):
    return min(max(math.ceil(math.log10(1.0 / cfg["tol"])) + 1, 2), 16)


def next_smooth(n):
    best = None
    p2 = 1
    while True:
        p23 = p2
        while True:
            v = p23
            while v < n:
                v *= 5
            best = v if best is None else min(best, v)
            if p23 >= n:
                break
            p23 *= 3
        if p2 >= n:
            break
        p2 *= 2
    return best


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        try:
            rows = [l.strip().split(",") for l in open(self.path) if l.strip()]
        except Exception:
            return out
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1]))
                mx.append(float(r[2]))
            except ValueError:
                continue
            for nm, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if sm:
            out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                   "reasons": sorted(reasons), "samples": len(sm)}
        try:
            os.unlink(self.path)
        except Exception:
            pass
        return out


# ---------------------------------------------------------------------------
# CPU reference arm (the oracle port of the reference path, all host threads)

def cpu_run(name, M_sample, T_sample, steps, warmup, dist="uniform"):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import esn_oracle as O
    O.build()
    cores = O.num_procs()
    coords, data, cfg = cases.make_inputs(name, M=M_sample, ntransf=T_sample, dist=dist)
    M_sample = cfg["M_actual"]
    wcoords, wdata, _ = cases.make_inputs(name, M=min(M_sample, 2000), ntransf=T_sample, dist=dist)

    stage = {}

    def one(cs, dd):
        st = {}
        if cfg["ttype"] == 1:
            batch = dd if dd.ndim == 2 else dd[None]
            for c in batch:  # the reference has no batch API: a loop of transforms
                tt = {}
                O.exec_type1(cs, c, cfg["nm"], tol=cfg["tol"], isign=cfg["isign"], threads=cores, timings=tt)
                for k, v in tt.items():
                    st[k] = st.get(k, 0.0) + v
        else:
            O.exec_type2(cs, dd, tol=cfg["tol"], isign=cfg["isign"], threads=cores, timings=st)
        return st

    one(wcoords, wdata)
    for _ in range(warmup):
        one(coords, data)
    ts, sts = [], []
    for _ in range(steps):
        t0 = time.perf_counter()
        sts.append(one(coords, data))
        ts.append(time.perf_counter() - t0)
    per_step = statistics.median(ts)
    T = T_sample if cfg["ttype"] == 1 else 1
    # M / t_total and M / t_spread (the spread / interp stage alone)
    spread_s = statistics.median([x.get("spread", float("nan")) for x in sts])
    stage.update({k: statistics.median([x.get(k, 0.0) for x in sts]) for k in ("sort", "spread", "fft", "correct")})
    cpu_run.last = {"value_spread_stage": M_sample * T / spread_s if spread_s > 0 else None,
                    "stages_s": stage}
    return M_sample * T / per_step, per_step, cores


def cpu_sample_size(name):
    cfg = cases.CONFIGS[name]
    M, T = cfg["M_full"], cfg["ntransf"]
    # bounded so one step is a few seconds of CPU work on an 8-32 core host
    if name == "c5":
        return M, 4
    if M > 2_000_000 and cfg["dim"] == 3:
        return 2_000_000, T
    return M, T


# ---------------------------------------------------------------------------
# GPU arm

def run_mode(cfg, world, reduce):
    """Multi-GPU mode of a config."""
    # (--reduce peer also runs the point-split path on one GPU: the fused
    # spread-into-the-root's-grid code with a world of one)
    if (world > 1 or reduce == "peer") and cfg["ttype"] == 1 and cfg["ntransf"] == 1 and cfg["dim"] == 3:
        return "points"
    if world > 1 and cfg["ntransf"] > 1:
        return "transforms"
    return "replica"


def gpu_run(args, name, rank, world, local_rank, *, steps, warmup, reduce, e2e, points="uniform"):
    """Device-resident timing of one config (+ the end-to-end leg).

    replica    : every rank its own independent M points (weak scaling);
    points     : one transform, its points split across ranks, the partial
                 fine grids (reduce="grid", north_star) or mode arrays
                 (reduce="modes") NCCL-reduced to rank 0 (strong scaling);
    transforms : a batch split across ranks, results all-gathered (strong)."""
    import torch
    import torch.distributed as dist
    from paper_1808_06736_b200.distributed import shard_range
    from paper_1808_06736_b200.plan import Plan

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    cfg = cases.CONFIGS[name]
    M, T = cfg["M_full"], cfg["ntransf"]
    mode = run_mode(cfg, world, reduce)
    coords, data, cfg = cases.make_inputs(name, M=M, ntransf=T, dist=points)
    M = cfg["M_actual"]
    Mr, Tr = M, T
    if mode == "points":
        lo, hi = shard_range(M, rank, world)
        coords = [x[lo:hi] for x in coords]
        data = data[lo:hi]
        Mr = hi - lo
    elif mode == "transforms":
        lo, hi = shard_range(T, rank, world)
        data = data[lo:hi]
        Tr = hi - lo
    elif rank > 0 and points == "uniform":
        # replicas: every rank owns an independent shard (its own seed)
        rng = np.random.default_rng(cfg["seed"] + 7919 * rank)
        coords = [rng.uniform(cfg["lo"], cfg["hi"], M) for _ in range(cfg["dim"])]
    real = torch.float64 if cfg["dtype"] == "float64" else torch.float32
    cplx = torch.complex128 if cfg["dtype"] == "float64" else torch.complex64
    xs = [torch.from_numpy(x).to(dev, real).contiguous() for x in coords]
    d = torch.from_numpy(np.ascontiguousarray(data)).to(dev, cplx).contiguous()
    if Tr < 1:
        raise SystemExit(f"rank {rank}: no transforms for world {world} (T={T})")
    plan = Plan(cfg["ttype"], cfg["dim"], nmodes=cfg["nm"], isign=cfg["isign"], ntransf=Tr,
                tol=cfg["tol"], device=dev, dtype=cfg["dtype"], method=args.method, timing=True)
    if cfg["ttype"] == 1:
        out = torch.empty(((Tr,) if T > 1 else ()) + tuple(reversed(cfg["nm"])), dtype=cplx, device=dev)
        cin, fout = d, out
    else:
        out = torch.empty((Tr, Mr) if T > 1 else (Mr,), dtype=cplx, device=dev)
        cin, fout = out, d
    stream = torch.cuda.current_stream(dev)
    gathered = None
    if mode == "transforms":
        width = max(h - l for l, h in (shard_range(T, r, world) for r in range(world)))
        gathered = [torch.empty((width,) + tuple(out.shape[1:]), dtype=cplx, device=dev) for _ in range(world)]
        padded = torch.zeros_like(gathered[0])
    fine = None
    if mode == "points" and reduce == "grid":
        fine = torch.empty(tuple(reversed(plan.nfine)), dtype=cplx, device=dev)
    peer_grid = peer_target = None
    if mode == "points" and reduce == "peer":
        # reduction fused into the spreader: rank 0 owns the fine grid in
        # peer-mappable memory, every rank's tile flushes RED into it over
        # NVLink (distributed.exec_type1_peer_reduced); no reduce collective
        from paper_1808_06736_b200 import peer
        shape = tuple(reversed(plan.nfine))
        box = [None]
        if rank == 0:
            pbuf = peer.PeerBuffer(int(np.prod(shape)) * (16 if cplx == torch.complex128 else 8), dev)
            peer_grid = pbuf.tensor(cplx, shape)
            box[0] = pbuf.handle
        if world > 1:
            dist.broadcast_object_list(box, src=0)
        peer_target = peer_grid if rank == 0 else peer.open_peer(box[0], dev)

    def step():
        plan.setpts(xs)
        if peer_target is not None:
            if rank == 0:
                peer_grid.zero_()
                stream.synchronize()
            if world > 1:
                dist.barrier()  # the grid is zeroed before any rank adds
            plan.spread_add(cin, peer_target)
            if world > 1:
                stream.synchronize()
                dist.barrier()  # every rank's REDs have landed
            if rank == 0:
                plan.finish_type1(peer_grid, fout)
            return
        if fine is not None:
            # fine-grid reduce (north_star): spread, NCCL-reduce the fine
            # grids, root alone runs FFT + deconvolution
            plan.spread(cin, fine)
            dist.reduce(torch.view_as_real(fine), dst=0, op=dist.ReduceOp.SUM)
            if rank == 0:
                plan.finish_type1(fine, fout)
            return
        plan.execute(cin, fout)
        if mode == "points":
            dist.reduce(torch.view_as_real(out), dst=0, op=dist.ReduceOp.SUM)
        elif mode == "transforms":
            padded[: out.shape[0]].copy_(out)
            dist.all_gather([torch.view_as_real(g) for g in gathered], torch.view_as_real(padded))

    for _ in range(max(warmup, 0)):
        step()
    plan.check()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    hot, stages = [], {"sort": 0.0, "spread": 0.0, "fft": 0.0, "correct": 0.0}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        for k in range(steps):
            step()
            if args.stage_sync:
                st = plan.stage_times()
                for key in stages:
                    stages[key] += st[key]
                hot.append(plan.hot_kernel_seconds())
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
    elapsed = ev0.elapsed_time(ev1) / 1e3
    if not args.stage_sync:
        st = plan.stage_times()
        stages = {k: v * steps for k, v in st.items()}
        hot = [plan.hot_kernel_seconds()]
    plan.check()
    t = torch.tensor([elapsed], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed = float(t.item())
    Tn = T if cfg["ttype"] == 1 else 1
    # units processed by the whole job per step: replicas each own M points;
    # a split transform / batch is M * T in total
    total_units = M * Tn * (world if mode == "replica" else 1)
    value = total_units * steps / elapsed
    B, G = algorithmic_bytes(cfg, Mr, Tr)
    hot_s = statistics.mean(hot)
    peak, peak_kind = peaks()
    res = dict(value=value, elapsed=elapsed, steps=steps, hot_s=hot_s, achieved=B / hot_s / 1e9, peak=peak,
               mode=mode, M=M, peak_kind=peak_kind, B=B, G=G, clocks=clk.summary(), reduce=reduce,
               fma=algorithmic_fma(cfg, Mr, Tr),
               stages={k: v / steps for k, v in st.items()} if not args.stage_sync
               else {k: v / steps for k, v in stages.items()})
    plan.close()
    if peer_target is not None:
        if world > 1:
            dist.barrier()  # nobody still adds into the root's grid
        peer_grid = None
        if rank == 0:
            pbuf.free()
    del xs, d, out, fine, gathered
    torch.cuda.empty_cache()
    if e2e:
        if mode == "replica":
            e2 = e2e_host_abi(args, cfg, coords, data, M, T, dev, warmup)
        else:
            e2 = e2e_sharded(cfg, coords, data, M, Mr, T, Tr, mode, reduce, rank, world, dev, warmup)
        te = torch.tensor([e2.pop("elapsed")], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        units = M * (T if cfg["ttype"] == 1 else 1) * (world if mode == "replica" else 1)
        e2["value"] = units * e2.pop("calls") / float(te.item())
        e2["ms_per_step"] = float(te.item()) / e2["calls_timed"] * 1e3
        res["e2e"] = e2
    return res


def e2e_host_abi(args, cfg, coords, data, M, T, dev, warmup):
    """End to end through the C ABI one-shot routine esn_nufft_host with
    pinned HOST buffers: H2D of the inputs and D2H of the result inside the
    timed region (this rank's own M points / T transforms)."""
    import torch
    from paper_1808_06736_b200 import _lib
    from paper_1808_06736_b200.plan import make_opts
    cplx = torch.complex128 if cfg["dtype"] == "float64" else torch.complex64
    # float32 configs take float32 coordinates (the values are float32-exact,
    # cases.make_inputs); the host routine reads them as such (coord_dtype)
    f32c = cfg["dtype"] == "float32"
    hx = [torch.from_numpy(x.astype(np.float32) if f32c else x).pin_memory() for x in coords]
    # a config whose strengths ARE complex64 (c3: "c_j complex64", computed in
    # float64) hands them over as such: upcast exactly on the device
    c64in = cfg["ttype"] == 1 and cfg["dtype"] == "float64" and cfg.get("cdtype") == "complex64"
    hd = torch.from_numpy(np.ascontiguousarray(data)).to(torch.complex64 if c64in else cplx).pin_memory()
    assert hx[0].numel() == M, "e2e buffers must hold exactly this rank's M points"
    if cfg["ttype"] == 1:
        assert hd.numel() == M * T
        hout = torch.empty(((T,) if T > 1 else ()) + tuple(reversed(cfg["nm"])), dtype=cplx).pin_memory()
        cptr, fptr = hd.data_ptr(), hout.data_ptr()
    else:
        hout = torch.empty((T, M) if T > 1 else (M,), dtype=cplx).pin_memory()
        cptr, fptr = hout.data_ptr(), hd.data_ptr()
    h2d = sum(x.numel() * x.element_size() for x in hx) + hd.numel() * hd.element_size()
    d2h = hout.numel() * hout.element_size()
    o, keep = make_opts(dtype=cfg["dtype"], method=args.method, timing=False,
                        strength_dtype="float32" if c64in else None,
                        coord_dtype="float32" if f32c else None)
    nm = _lib.i64_array(cfg["nm"])
    xp = [ctypes.c_void_p(x.data_ptr()) for x in hx] + [None] * (3 - len(hx))

    def call():
        _lib.check(_lib.lib.esn_nufft_host(cfg["ttype"], cfg["dim"], M, xp[0], xp[1], xp[2], T,
                                           ctypes.c_void_p(cptr), cfg["isign"], cfg["tol"], nm,
                                           ctypes.c_void_p(fptr), ctypes.byref(o)))

    for _ in range(max(1, warmup)):
        call()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(K_E2E):
        call()
    el = time.perf_counter() - t0
    return {"elapsed": el, "calls": K_E2E, "calls_timed": K_E2E, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "api": "esn_nufft_host (C ABI, pinned host buffers)"}


def e2e_sharded(cfg, coords, data, M, Mr, T, Tr, mode, reduce, rank, world, dev, warmup):
    """End to end of the sharded paths through the package's public
    distributed API (paper_1808_06736_b200.distributed) with pinned HOST
    buffers: each rank's shard goes H2D, is spread (and, for the modes
    reduce / transform split, FFT'd + deconvolved), the NCCL reduce /
    all-gather runs, and rank 0 reads the result back D2H."""
    import torch
    import torch.distributed as dist
    import paper_1808_06736_b200 as E
    from paper_1808_06736_b200 import distributed as DD
    cplx = torch.complex128 if cfg["dtype"] == "float64" else torch.complex64
    real = torch.float64 if cfg["dtype"] == "float64" else torch.float32
    hx = [torch.from_numpy(np.ascontiguousarray(x)).to(real).pin_memory() for x in coords]
    opts = E.TransformOptions(tolerance=cfg["tol"], isign=cfg["isign"], dtype=cfg["dtype"], device=dev)
    if mode == "points":
        hd = torch.from_numpy(np.ascontiguousarray(data)).to(cplx).pin_memory()
        assert hx[0].numel() == Mr and hd.numel() == Mr

        def call():
            if reduce == "grid":
                r = DD.exec_type1_grid_reduced(hx, hd, cfg["nm"], opts, dst=0)
            elif reduce == "peer":
                r = DD.exec_type1_peer_reduced(hx, hd, cfg["nm"], opts, dst=0)
            else:
                r = DD.exec_type1_point_sharded(hx, hd, cfg["nm"], opts, dst=0)
            return r.cpu() if rank == 0 else None
        h2d = sum(x.numel() * x.element_size() for x in hx) + hd.numel() * hd.element_size()
        d2h = int(np.prod(cfg["nm"])) * hd.element_size() if rank == 0 else 0
    else:
        # the transform split reads only this rank's rows of the (T, M)
        # host batch; the other rows are never touched
        from paper_1808_06736_b200.distributed import shard_range
        lo, hi = shard_range(T, rank, world)
        hd = torch.empty((T, M), dtype=cplx).pin_memory()
        hd[lo:hi].copy_(torch.from_numpy(np.ascontiguousarray(data)).to(cplx))

        def call():
            r = DD.exec_type1_transform_sharded(hx, hd, cfg["nm"], opts)
            return r.cpu() if rank == 0 else None
        h2d = sum(x.numel() * x.element_size() for x in hx) + (hi - lo) * M * hd.element_size()
        d2h = T * int(np.prod(cfg["nm"])) * hd.element_size() if rank == 0 else 0
    for _ in range(max(1, warmup)):
        call()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    k = 5
    t0 = time.perf_counter()
    for _ in range(k):
        call()
    torch.cuda.synchronize(dev)
    el = time.perf_counter() - t0
    return {"elapsed": el, "calls": k, "calls_timed": k, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h),
            "api": ("distributed.exec_type1_peer_reduced" if mode == "points" and reduce == "peer" else
                    "distributed.exec_type1_grid_reduced" if mode == "points" and reduce == "grid" else
                    "distributed.exec_type1_point_sharded" if mode == "points" else
                    "distributed.exec_type1_transform_sharded")
                   + " (pinned host shards; H2D, spread/FFT, NCCL, D2H on rank 0)"}


def config_block(name, world, dist="uniform", M=None, mode="replica", reduce="grid"):
    cfg = cases.CONFIGS[name]
    nm = "x".join(str(v) for v in cfg["nm"])
    M = cfg["M_full"] if M is None else M
    pts = "iid uniform, seeded" if dist == "uniform" else f"{dist} quadrature cloud (clustered)"
    per = " per GPU" if mode == "replica" else " total"
    par = "1 GPU"
    if world > 1:
        par = {"replica": f"replica shards x{world} (independent points per GPU)",
               "points": f"points split x{world}, "
                         + ("spreaders RED into the root's peer-mapped fine grid (no reduce collective), "
                            "root FFT + deconv" if reduce == "peer" else
                            "NCCL reduce of the partial "
                            + ("fine grids, root FFT + deconv" if reduce == "grid" else "mode arrays")),
               "transforms": f"transforms split x{world}, all-gather of the results"}[mode]
    return {
        "workload": f"{name}: {cfg['dim']}D type-{cfg['ttype']}, modes {nm}, M={M:.0e}{per}, "
                    f"eps={cfg['tol']:g}, isign={cfg['isign']:+d}, ntransf={cfg['ntransf']}"
                    + ("" if dist == "uniform" else f", points {dist}"),
        "dim": cfg["dim"], "type": cfg["ttype"], "modes": list(cfg["nm"]),
        ("M_per_gpu" if mode == "replica" else "M_total"): M,
        "tol": cfg["tol"], "ntransf": cfg["ntransf"], "points": pts, "parallelism": par,
        "l2": "inputs larger than L2 (coords + outputs > 126 MB), no explicit flush",
    }


def cpu_info():
    """CPU model and core counts of this host."""
    info = {"logical_cores": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {}
        for line in out.splitlines():
            if ":" in line:
                k, v = line.split(":", 1)
                kv[k.strip()] = v.strip()
        info["cpu_model"] = kv.get("Model name")
        sockets = int(kv.get("Socket(s)", "1") or 1)
        cps = int(kv.get("Core(s) per socket", "0") or 0)
        info["physical_cores"] = sockets * cps if cps else None
        info["threads_per_core"] = int(kv.get("Thread(s) per core", "1") or 1)
    except Exception:
        pass
    try:
        info["affinity_cores"] = len(os.sched_getaffinity(0))
    except Exception:
        pass
    return info


def n_launches(cfg):
    """Our kernels per step: setpts = count, scan x2 (reduce, down sweep),
    scatter, subproblem scan + fill (6); type 2: amplify + interp; type 1:
    spread (batched: permute + row table + spread) + deconv.  cuFFT's own
    kernels excluded."""
    hk = hot_kernel_name(cfg)
    return 6 + (2 if cfg["ttype"] == 2 else (3 if hk in ("k_spread_batch2d", "k_spread_b2own", "k_spread_b2roll") else 1) + 1)


def line_for(args, name, res, world, base):
    cfg = cases.CONFIGS[name]
    frac = res["achieved"] / res["peak"]
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(name)
        except Exception:
            traffic = None
    kern = "interp" if cfg["ttype"] == 2 else "spread"
    b = dict(base)
    if res["mode"] != "replica":
        b["scaling"] = "strong"
    line = dict(b, value=res["value"], ms_per_step=res["elapsed"] / res["steps"] * 1e3,
                config=config_block(name, world, args.points, res["M"], res["mode"], res["reduce"]),
                roofline={"bound": "hbm", "achieved": res["achieved"], "peak": res["peak"],
                          "unit": "GB/s", "frac": frac, "traffic": traffic,
                          "kernel": f"{kern} ({hot_kernel_name(cfg)})",
                          "algorithmic_bytes": res["B"], "kernel_ms": res["hot_s"] * 1e3,
                          "peak_source": f"{res['peak_kind']} MEASURED_PEAKS.json hbm_gbs",
                          "binding": BINDING.get(name)},
                stages_ms={k: v * 1e3 for k, v in res["stages"].items()},
                clocks=res["clocks"], gpu_launches=n_launches(cfg) * res["steps"])
    if "fma" in res:  # the compute roof beside the HBM one (which binds for fp64 interp / 3D spread)
        fpk = FMA_PEAK["float32" if cfg["dtype"] == "float32" else "float64"]
        ach = res["fma"] / res["hot_s"]
        line["roofline"]["compute"] = {"unit": "FMA/s", "algorithmic_fma": res["fma"], "achieved": ach,
                                       "peak": fpk, "frac": ach / fpk,
                                       "peak_source": "measured on a B200 (tools/micro/fma_peak.cu, "
                                                      "profiles/r01/fma_peak.txt)"}
    if traffic is not None:
        line["roofline"]["traffic_source"] = "profiles/traffic.json (ncu dram__bytes_read+write of this kernel)"
        try:  # was it measured on the library being benched? (tools/kernel_table.py)
            stamp = json.load(open(tp)).get("_so", {}).get(name)
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            import kernel_table
            line["roofline"]["traffic_same_build"] = stamp == kernel_table.so_sha()
        except Exception:
            line["roofline"]["traffic_same_build"] = None
    if "e2e" in res:
        line["e2e"] = res["e2e"]
    return line


def self_launch(args):
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-run this
    script under torch.distributed.run with N ranks on 127.0.0.1."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible", file=sys.stderr)
        sys.exit(2)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    print("bench.py: launching " + " ".join(cmd), file=sys.stderr, flush=True)
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=list(cases.CONFIGS))
    ap.add_argument("--method", default="auto")
    ap.add_argument("--reduce", default="grid", choices=["modes", "grid", "peer"],
                    help="multi-GPU single 3D type 1: NCCL-reduce the fine grids (north_star; root alone "
                         "runs FFT + deconv) or the per-rank mode arrays (each rank FFTs + deconvolves)")
    ap.add_argument("--points", default="uniform", choices=list(cases.DISTRIBUTIONS),
                    help="point cloud: the config's iid uniform points, or the paper's clustered "
                         "disc-quad (2D) / sph-quad (3D) quadrature clouds of about M points")
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-cpu", dest="cpu", action="store_false")
    ap.add_argument("--no-sharded", dest="sharded", action="store_false",
                    help="skip the sharded-config measurements (c3 point split, c5 transform split) "
                         "attached to the default c2 line")
    ap.add_argument("--stage-sync", action="store_true",
                    help="read stage events after every step (adds a host sync per step)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    in_torchrun = "WORLD_SIZE" in os.environ
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = cases.CONFIGS[args.config]
    base = {"metric": METRIC, "unit": UNIT, "n_gpus": world if in_torchrun else args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64" if cfg["dtype"] == "float64" else "f32",
            "data": "synthetic (seeded " + ("iid uniform" if args.points == "uniform" else args.points)
                    + " points, N(0,1) complex data; BASELINE.json shapes)"}

    if args.impl == "reference":
        if rank != 0:
            return
        Ms, Ts = cpu_sample_size(args.config)
        v, per, cores = cpu_run(args.config, Ms, Ts, max(1, args.steps), args.warmup, args.points)
        line = dict(base, value=v, ms_per_step=per * 1e3, impl="reference",
                    config=config_block(args.config, 1, args.points),
                    cpu_baseline=dict({"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                                       "sample": f"{args.config} with M={Ms:.0e}, ntransf={Ts} per step "
                                                 "(oracle/ C+OpenMP restatement of the reference path, "
                                                 "scipy pocketfft)"}, **cpu_info(), **getattr(cpu_run, "last", {})),
                    e2e={"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
        line["n_gpus"] = args.gpus
        print(json.dumps(line), flush=True)
        return

    if not in_torchrun and args.gpus > 1:
        self_launch(args)
    import torch
    import torch.distributed as dist
    if in_torchrun and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if torch.cuda.device_count() < (local_rank + 1):
        print(f"bench.py: rank {rank} needs cuda:{local_rank}, {torch.cuda.device_count()} visible",
              file=sys.stderr)
        sys.exit(2)
    if in_torchrun:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        print(f"bench.py: rank {rank}/{world} on cuda:{local_rank} "
              f"({torch.cuda.get_device_name(local_rank)}), NCCL {torch.cuda.nccl.version()}",
              file=sys.stderr, flush=True)
    res = gpu_run(args, args.config, rank, world, local_rank, steps=args.steps, warmup=args.warmup,
                  reduce=args.reduce, e2e=args.e2e, points=args.points)
    sharded = {}
    if args.sharded and args.config == "c2" and args.points == "uniform":
        # north_star: the sharded configs at every N -- c3 one transform with
        # its points split (fine-grid reduce, and the mode-array variant)
        # and c5's batch split; printed inside the same line
        runs = [("c3_grid_reduce", "c3", "grid"), ("c3_modes_reduce", "c3", "modes"),
                ("c5_transform_split", "c5", "grid")]
        if world == 1:  # (one GPU: no reduce, the two c3 variants coincide)
            runs = [("c3", "c3", "grid"), ("c5", "c5", "grid")]
        for key, name, red in runs:
            r = gpu_run(args, name, rank, world, local_rank, steps=5, warmup=3, reduce=red,
                        e2e=args.e2e and red == "grid")
            if rank == 0:
                ln = line_for(args, name, r, world, base)
                sharded[key] = {k: ln[k] for k in ("value", "ms_per_step", "scaling", "config", "roofline",
                                                   "stages_ms") if k in ln}
                sharded[key]["n_gpus"] = world
                sharded[key]["gpu_launches"] = n_launches(cases.CONFIGS[name]) * 5
                if "e2e" in ln:
                    sharded[key]["e2e"] = ln["e2e"]
    if world > 1:
        dist.barrier()
    if rank == 0:
        line = line_for(args, args.config, res, world, base)
        if sharded:
            line["sharded_configs"] = sharded
            line["gpu_launches"] += sum(v["gpu_launches"] for v in sharded.values())
        if args.cpu and world == 1:
            try:
                Ms, Ts = cpu_sample_size(args.config)
                v, per, cores = cpu_run(args.config, Ms, Ts, 1, 0, args.points)
                line["cpu_baseline"] = dict({"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                                             "sample": f"{args.config} with M={Ms:.0e}, ntransf={Ts}, one "
                                                       "full transform (oracle/ C+OpenMP port, scipy FFT)"},
                                            **cpu_info(), **getattr(cpu_run, "last", {}))
            except Exception as exc:  # the baseline must never sink the GPU line
                line["cpu_baseline"] = {"value": None, "error": str(exc)[:200]}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
