#!/usr/bin/env python3
"""bench.py -- SSAM engine benchmark (driver contract).

Headline workload (BASELINE.json configs[4], the config its metric is quoted
on "at 1/2/4/8 B200"): 3D 7-point Jacobi, fp32, on a 2048 x 2048 x (512*N)
grid z-slab-sharded over N GPUs (one process per GPU, NCCL halo exchange of
one 16 MiB plane per neighbour per sweep, overlapped with the interior).
One step = `--iters` (default 100) sweeps of the whole grid.  Weak scaling:
each GPU always owns 2048 x 2048 x 512 cells.

  value   whole-job cell-updates per second (GCells/s), device-resident
          inputs, CUDA events on the compute stream, max over ranks.
  e2e     the same metric through the public C ABI with HOST buffers
          (ssam_b200_stencil3d at N=1; the slab runner at N>1): pinned
          host->device copy of the step's input, the sweeps, and the
          device->host copy of the result inside the timed region.
  roofline  the dominant kernel (ssam3d_kernel, 3d7pt fp32): algorithmic
          bytes (4 B read + 4 B write per updated cell) / mean launch time.
  kernels per-kernel GCells/s and %-of-peak for the other configs (conv
          sweep 3x3..20x20, 2D stencils x100 sweeps, 3D stencils at 512^3),
          rank 0 at N=1.
  cpu_baseline  the reference's own CPU path (oracle/_ref, ssam::stencil3d,
          all host threads) on a bounded sample of the same workload.

--impl reference times that reference CPU path alone (rank 0; other ranks
exit 0).  Data are synthetic: the reference's SplitMix64 stream generated on
the device (bit-identical to random_grid3d), seed 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GCells/s and achieved HBM GB/s (% of peak) per kernel at 1/2/4/8 B200"
NX = NY = 2048
NZ_PER_GPU = 512
STENCIL = "3d7pt"


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured", float(p.get("sm_max_mhz", 1965.0))
    except Exception:
        return 6650.0, "fallback", 1965.0


def load_traffic():
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref) -- cpu_baseline and --impl reference
# ---------------------------------------------------------------------------

def cpu_model() -> str:
    """Host CPU model (record nproc and the CPU model beside the CPU timing)."""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_sample(seconds: float = 10.0, max_reps: int = 1000):
    """ssam::stencil3d<float> 3d7pt (the reference's CPU SSAM path, all host
    threads) on a 2048 x 2048 x 16 block of the same seeded grid, repeated
    single sweeps until `seconds` of CPU work.  Returns (GCells/s, cores, sample)."""
    import numpy as np
    from oracle import Oracle, Reference
    ref = Reference()
    orc = Oracle()
    st = ref.benchmark_stencil(STENCIL)
    nz = 16
    g = orc.random_grid((nz, NY, NX), np.float32, 0)
    cf = st["coeffs"].astype(np.float32)
    cells = 0
    t0 = time.perf_counter()
    reps = 0
    while reps < max_reps:
        rc, _, _ = ref.stencil3d(g, st["offsets"], cf, st["order"], 1, p=2, b=128)
        assert rc == 0
        cells += g.size
        reps += 1
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    return cells / dt / 1e9, ref.max_threads(), \
        f"{reps} sweep(s) of 3d7pt f32 on a {NX}x{NY}x{nz} block (seed 0), ssam::stencil3d threads=0"


def run_reference_arm(args, rank: int, world: int):
    if rank != 0:
        return
    import numpy as np
    from oracle import Oracle, Reference
    ref = Reference()
    orc = Oracle()
    st = ref.benchmark_stencil(STENCIL)
    nz = 16
    g = orc.random_grid((nz, NY, NX), np.float32, 0)
    cf = st["coeffs"].astype(np.float32)
    for _ in range(args.warmup):
        ref.stencil3d(g, st["offsets"], cf, st["order"], 1, p=2, b=128)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        rc, _, _ = ref.stencil3d(g, st["offsets"], cf, st["order"], 1, p=2, b=128)
        assert rc == 0
    dt = time.perf_counter() - t0
    value = g.size * args.steps / dt / 1e9
    sample = (f"each step: 1 sweep of 3d7pt f32 on a {NX}x{NY}x{nz} block of the workload "
              f"(seed 0), ssam::stencil3d from oracle/_ref, threads=0")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "GCells/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(world, args),
        "cpu_baseline": {"value": round(value, 6), "unit": "GCells/s",
                         "cores": ref.max_threads(), "kind": "reference", "sample": sample,
                         "cpu_model": cpu_model(), "nproc": os.cpu_count()},
        "e2e": {"value": round(value, 6), "unit": "GCells/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def backend() -> str:
    """NCCL in production; SSAM_BENCH_BACKEND=gloo runs the N > 1 flow on fewer GPUs
    (ranks share devices, halos staged through host memory) to test it on one B200."""
    return os.environ.get("SSAM_BENCH_BACKEND", "nccl")


def rank_device(local_rank: int) -> int:
    import torch
    return local_rank % max(1, torch.cuda.device_count())


def reduce_host(x: float, op: str) -> float:
    """Max / sum of a scalar over ranks (device tensor for NCCL, host for gloo)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64,
                     device="cuda" if backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def workload_config(world: int, args):
    return {"workload": f"{STENCIL} f32 {NX}x{NY}x({NZ_PER_GPU}*N) z-slab, NVLink halo exchange",
            "stencil": STENCIL, "nx": NX, "ny": NY, "nz": NZ_PER_GPU * world,
            "nz_per_gpu": NZ_PER_GPU, "iters_per_step": args.iters,
            "temporal_block": max(1, args.tb),
            "temporal_blocking": ("each launch fuses temporal_block sweeps (one HBM pass, "
                                  "bit-identical to single sweeps), as ssam_b200_stencil3d_run "
                                  "does for this stencil; --tb 1 times single sweeps"),
            "halo": ("kernel stores into neighbours' CUDA IPC buffers (peer.py)"
                     if args.halo == "peer" and world > 1 else
                     "boundary planes first, NCCL send/recv overlapped with the interior"),
            "parallelism": f"z-slab x{world}", "seed": 0,
            "l2": "no flush needed: 8 GiB per buffer >> 126 MB L2"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args, rank: int, world: int, local_rank: int):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1907_06154_b200 as ssam
    from paper_1907_06154_b200 import device as dev
    from paper_1907_06154_b200.slab import SlabRunner, decompose, fill_slab

    torch.cuda.set_device(rank_device(local_rank))
    peak, peak_kind, sm_max_nominal = load_peaks()
    st = ssam.convert_stencil(ssam.make_benchmark_stencil(STENCIL), np.float32)
    k = st.order
    tb = max(1, args.tb)
    slab = decompose(NZ_PER_GPU * world, world, rank, k, ghost=k * tb)
    peer = args.halo == "peer" and world > 1
    if peer:  # the kernels store the halo into the neighbours' IPC-mapped buffers
        from paper_1907_06154_b200.peer import PeerSlabRunner
        group = None if backend() == "gloo" else dist.new_group(backend="gloo")
        prun = PeerSlabRunner(slab, st, NX, NY, torch.float32, group=group, tb=tb)
        a, b = prun.a, prun.b
    else:
        a = torch.empty((slab.nz_local, NY, NX), dtype=torch.float32, device="cuda")
    fill_slab(a, slab, NX, NY, seed=0)
    if peer:
        b.copy_(a)
    else:
        b = a.clone()
    comm = torch.cuda.Stream() if world > 1 else None

    launch_ms = []
    timing = {"on": False}

    def sweep(cur, nxt, zb, ze):
        if ze <= zb:
            return
        if timing["on"] and zb == slab.compute_range()[0] and world == 1:
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            dev.stencil3d_sweep(cur, nxt, st, zb, ze)
            e.record()
            launch_ms.append((s, e))
        else:
            dev.stencil3d_sweep(cur, nxt, st, zb, ze)

    rlo, rhi = slab.ring_bounds()

    def fused(cur, nxt, zb, ze):
        if ze <= zb:
            return
        if timing["on"] and zb == slab.compute_range()[0] and world == 1:
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            dev.stencil3d_tb(cur, nxt, st, tb, zb, ze, rlo, rhi)
            e.record()
            launch_ms.append((s, e))
        else:
            dev.stencil3d_tb(cur, nxt, st, tb, zb, ze, rlo, rhi)

    runner = SlabRunner(slab, sweep, comm_stream=comm, fused=fused if tb > 1 else None, tb=tb)

    def run_step():
        if peer:
            prun.run(args.iters)
        else:
            runner.run(a, b, args.iters)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        run_step()
    torch.cuda.synchronize()
    barrier()

    clocks = ClockSampler(torch.cuda.current_device())  # nvidia-smi index = CUDA index here
    clocks.start()
    time.sleep(0.3)
    n_launch0 = ssam.launch_count()
    barrier()
    torch.cuda.synchronize()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    timing["on"] = True
    t_start.record()
    for _ in range(args.steps):
        run_step()
    t_end.record()
    torch.cuda.synchronize()
    timing["on"] = False
    barrier()
    clk = clocks.stop()
    elapsed_ms = t_start.elapsed_time(t_end)
    launches = ssam.launch_count() - n_launch0

    max_ms, n_launches = elapsed_ms, float(launches)
    if world > 1:
        max_ms = reduce_host(elapsed_ms, "max")
        n_launches = reduce_host(float(launches), "sum")
    total_cells = NX * NY * NZ_PER_GPU * world * args.iters * args.steps
    value = total_cells / (max_ms / 1e3) / 1e9

    # dominant kernel: ssam3d_kernel over the whole slab (N=1 timing by launch)
    interior = (NX - 2 * k) * (NY - 2 * k)
    lo, hi = slab.compute_range()
    cells_per_launch = interior * (hi - lo)
    if launch_ms:
        durs = [s.elapsed_time(e) for s, e in launch_ms]
        mean_ms = sum(durs) / len(durs)
    else:
        mean_ms = max_ms / (args.steps * args.iters / tb)
    # a fused launch reads and writes every cell once for its tb updates
    achieved = 8.0 * cells_per_launch / (mean_ms / 1e3) / 1e9
    traffic = load_traffic().get(f"ssam3d_{STENCIL}_f32_{NX}x{NY}x{slab.nz_local}"
                                 + ("_tb2" if tb > 1 else ""))

    # free the slab before the e2e / per-kernel phases
    del a, b
    if peer:
        prun.close()
    torch.cuda.empty_cache()

    e2e = None
    if not args.no_e2e:
        try:
            e2e = e2e_slab(args, slab, st, world, rank)
        except Exception as ex:  # e.g. pinned host memory exhausted on a big box
            e2e = {"value": None, "unit": "GCells/s", "error": f"{type(ex).__name__}: {ex}"[:300]}
            torch.cuda.empty_cache()

    kernels = None
    cpu = None
    if rank == 0 and world == 1 and not args.no_suite:
        kernels = kernel_suite(peak, sm_max_nominal)
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            v, cores, sample = reference_sample(args.cpu_seconds)
            cpu = {"value": round(v, 6), "unit": "GCells/s", "cores": cores, "kind": "reference",
                   "sample": sample, "cpu_model": cpu_model(), "nproc": os.cpu_count()}
        except Exception as ex:  # the reference build may be absent
            cpu = {"value": None, "unit": "GCells/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GCells/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(max_ms / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference SplitMix64 stream, seed 0, generated on device)",
            "config": workload_config(world, args),
            "hbm_gbs_algorithmic": round(value * 8.0 / tb, 1),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": (f"ssam3d_tb2_kernel {STENCIL} f32 (Tb=2: 8 B per "
                                    f"cell per launch = 2 updates)" if tb > 1
                                    else f"ssam3d_halo_kernel {STENCIL} f32"),
                         "bytes_per_launch": 8 * cells_per_launch,
                         "mean_launch_ms": round(mean_ms, 4)},
            "e2e": e2e, "gpu_launches": int(n_launches), "clocks": clk,
            "cpu_baseline": cpu, "kernels": kernels,
        }
        print(json.dumps(line), flush=True)


def e2e_slab(args, slab, st, world, rank):
    """Public-API end to end: pinned host input -> GPU -> host output per step."""
    import numpy as np
    import torch
    import paper_1907_06154_b200 as ssam
    from paper_1907_06154_b200.slab import SlabRunner
    from paper_1907_06154_b200 import device as dev

    nzl = slab.nz_local
    host_in = torch.empty((nzl, NY, NX), dtype=torch.float32, pin_memory=True)
    host_out = torch.empty((nzl, NY, NX), dtype=torch.float32, pin_memory=True)
    tmp = torch.empty((nzl, NY, NX), dtype=torch.float32, device="cuda")
    from paper_1907_06154_b200.slab import fill_slab
    fill_slab(tmp, slab, NX, NY, seed=0)
    host_in.copy_(tmp)
    del tmp
    torch.cuda.empty_cache()
    steps = max(1, args.e2e_steps)
    if world == 1:
        import ctypes
        cfg = ssam.KernelConfig(p=2, b=128)._c()
        sa = ssam._StencilArgs(st, np.float32)

        def one():
            ssam._raise(ssam.lib.ssam_b200_stencil3d(
                0, host_in.data_ptr(), NX, NY, nzl, sa.ref, ctypes.byref(cfg), args.iters,
                host_out.data_ptr(), None))
    else:
        import torch.distributed as dist
        comm = torch.cuda.Stream()
        dev_a = torch.empty((nzl, NY, NX), dtype=torch.float32, device="cuda")
        dev_b = torch.empty_like(dev_a)
        tb = max(1, args.tb)  # the slab carries k * tb ghost planes (run_ours)
        rlo, rhi = slab.ring_bounds()
        runner = SlabRunner(
            slab, lambda c, n, zb, ze: dev.stencil3d_sweep(c, n, st, zb, ze), comm_stream=comm,
            fused=(lambda c, n, zb, ze: dev.stencil3d_tb(c, n, st, tb, zb, ze, rlo, rhi))
            if tb > 1 else None, tb=tb)

        def one():
            dev_a.copy_(host_in, non_blocking=True)
            dev_b.copy_(dev_a)
            res = runner.run(dev_a, dev_b, args.iters)
            host_out.copy_(res, non_blocking=True)
            torch.cuda.synchronize()

    one()  # warm-up (pool allocation, first-touch of pinned pages)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    dt = time.perf_counter() - t0
    if world > 1:
        dt = reduce_host(dt, "max")
    cells = NX * NY * NZ_PER_GPU * world * args.iters * steps
    nbytes = nzl * NY * NX * 4
    return {"value": round(cells / dt / 1e9, 3), "unit": "GCells/s",
            "h2d_bytes_per_step": nbytes * world, "d2h_bytes_per_step": nbytes * world,
            "steps": steps, "ms_per_step": round(dt / steps * 1e3, 3),
            "api": "ssam_b200_stencil3d (C ABI, host buffers)" if world == 1 else
                   "SlabRunner over ssam_b200_stencil3d_sweep / _tb (host buffers)"}


def kernel_suite(peak, sm_mhz):
    """Per-kernel throughput for the other BASELINE configs (device-resident)."""
    import numpy as np
    import torch
    import paper_1907_06154_b200 as ssam
    from paper_1907_06154_b200 import device as dev
    from oracle import Oracle
    orc = Oracle()
    fp32_peak_tflops = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12

    def timed(fn, reps):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps

    out = {}
    H = W = 8192
    g = torch.empty((H, W), dtype=torch.float32, device="cuda")
    dev.fill_random(g, 0)
    o = torch.empty_like(g)
    for K in range(3, 21):
        f = orc.random_filter(K, K, np.float32, 1)
        ms = timed(lambda: dev.conv2d(g, o, f), 5)
        gc = H * W / ms / 1e6
        out[f"conv2d_f32_8192_{K}x{K}"] = {
            "gcells": round(gc, 2), "hbm_gbs": round(gc * 8, 1),
            "hbm_frac": round(gc * 8 / peak, 4), "tflops": round(gc * 2 * K * K / 1e3, 2),
            "fp32_frac": round(gc * 2 * K * K / 1e3 / fp32_peak_tflops, 4), "ms": round(ms, 4)}
    del g, o
    for dt, tdt, npdt, sz in (("f32", torch.float32, np.float32, 4),
                              ("f64", torch.float64, np.float64, 8)):
        a = torch.empty((H, W), dtype=tdt, device="cuda")
        dev.fill_random(a, 0)
        bb = torch.empty_like(a)
        for name in ("2d5pt", "2d9pt", "2ds25pt"):
            st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), npdt)
            iters = 100
            ms = timed(lambda: dev.stencil2d_run(a, bb, st, iters), 1)
            gc = H * W * iters / ms / 1e6
            out[f"stencil2d_{name}_{dt}_8192_x100"] = {
                "gcells": round(gc, 2), "hbm_gbs_equiv": round(gc * 2 * sz, 1),
                "hbm_frac": round(gc * 2 * sz / peak, 4), "ms": round(ms, 3),
                "tb": dev.stencil2d_tb_max(st, npdt)}
        del a, bb
    n = 512
    for dt, tdt, npdt, sz in (("f32", torch.float32, np.float32, 4),
                              ("f64", torch.float64, np.float64, 8)):
        a = torch.empty((n, n, n), dtype=tdt, device="cuda")
        dev.fill_random(a, 0)
        bb = torch.empty_like(a)
        for name in ("3d7pt", "3d13pt", "3d27pt", "poisson"):
            st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), npdt)
            iters = 20
            ms = timed(lambda: dev.stencil3d_run(a, bb, st, iters), 1)
            gc = n ** 3 * iters / ms / 1e6
            out[f"stencil3d_{name}_{dt}_512_x{iters}"] = {
                "gcells": round(gc, 2), "hbm_gbs_equiv": round(gc * 2 * sz, 1),
                "hbm_frac": round(gc * 2 * sz / peak, 4), "ms": round(ms, 3),
                "tb": dev.stencil3d_tb_max(st, npdt) if name == "3d7pt" else 1}
        del a, bb
    # the headline slab with two fused sweeps per HBM pass (engine3d_tb.cuh)
    a = torch.empty((NZ_PER_GPU + 2, NY, NX), dtype=torch.float32, device="cuda")
    dev.fill_random(a, 0)
    bb = a.clone()
    st = ssam.convert_stencil(ssam.make_benchmark_stencil("3d7pt"), np.float32)
    ms1 = timed(lambda: dev.stencil3d_sweep(a, bb, st), 5)
    gc1 = (NX - 2) * (NY - 2) * NZ_PER_GPU / ms1 / 1e6
    out[f"stencil3d_3d7pt_f32_{NX}x{NY}x{NZ_PER_GPU + 2}_tb1"] = {
        "gcells": round(gc1, 2), "hbm_gbs": round(gc1 * 8, 1),
        "hbm_frac": round(gc1 * 8 / peak, 4), "ms": round(ms1, 3), "tb": 1,
        "note": "one sweep per launch (ssam3d_halo_kernel), 8 B/cell"}
    ms = timed(lambda: dev.stencil3d_tb(a, bb, st, 2), 5)
    gc = 2 * (NX - 2) * (NY - 2) * NZ_PER_GPU / ms / 1e6
    out[f"stencil3d_3d7pt_f32_{NX}x{NY}x{NZ_PER_GPU + 2}_tb2"] = {
        "gcells": round(gc, 2), "hbm_gbs": round(gc * 4, 1), "hbm_frac": round(gc * 4 / peak, 4),
        "hbm_gbs_equiv": round(gc * 8, 1), "ms": round(ms, 3), "tb": 2,
        "note": "cell-updates/s of one fused 2-sweep launch (8 B/cell per launch)"}
    del a, bb
    # 1D (kernels.hpp:390-447): conv1d 9 taps and the one-pass scan over 2^28 elements
    # (1 GiB fp32, far above L2), HBM-bound at 2 * sizeof(T) bytes per element.
    n1 = 1 << 28
    for dt, tdt, npdt, sz in (("f32", torch.float32, np.float32, 4),
                              ("f64", torch.float64, np.float64, 8)):
        x = torch.empty(n1, dtype=tdt, device="cuda")
        dev.fill_random(x, 0)
        y = torch.empty_like(x)
        f = orc.random_filter(9, 1, npdt, 1).reshape(-1)
        for kname, fn in (("conv1d_m9", lambda: dev.conv1d(x, y, f)),
                          ("scan", lambda: dev.scan(x, y))):
            ms = timed(fn, 5)
            ge = n1 / ms / 1e6
            out[f"{kname}_{dt}_2^28"] = {"gelems": round(ge, 2), "hbm_gbs": round(ge * 2 * sz, 1),
                                         "hbm_frac": round(ge * 2 * sz / peak, 4),
                                         "ms": round(ms, 4)}
        del x, y
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--iters", type=int, default=100, help="sweeps per step")
    ap.add_argument("--tb", type=int, default=0,
                    help="temporal block depth of the headline sweeps: 0 = what the "
                         "product's ssam_b200_stencil3d_run uses for this stencil (2 for "
                         "3d7pt f32: fused sweep pairs), 1 = single sweeps")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--halo", choices=["nccl", "peer"], default="nccl",
                    help="N > 1 halo transport: NCCL send/recv, or the sweep kernel's own "
                         "stores into the neighbours' buffers (CUDA IPC / NVLink P2P)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-suite", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.tb <= 0:  # resolve once so both arms report the same config
        import numpy as np
        import paper_1907_06154_b200 as ssam
        from paper_1907_06154_b200 import device as dev
        st = ssam.convert_stencil(ssam.make_benchmark_stencil(STENCIL), np.float32)
        args.tb = dev.stencil3d_tb_max(st, np.float32)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE",
              file=sys.stderr)

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        dev_index = rank_device(local_rank)
        torch.cuda.set_device(dev_index)
        if backend() == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend())
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
