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
          (ssam_b200_stencil_batch on the 512-plane grid at N=1, bit-compared
          with the device-resident result; the slab runner at N>1): pinned
          host->device copy of each step's input, the sweeps, and the
          device->host copy of its result inside the timed region.
  roofline  the dominant kernel (pipe3d_kernel, TB fused sweeps per launch):
          algorithmic bytes (4 B read + 4 B write per interior cell per
          launch) / mean launch time; traffic from ncu on this build.
  parity  every cell of one step (100 sweeps) at N=1 against the
          direct-gather kernels (the oracle's arithmetic on the GPU):
          max_rel / max_abs.
  kernels per-kernel GCells/s and %-of-peak for the other configs (conv
          sweep 3x3..20x20, 2D stencils x100 sweeps, 3D stencils at 512^3),
          rank 0 at N=1.
  cpu_baseline  the reference's own CPU path (oracle/_ref, ssam::stencil3d)
          on bounded samples of the same workload: every host thread and threads=1,
          best of 3 each.

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


CPU_BLOCK_NZ = 16     # planes of the all-threads sample block (14 of them updated per sweep)
CPU_BLOCK1_NZ = 4     # planes of the threads=1 sample block (2 updated)


def _ref_block(nz: int):
    """A 2048 x 2048 x nz block of the workload's seeded grid (global planes
    0..nz-1) and the reference's own 3d7pt stencil, for the CPU path."""
    import numpy as np
    from oracle import Oracle, Reference
    ref = Reference()
    st = ref.benchmark_stencil(STENCIL)
    g = Oracle().random_grid((nz, NY, NX), np.float32, 0)
    return ref, st, g, st["coeffs"].astype(np.float32)


def host_threads() -> int:
    """Every host thread, passed to the reference as KernelConfig::threads
    (kernels.hpp:42-45 num_threads): torchrun exports OMP_NUM_THREADS=1,
    which would otherwise pin threads=0 to one core."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return os.cpu_count() or 1


def _ref_sweep_seconds(ref, st, g, cf, threads: int) -> float:
    t0 = time.perf_counter()
    rc, _, _ = ref.stencil3d(g, st["offsets"], cf, st["order"], 1, p=2, b=128, threads=threads)
    assert rc == 0
    return time.perf_counter() - t0


def reference_sample(seconds: float = 10.0):
    """The reference's own CPU SSAM path (ssam::stencil3d from oracle/_ref,
    -O3 -fopenmp) on bounded samples of the workload, best of 3 as
    proj/tools/threads_bench.cpp:25-35 times it: every host thread (threads = the
    host thread count) on a 2048x2048x16 block and threads=1 on a 2048x2048x4 block.
    The rate counts the cells of the planes a sweep advances (nz - 2 planes
    of 2048 x 2048), the same W*H-per-plane convention as the GPU value."""
    ref, st, g, cf = _ref_block(CPU_BLOCK_NZ)
    upd = (CPU_BLOCK_NZ - 2) * NX * NY
    nall = host_threads()
    best = min(_ref_sweep_seconds(ref, st, g, cf, nall) for _ in range(3))
    ref1, st1, g1, cf1 = _ref_block(CPU_BLOCK1_NZ)
    upd1 = (CPU_BLOCK1_NZ - 2) * NX * NY
    best1 = min(_ref_sweep_seconds(ref1, st1, g1, cf1, 1) for _ in range(3))
    return {
        "value": round(upd / best / 1e9, 6), "unit": "GCells/s", "cores": nall,
        "kind": "reference",
        "sample": (f"best of 3 single sweeps of ssam::stencil3d<float> 3d7pt (oracle/_ref, "
                   f"threads={nall}, every host thread) on global planes 0..{CPU_BLOCK_NZ - 1} "
                   f"of the seed-0 grid ({NX}x{NY}x{CPU_BLOCK_NZ}; {CPU_BLOCK_NZ - 2} planes "
                   f"updated per sweep, counted as {CPU_BLOCK_NZ - 2}*{NX}*{NY} cells)"),
        "threads1": {"value": round(upd1 / best1 / 1e9, 6), "unit": "GCells/s", "cores": 1,
                     "sample": (f"best of 3 single sweeps, threads=1, {NX}x{NY}x{CPU_BLOCK1_NZ} "
                                f"block ({CPU_BLOCK1_NZ - 2} planes updated)")},
        "cpu_model": cpu_model(), "nproc": os.cpu_count()}


def run_reference_arm(args, rank: int, world: int):
    """--impl reference: the reference's own CPU path only (oracle/_ref via
    oracle/__init__.py); the product library is never loaded here."""
    if rank != 0:
        return
    ref, st, g, cf = _ref_block(CPU_BLOCK_NZ)
    upd = (CPU_BLOCK_NZ - 2) * NX * NY
    nall = host_threads()
    for _ in range(args.warmup):
        _ref_sweep_seconds(ref, st, g, cf, nall)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        _ref_sweep_seconds(ref, st, g, cf, nall)
    dt = time.perf_counter() - t0
    value = upd * args.steps / dt / 1e9
    sample = (f"each step: 1 sweep of ssam::stencil3d<float> 3d7pt (oracle/_ref, threads={nall}, "
              f"every host thread) on global planes 0..{CPU_BLOCK_NZ - 1} of the seed-0 "
              f"workload grid ({CPU_BLOCK_NZ - 2} planes of {NX}x{NY} updated and counted)")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "GCells/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(world, args),
        "cpu_baseline": {"value": round(value, 6), "unit": "GCells/s",
                         "cores": nall, "kind": "reference", "sample": sample,
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
    """The workload (identical for both arms); engine choices are reported
    separately under "engine"."""
    return {"workload": f"{STENCIL} f32 {NX}x{NY}x({NZ_PER_GPU}*N) z-slab, NVLink halo exchange",
            "stencil": STENCIL, "nx": NX, "ny": NY, "nz": NZ_PER_GPU * world,
            "nz_per_gpu": NZ_PER_GPU, "iters_per_step": args.iters,
            "parallelism": f"z-slab x{world}", "seed": 0,
            "l2": "no flush needed: 8 GiB per buffer >> 126 MB L2"}


def engine_config(world: int, args, tb: int):
    return {"temporal_block": tb,
            "temporal_blocking": ("each launch of pipe3d_kernel fuses temporal_block sweeps (one "
                                  "HBM pass, bit-identical to single sweeps), as "
                                  "ssam_b200_stencil3d_run does for this stencil; --tb 1 times "
                                  "single sweeps"),
            "halo": ("kernel stores into neighbours' CUDA IPC buffers (peer.py)"
                     if args.halo == "peer" and world > 1 else
                     "boundary planes first, NCCL send/recv overlapped with the interior")}


def measure_traffic(tb: int, timeout: float = 240.0):
    """dram__bytes_read.sum + dram__bytes_write.sum of one dominant-kernel
    launch on the headline slab, from ncu run on THIS build (a subprocess:
    the number is traffic only, never a timing)."""
    import csv
    import shutil
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None, "ncu not found"
    kind = ["st3dtb", STENCIL, "f32", str(NX), str(NZ_PER_GPU + 2 * tb), str(tb)] if tb > 1 \
        else ["st3d", STENCIL, "f32", str(NX), str(NZ_PER_GPU + 2)]
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--csv", "-k", "regex:pipe3d", "-s", "1", "-c", "1", sys.executable,
           os.path.join(ROOT, "tools", "prof_one.py")] + kind
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout).stdout
    except Exception as ex:
        return None, f"ncu failed: {type(ex).__name__}"
    vals = {}
    for row in csv.reader(out.splitlines()):
        if len(row) > 3 and row[-3] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(row[-2], None)
            try:
                vals[row[-3]] = float(row[-1].replace(",", "")) * (scale or 1)
            except ValueError:
                pass
    if len(vals) != 2:
        return None, "ncu output not parsed"
    return int(vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]), \
        f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum, {' '.join(kind)}"


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
    # --tb 0: the depth the product's ssam_b200_stencil3d_run uses for this stencil
    tb = args.tb if args.tb > 0 else dev.stencil3d_tb_max(st, np.float32)
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
    lo, hi = slab.compute_range()
    rlo, rhi = slab.ring_bounds()

    def timed_launch(fn, zb):
        if timing["on"] and zb == lo and world == 1:
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            launch_ms.append((s, e))
        else:
            fn()

    def sweep(cur, nxt, zb, ze):
        if ze > zb:
            timed_launch(lambda: dev.stencil3d_sweep(cur, nxt, st, zb, ze), zb)

    def fused(cur, nxt, zb, ze):
        if ze > zb:
            timed_launch(lambda: dev.stencil3d_tb(cur, nxt, st, tb, zb, ze, rlo, rhi), zb)

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

    # dominant kernel: one launch over the whole slab (N=1 timing by launch)
    interior = (NX - 2 * k) * (NY - 2 * k)
    cells_per_launch = interior * (hi - lo)
    fused_launches = [(s_, e_) for s_, e_ in launch_ms]
    if fused_launches:
        durs = [s_.elapsed_time(e_) for s_, e_ in fused_launches]
        # a run of iters % tb trailing single sweeps is not the dominant kernel
        if tb > 1 and args.iters % tb:
            per_step = args.iters // tb + args.iters % tb
            durs = [d for i, d in enumerate(durs) if i % per_step < args.iters // tb]
        mean_ms = sum(durs) / len(durs)
    else:
        mean_ms = max_ms / (args.steps * max(1, args.iters // tb))
    # a launch reads and writes every cell once for its tb updates
    achieved = 8.0 * cells_per_launch / (mean_ms / 1e3) / 1e9

    # ---- per-cell parity of one step at N=1 (the product run vs the
    # direct-gather kernels, the oracle's order and arithmetic on the GPU)
    parity = None
    ref_result = None
    if world == 1 and not args.no_parity:
        fill_slab(a, slab, NX, NY, seed=0)
        b.copy_(a)
        res = runner.run(a, b, args.iters)
        g0 = torch.empty((NZ_PER_GPU, NY, NX), dtype=torch.float32, device="cuda")
        dev.fill_random(g0, 0)
        g1 = torch.empty_like(g0)
        want = dev.gather_run(g0, g1, st, args.iters)
        got = res[slab.local(0):slab.local(0) + NZ_PER_GPU]
        rel, ab = dev.max_rel_err(got, want)
        torch.cuda.synchronize()
        parity = {"max_rel": rel, "max_abs": ab, "tolerance": 1e-5, "pass": rel <= 1e-5,
                  "cells": NX * NY * NZ_PER_GPU, "iters": args.iters,
                  "vs": "ssam_b200_gather_stencil_run (one thread per cell, the oracle's tap "
                        "order in double, oracle.hpp:77-116) on the full grid, every cell"}
        ref_result = got.clone()
        del g0, g1, want, got, res

    # free the slab before the e2e / per-kernel phases
    del a, b
    if peer:
        prun.close()
    torch.cuda.empty_cache()

    e2e = None
    if not args.no_e2e:
        try:
            e2e = e2e_run(args, slab, st, world, rank, tb, ref_result)
        except Exception as ex:  # e.g. pinned host memory exhausted on a big box
            e2e = {"value": None, "unit": "GCells/s", "error": f"{type(ex).__name__}: {ex}"[:300]}
            torch.cuda.empty_cache()
    del ref_result
    ssam.lib.ssam_b200_trim_cache()
    torch.cuda.empty_cache()

    kernels = None
    cpu = None
    if rank == 0 and world == 1 and not args.no_suite:
        kernels = kernel_suite(peak, sm_max_nominal)
    if rank == 0 and not args.no_cpu:
        try:
            cpu = reference_sample()
        except Exception as ex:  # the reference build may be absent
            cpu = {"value": None, "unit": "GCells/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {ex}"}
    traffic, traffic_how = None, "skipped (--no-traffic)"
    if rank == 0 and not args.no_traffic:
        traffic, traffic_how = measure_traffic(tb)
    if world > 1:
        barrier()

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GCells/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(max_ms / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference SplitMix64 stream, seed 0, generated on device)",
            "config": workload_config(world, args),
            "engine": engine_config(world, args, tb),
            "hbm_gbs_algorithmic": round(value * 8.0 / tb, 1),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic, "traffic_how": traffic_how, "peak_kind": peak_kind,
                         "kernel": (f"pipe3d_kernel<float, PipeStar<1>, TB={tb}> {STENCIL} (8 B per interior "
                                    f"cell per launch = {tb} updates)"),
                         "bytes_per_launch": 8 * cells_per_launch,
                         "mean_launch_ms": round(mean_ms, 4)},
            "parity": parity,
            "max_rel": parity["max_rel"] if parity else None,
            "max_abs": parity["max_abs"] if parity else None,
            "e2e": e2e, "gpu_launches": int(n_launches), "clocks": clk,
            "cpu_baseline": cpu, "kernels": kernels,
        }
        print(json.dumps(line), flush=True)


def e2e_run(args, slab, st, world, rank, tb, ref_result):
    """Public-API end to end: pinned host input -> GPU -> host output per step.

    N = 1: the C ABI on the 512-plane global grid (not the ghost-padded
    slab).  Headline: ssam_b200_stencil_batch over `--e2e-steps` steps (each
    step's H2D, sweeps and D2H on their own streams, so step k+1's input
    copy and step k-1's result copy run under step k's sweeps); also the
    one-call-per-step ssam_b200_stencil3d number.  The result is compared
    bit for bit with the device-resident run's.
    N > 1: the slab runner with host buffers."""
    import ctypes
    import numpy as np
    import torch
    import paper_1907_06154_b200 as ssam
    from paper_1907_06154_b200.slab import SlabRunner, fill_slab
    from paper_1907_06154_b200 import device as dev

    steps = max(1, args.e2e_steps)
    if world == 1:
        shape = (NZ_PER_GPU, NY, NX)
        host_in = torch.empty(shape, dtype=torch.float32, pin_memory=True)
        depth = 3  # grids in flight: H2D of k+1, sweeps of k, D2H of k-1 (2 x 8 GiB each)
        outs = [torch.empty(shape, dtype=torch.float32, pin_memory=True) for _ in range(depth)]
        tmp = torch.empty(shape, dtype=torch.float32, device="cuda")
        dev.fill_random(tmp, 0)
        host_in.copy_(tmp)
        del tmp
        torch.cuda.empty_cache()
        cfg = ssam.KernelConfig(p=2, b=128)._c()
        sa = ssam._StencilArgs(st, np.float32)
        nbytes = host_in.numel() * 4

        def single():
            ssam._raise(ssam.lib.ssam_b200_stencil3d(
                0, host_in.data_ptr(), NX, NY, NZ_PER_GPU, sa.ref, ctypes.byref(cfg), args.iters,
                outs[0].data_ptr(), None))

        single()  # warm-up (pool allocation, first touch of pinned pages)
        same = None
        if ref_result is not None:
            chk = outs[0].to("cuda", non_blocking=False)
            same = bool(torch.equal(chk, ref_result))
            del chk
            torch.cuda.empty_cache()
        steps1 = min(steps, 4)  # the one-call-per-step number is a side figure
        t0 = time.perf_counter()
        for _ in range(steps1):
            single()
        dt1 = time.perf_counter() - t0

        def batch(n):
            ssam.stencil_batch([host_in] * n, [outs[i % depth] for i in range(n)], st, args.iters,
                               depth=depth)

        batch(depth)  # warm-up of the batch buffers
        t0 = time.perf_counter()
        batch(steps)
        dtb = time.perf_counter() - t0
        same_b = None
        if ref_result is not None:
            chk = outs[(steps - 1) % depth].to("cuda", non_blocking=False)
            same_b = bool(torch.equal(chk, ref_result))
            del chk
        cells = NX * NY * NZ_PER_GPU * args.iters * steps
        return {"value": round(cells / dtb / 1e9, 3), "unit": "GCells/s",
                "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "steps": steps,
                "ms_per_step": round(dtb / steps * 1e3, 3),
                "api": ("ssam_b200_stencil_batch (C ABI, pinned host grids, copies of "
                        "neighbouring steps overlapped with each step's sweeps)"),
                "bit_identical_to_device_run": same_b,
                "single_call": {"value": round(cells / steps * steps1 / dt1 / 1e9, 3),
                                "unit": "GCells/s", "steps": steps1,
                                "ms_per_step": round(dt1 / steps1 * 1e3, 3),
                                "api": "ssam_b200_stencil3d (C ABI, one synchronous call per step)",
                                "bit_identical_to_device_run": same}}

    import torch.distributed as dist
    nzl = slab.nz_local
    host_in = torch.empty((nzl, NY, NX), dtype=torch.float32, pin_memory=True)
    host_out = torch.empty((nzl, NY, NX), dtype=torch.float32, pin_memory=True)
    tmp = torch.empty((nzl, NY, NX), dtype=torch.float32, device="cuda")
    fill_slab(tmp, slab, NX, NY, seed=0)
    host_in.copy_(tmp)
    del tmp
    torch.cuda.empty_cache()
    rlo, rhi = slab.ring_bounds()
    # Two slabs in flight per rank, as the one-GPU batch API does: step k+1's
    # H2D and step k-1's D2H run on their own streams under step k's sweeps
    # (host buffers reused: one input, one output per rank).
    depth = 2
    slots = [(torch.empty((nzl, NY, NX), dtype=torch.float32, device="cuda"),
              torch.empty((nzl, NY, NX), dtype=torch.float32, device="cuda")) for _ in range(depth)]
    s_in, s_comp, s_out, comm = (torch.cuda.Stream() for _ in range(4))
    ev_in = [torch.cuda.Event() for _ in range(depth)]
    ev_done = [torch.cuda.Event() for _ in range(depth)]
    ev_out = [torch.cuda.Event() for _ in range(depth)]
    runner = SlabRunner(
        slab, lambda c, n, zb, ze: dev.stencil3d_sweep(c, n, st, zb, ze), comm_stream=comm,
        fused=(lambda c, n, zb, ze: dev.stencil3d_tb(c, n, st, tb, zb, ze, rlo, rhi))
        if tb > 1 else None, tb=tb)

    def batch(n):
        for k in range(n):
            sl = k % depth
            a, b = slots[sl]
            if k >= depth:
                s_in.wait_event(ev_out[sl])
            with torch.cuda.stream(s_in):
                a.copy_(host_in, non_blocking=True)
                ev_in[sl].record(s_in)
            s_comp.wait_event(ev_in[sl])
            with torch.cuda.stream(s_comp):
                b.copy_(a)
                res = runner.run(a, b, args.iters)
                ev_done[sl].record(s_comp)
            s_out.wait_event(ev_done[sl])
            with torch.cuda.stream(s_out):
                host_out.copy_(res, non_blocking=True)
                ev_out[sl].record(s_out)
        torch.cuda.synchronize()

    batch(depth)
    dist.barrier()
    t0 = time.perf_counter()
    batch(steps)
    dt = time.perf_counter() - t0
    dt = reduce_host(dt, "max")
    cells = NX * NY * NZ_PER_GPU * world * args.iters * steps
    nbytes = nzl * NY * NX * 4
    return {"value": round(cells / dt / 1e9, 3), "unit": "GCells/s",
            "h2d_bytes_per_step": nbytes * world, "d2h_bytes_per_step": nbytes * world,
            "steps": steps, "ms_per_step": round(dt / steps * 1e3, 3),
            "api": ("SlabRunner over ssam_b200_stencil3d_sweep / _tb (host slabs, two in "
                    "flight per rank: copies of neighbouring steps under each step's sweeps)")}


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
    # FP32 peak at the clock the SMs actually ran during the sweep (power cap)
    csamp = ClockSampler(torch.cuda.current_device())
    csamp.start()
    time.sleep(0.3)  # nvidia-smi's first sample
    conv = {}
    for K in range(3, 21):
        f = orc.random_filter(K, K, np.float32, 1)
        ms = timed(lambda: dev.conv2d(g, o, f), 20)
        conv[K] = ms
    clk = csamp.stop()
    run_mhz = clk.get("sm_mhz") or sm_mhz
    peak_at_clock = 148 * 128 * 2 * run_mhz * 1e6 / 1e12
    for K, ms in conv.items():
        gc = H * W / ms / 1e6
        out[f"conv2d_f32_8192_{K}x{K}"] = {
            "gcells": round(gc, 2), "hbm_gbs": round(gc * 8, 1),
            "hbm_frac": round(gc * 8 / peak, 4), "tflops": round(gc * 2 * K * K / 1e3, 2),
            "fp32_frac": round(gc * 2 * K * K / 1e3 / fp32_peak_tflops, 4),
            "fp32_frac_at_clock": round(gc * 2 * K * K / 1e3 / peak_at_clock, 4),
            "sm_mhz": run_mhz, "ms": round(ms, 4)}
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
    # the headline slab: single sweeps and the product's fused depth (engine3d_pipe.cuh)
    a = torch.empty((NZ_PER_GPU + 2, NY, NX), dtype=torch.float32, device="cuda")
    dev.fill_random(a, 0)
    bb = a.clone()
    st = ssam.convert_stencil(ssam.make_benchmark_stencil("3d7pt"), np.float32)
    ms1 = timed(lambda: dev.stencil3d_sweep(a, bb, st), 5)
    gc1 = (NX - 2) * (NY - 2) * NZ_PER_GPU / ms1 / 1e6
    out[f"stencil3d_3d7pt_f32_{NX}x{NY}x{NZ_PER_GPU + 2}_tb1"] = {
        "gcells": round(gc1, 2), "hbm_gbs": round(gc1 * 8, 1),
        "hbm_frac": round(gc1 * 8 / peak, 4), "ms": round(ms1, 3), "tb": 1,
        "note": "one sweep per launch (ssam3d_halo_kernel, the pipeline's per-cell chain), 8 B/cell"}
    for tbk in sorted({2, dev.stencil3d_tb_max(st, np.float32)} - {1}):
        ms = timed(lambda: dev.stencil3d_tb(a, bb, st, tbk), 5)
        gc = tbk * (NX - 2) * (NY - 2) * NZ_PER_GPU / ms / 1e6
        out[f"stencil3d_3d7pt_f32_{NX}x{NY}x{NZ_PER_GPU + 2}_tb{tbk}"] = {
            "gcells": round(gc, 2), "hbm_gbs": round(gc * 8 / tbk, 1),
            "hbm_frac": round(gc * 8 / tbk / peak, 4), "hbm_gbs_equiv": round(gc * 8, 1),
            "ms": round(ms, 3), "tb": tbk,
            "note": f"cell-updates/s of one fused {tbk}-sweep launch (8 B/cell per launch)"}
    del a, bb
    # 1D (kernels.hpp:390-447): conv1d 9 taps and the chunked two-pass scan over 2^28 elements
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
                         "product's ssam_b200_stencil3d_run uses for this stencil, "
                         "1 = single sweeps")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--halo", choices=["nccl", "peer"], default="nccl",
                    help="N > 1 halo transport: NCCL send/recv, or the sweep kernel's own "
                         "stores into the neighbours' buffers (CUDA IPC / NVLink P2P)")
    ap.add_argument("--e2e-steps", type=int, default=24)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-suite", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-traffic", action="store_true")
    args = ap.parse_args()

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
        # NCCL's init log (stderr) shows the rank count and the NVLink transport
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
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
