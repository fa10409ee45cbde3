"""3D pipeline engine (engine3d_pipe.cuh) check + timing on one GPU.

  python tools/pipe_check.py [check] [time] [quick] [shapes]

check: fused launches == TB single sweeps bit for bit, == the oracle within
tolerance, on odd shapes, for every shape and compiled depth; unaligned
grids (direct kernel) through stencil3d_run.
time: 2048^2 x 514 f32 (headline slab) single sweep and TB = 2/3/4, 512^3
f32/f64 x20 through stencil3d_run, in GCells/s (cell-updates, interior).
shapes: 512^3 f32/f64 of 3d13pt / 3d27pt / poisson at TB = 1, 2 and run x20.
"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
from oracle import Oracle, max_rel_err


TBS = {"3d7pt": (2, 3, 4), "3d13pt": (2,), "3d27pt": (2,), "poisson": (2,)}


def check():
    orc = Oracle()
    bad = 0
    for (dt, tol), name in [(d, n) for d in ((np.float32, 1e-5), (np.float64, 1e-12))
                            for n in TBS]:
        st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), dt)
        offs = [t.offset for t in st.taps]
        cf = np.asarray([t.coeff for t in st.taps], dt)
        k = st.order
        for (nx, ny, nz) in ((132, 70, 37), (256, 97, 80), (64, 19, 9), (520, 40, 150), (16, 5, 5)):
            if min(nx, ny, nz) < 2 * k + 1:
                continue
            g = orc.random_grid((nz, ny, nx), dt, 21)
            for tb in TBS[name]:
                a = torch.from_numpy(g).cuda()
                singles = [a]
                for _ in range(tb):
                    o = singles[-1].clone()
                    dev.stencil3d_sweep(singles[-1], o, st)
                    singles.append(o)
                f = a.clone()
                dev.stencil3d_tb(a, f, st, tb)
                same = torch.equal(f, singles[-1])
                want = orc.stencil3d(g, offs, cf, st.order, tb)
                e = max_rel_err(f.cpu().numpy(), want)
                ok = same and e <= tol
                bad += not ok
                print(f"{name} {np.dtype(dt).name} {nx}x{ny}x{nz} tb={tb}: bit-identical={same} "
                      f"max_rel={e:.3g} {'ok' if ok else 'FAIL'}", flush=True)
        # unaligned width -> direct kernel, and run3d (mixed fused/single)
        for (nx, ny, nz, iters) in ((131, 33, 21, 3), (128, 64, 40, 7), (130, 17, 30, 5)):
            g = orc.random_grid((nz, ny, nx), dt, 5)
            got = ssam.stencil3d(g, st, ssam.KernelConfig(p=2, b=max(128, 32 * (2 * k + 1))), iters)
            want = orc.stencil3d(g, offs, cf, st.order, iters)
            e = max_rel_err(got, want)
            ok = e <= tol
            bad += not ok
            print(f"{name} {np.dtype(dt).name} run {nx}x{ny}x{nz} x{iters}: max_rel={e:.3g} "
                  f"{'ok' if ok else 'FAIL'}", flush=True)
    print("CHECK", "FAIL" if bad else "OK", bad)


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def time_all():
    st32 = ssam.convert_stencil(ssam.make_benchmark_stencil("3d7pt"), np.float32)
    nz = 514
    a = torch.empty((nz, 2048, 2048), dtype=torch.float32, device="cuda")
    dev.fill_random(a, 0)
    b = a.clone()
    cells = 2046 * 2046 * (nz - 2)
    ms = timed(lambda: dev.stencil3d_sweep(a, b, st32), 10)
    print(f"2048^2x514 f32 tb=1: {ms:.3f} ms {cells / ms / 1e6:.1f} GCells/s "
          f"({cells * 8 / ms / 1e6:.0f} GB/s)", flush=True)
    for tb in (2, 3, 4):
        ms = timed(lambda: dev.stencil3d_tb(a, b, st32, tb), 10)
        print(f"2048^2x514 f32 tb={tb}: {ms:.3f} ms {tb * cells / ms / 1e6:.1f} GCells/s "
              f"(per-launch HBM {cells * 8 / ms / 1e6:.0f} GB/s)", flush=True)
    del a, b
    torch.cuda.empty_cache()
    n = 512
    for tdt, npdt in ((torch.float32, np.float32), (torch.float64, np.float64)):
        st = ssam.convert_stencil(ssam.make_benchmark_stencil("3d7pt"), npdt)
        a = torch.empty((n, n, n), dtype=tdt, device="cuda")
        dev.fill_random(a, 0)
        b = a.clone()
        ms = timed(lambda: dev.stencil3d_run(a, b, st, 20), 2)
        print(f"512^3 {np.dtype(npdt).name} run x20 (tb={dev.stencil3d_tb_max(st, npdt)}): "
              f"{ms:.3f} ms {n ** 3 * 20 / ms / 1e6:.1f} GCells/s", flush=True)
        for tb in (1, 2, 3, 4):
            fn = (lambda: dev.stencil3d_sweep(a, b, st)) if tb == 1 else \
                 (lambda: dev.stencil3d_tb(a, b, st, tb))
            ms = timed(fn, 10)
            print(f"512^3 {np.dtype(npdt).name} tb={tb}: {ms:.3f} ms "
                  f"{tb * 510 ** 3 / ms / 1e6:.1f} GCells/s", flush=True)
        del a, b
        torch.cuda.empty_cache()
    # f64 on the headline geometry (256 planes)
    st64 = ssam.convert_stencil(ssam.make_benchmark_stencil("3d7pt"), np.float64)
    nz = 258
    a = torch.empty((nz, 2048, 2048), dtype=torch.float64, device="cuda")
    dev.fill_random(a, 0)
    b = a.clone()
    cells = 2046 * 2046 * (nz - 2)
    for tb in (1, 2, 3, 4):
        fn = (lambda: dev.stencil3d_sweep(a, b, st64)) if tb == 1 else \
             (lambda: dev.stencil3d_tb(a, b, st64, tb))
        ms = timed(fn, 10)
        print(f"2048^2x258 f64 tb={tb}: {ms:.3f} ms {tb * cells / ms / 1e6:.1f} GCells/s", flush=True)


def quick():
    """TB=2 timings only (A/B of build variants): 2048^2x514 f32, 512^3 f32/f64, 2048^2x258 f64."""
    out = []
    for npdt, tdt, shape in ((np.float32, torch.float32, (514, 2048, 2048)),
                             (np.float32, torch.float32, (512, 512, 512)),
                             (np.float64, torch.float64, (512, 512, 512)),
                             (np.float64, torch.float64, (258, 2048, 2048))):
        st = ssam.convert_stencil(ssam.make_benchmark_stencil("3d7pt"), npdt)
        a = torch.empty(shape, dtype=tdt, device="cuda")
        dev.fill_random(a, 0)
        b = a.clone()
        nz, ny, nx = shape
        cells = (nx - 2) * (ny - 2) * (nz - 2)
        ms = timed(lambda: dev.stencil3d_tb(a, b, st, 2), 10)
        out.append(f"{np.dtype(npdt).name[0]}{np.dtype(npdt).itemsize * 8}:{nx}x{nz}={2 * cells / ms / 1e6:.0f}")
        del a, b
        torch.cuda.empty_cache()
    print(os.environ.get("SSAM_B200_LIB", "main"), " ".join(out), flush=True)


def shapes():
    """512^3 single sweeps / TB = 2 / stencil3d_run x20 of the heavier shapes."""
    n = 512
    for tdt, npdt in ((torch.float32, np.float32), (torch.float64, np.float64)):
        a = torch.empty((n, n, n), dtype=tdt, device="cuda")
        dev.fill_random(a, 0)
        b = a.clone()
        for name in ("3d7pt", "3d13pt", "3d27pt", "poisson"):
            st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), npdt)
            k = st.order
            cells = (n - 2 * k) ** 3
            line = [f"{name} {np.dtype(npdt).name}"]
            ms = timed(lambda: dev.stencil3d_sweep(a, b, st), 10)
            line.append(f"tb1={cells / ms / 1e6:.0f}")
            try:
                ms = timed(lambda: dev.stencil3d_tb(a, b, st, 2), 10)
                line.append(f"tb2={2 * cells / ms / 1e6:.0f}")
            except Exception as ex:  # no fused kernel for this shape
                line.append(f"tb2=n/a")
            ms = timed(lambda: dev.stencil3d_run(a, b, st, 20), 2)
            line.append(f"run20={n ** 3 * 20 / ms / 1e6:.0f} (tb={dev.stencil3d_tb_max(st, npdt)})")
            print(os.environ.get("SSAM_B200_PIPE", "pipe"), " ".join(line), flush=True)
        del a, b
        torch.cuda.empty_cache()


if __name__ == "__main__":
    what = sys.argv[1:] or ["check", "time"]
    if "check" in what:
        check()
    if "time" in what:
        time_all()
    if "quick" in what:
        quick()
    if "shapes" in what:
        shapes()
