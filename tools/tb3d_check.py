"""Fused Tb=2 3D sweeps vs two single sweeps (bit-identical) and timing.
   python tools/tb3d_check.py [nx ny nz]"""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev

dims = [int(v) for v in sys.argv[1:4]] if len(sys.argv) > 3 else [512, 512, 512]
nx, ny, nz = dims
for dt, tdt, npdt in (("f32", torch.float32, np.float32), ("f64", torch.float64, np.float64)):
    a = torch.empty((nz, ny, nx), dtype=tdt, device="cuda"); dev.fill_random(a, 3)
    for name in ("3d7pt", "poisson", "3d27pt"):
        st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), npdt)
        b = a.clone(); c = a.clone()
        dev.stencil3d_sweep(a, b, st); dev.stencil3d_sweep(b, c, st)  # two sweeps
        f = a.clone()
        try:
            dev.stencil3d_tb(a, f, st, 2)
        except Exception as ex:
            print(name, dt, "tb unavailable:", ex); continue
        torch.cuda.synchronize()
        same = torch.equal(f.view(torch.int32 if dt == "f32" else torch.int64),
                           c.view(torch.int32 if dt == "f32" else torch.int64))
        diff = (f.double() - c.double()).abs().max().item()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(2): dev.stencil3d_tb(a, f, st, 2)
        torch.cuda.synchronize(); s.record()
        for _ in range(5): dev.stencil3d_tb(a, f, st, 2)
        e.record(); torch.cuda.synchronize(); ms = s.elapsed_time(e) / 5
        s.record()
        for _ in range(5): dev.stencil3d_sweep(a, b, st)
        e.record(); torch.cuda.synchronize(); ms1 = s.elapsed_time(e) / 5
        print(f"{name} {dt} {nx}x{ny}x{nz}: bit-identical={same} maxdiff={diff:.3g}  "
              f"tb2 {2*nx*ny*nz/ms/1e6:.0f} GCells/s  vs single {nx*ny*nz/ms1/1e6:.0f}")
    del a
