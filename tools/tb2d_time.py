"""2D x100 runs at each temporal-block depth: python tools/tb2d_time.py"""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
H = W = 8192
for dt, tdt, npdt in (("f32", torch.float32, np.float32), ("f64", torch.float64, np.float64)):
    a = torch.empty((H, W), dtype=tdt, device="cuda"); dev.fill_random(a, 0); b = torch.empty_like(a)
    for name in ("2d5pt", "2d9pt"):
        st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), npdt)
        for tb in (1, 2, 4, 8):
            try:
                dev.stencil2d_run(a, b, st, 8, tb)
            except Exception:
                continue
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); dev.stencil2d_run(a, b, st, 100, tb); e.record(); torch.cuda.synchronize()
            ms = s.elapsed_time(e)
            print(f"{name} {dt} tb={tb}: {H*W*100/ms/1e6:.0f} GCells/s")
