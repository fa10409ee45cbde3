"""2D stencils x100 on 8192^2 (GCells/s): python tools/st2d_time.py [names...]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev

names = sys.argv[1:] or ["2d17pt", "2d21pt", "2ds25pt", "2d121pt"]
H = W = 8192
out = []
for dt, tdt, npdt in (("f32", torch.float32, np.float32), ("f64", torch.float64, np.float64)):
    a = torch.empty((H, W), dtype=tdt, device="cuda")
    dev.fill_random(a, 0)
    b = torch.empty_like(a)
    for name in names:
        st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), npdt)
        dev.stencil2d_run(a, b, st, 4)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        dev.stencil2d_run(a, b, st, 100)
        e.record()
        torch.cuda.synchronize()
        out.append(f"{name}/{dt}={H * W * 100 / s.elapsed_time(e) / 1e6:.0f}")
print(os.environ.get("SSAM_B200_ST2D_REG", "-"), " ".join(out), flush=True)
