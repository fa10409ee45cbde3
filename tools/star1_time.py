"""3d7pt single sweeps (GCells/s): python tools/star1_time.py"""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import numpy as np
import torch

import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
from pipe_check import timed

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
    ms = timed(lambda: dev.stencil3d_sweep(a, b, st), 10)
    out.append(f"{np.dtype(npdt).name}:{nx}x{nz}={(nx - 2) * (ny - 2) * (nz - 2) / ms / 1e6:.0f}")
    del a, b
    torch.cuda.empty_cache()
print(os.environ.get("SSAM_B200_STAR1_HALO", "-"), " ".join(out), flush=True)
