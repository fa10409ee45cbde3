"""Device-set path overhead on ONE GPU: ssam_b200_stencil3d_multi with the
slabs sharing device 0 vs the one-device host-grid call, 3d7pt f32
2048 x 2048 x 512 x 100 sweeps (host grids in and out, pinned).  With one
GPU the slabs run one after another on it, so the ratio shows the cost of
the boundary bands and halo copies, not a speed-up."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import paper_1907_06154_b200 as ssam

st = ssam.convert_stencil(ssam.make_benchmark_stencil("3d7pt"), np.float32)
nz, ny, nx = 512, 2048, 2048
g = torch.empty((nz, ny, nx), dtype=torch.float32, pin_memory=True).numpy()
g[:] = ssam.random_grid3d(nx, ny, nz, 0, np.float32)
cfg = ssam.KernelConfig(p=2, b=128)
one = ssam.stencil3d(g, st, cfg, 100)  # warm-up
t0 = time.perf_counter()
one = ssam.stencil3d(g, st, cfg, 100)
t1 = time.perf_counter() - t0
cells = nx * ny * nz * 100
print(f"one device: {t1 * 1e3:.0f} ms  {cells / t1 / 1e9:.0f} GCells/s (incl. 8+8 GiB PCIe)")
for n in (2, 4):
    got, used = ssam.stencil_multi(g, st, [0] * n, cfg, 100)
    t0 = time.perf_counter()
    got, used = ssam.stencil_multi(g, st, [0] * n, cfg, 100)
    tn = time.perf_counter() - t0
    print(f"{used} slabs on device 0: {tn * 1e3:.0f} ms  {cells / tn / 1e9:.0f} GCells/s  "
          f"bit-identical={np.array_equal(got, one)}  ratio={t1 / tn:.3f}")
