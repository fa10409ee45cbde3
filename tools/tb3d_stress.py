"""Repeat the fused Tb=2 3D kernel many times against two single sweeps (race hunting)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
bad = 0
for (nx, ny, nz) in ((2048, 2048, 66), (516, 300, 200), (132, 70, 37)):
    for name in ("3d7pt", "poisson"):
        st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), np.float32)
        a = torch.empty((nz, ny, nx), dtype=torch.float32, device="cuda"); dev.fill_random(a, 5)
        b, c = a.clone(), a.clone()
        dev.stencil3d_sweep(a, b, st); dev.stencil3d_sweep(b, c, st)
        for rep in range(30):
            f = a.clone()
            dev.stencil3d_tb(a, f, st, 2)
            if not torch.equal(f, c):
                bad += 1
                print("MISMATCH", name, nx, ny, nz, rep, (f - c).abs().max().item())
        del a, b, c
print("stress done, mismatches:", bad)
