"""Launch one kernel config a few times (for ncu captures): prof_one.py KIND [args]
   conv K | st2d NAME DT | st3d NAME DT N [NZ] | st3dtb NAME DT N [NZ [TB]] | conv1d M DT | scan DT"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
kind = sys.argv[1]
reps = 3
if kind == "conv":
    K = int(sys.argv[2]); H = W = 8192
    g = torch.empty((H, W), dtype=torch.float32, device="cuda"); dev.fill_random(g, 0)
    o = torch.empty_like(g)
    f = np.random.default_rng(1).uniform(-1, 1, (K, K)).astype(np.float32)
    for _ in range(reps): dev.conv2d(g, o, f)
elif kind in ("conv1d", "scan"):
    dt = sys.argv[-1]
    tdt, npdt = (torch.float32, np.float32) if dt == "f32" else (torch.float64, np.float64)
    x = torch.empty(1 << 28, dtype=tdt, device="cuda"); dev.fill_random(x, 0); y = torch.empty_like(x)
    if kind == "conv1d":
        f = np.random.default_rng(1).uniform(-1, 1, int(sys.argv[2])).astype(npdt)
        for _ in range(reps): dev.conv1d(x, y, f)
    else:
        for _ in range(reps): dev.scan(x, y)
elif kind == "st2dtb":
    name, dt, tb = sys.argv[2], sys.argv[3], int(sys.argv[4]); H = W = 8192
    tdt, npdt = (torch.float32, np.float32) if dt == "f32" else (torch.float64, np.float64)
    a = torch.empty((H, W), dtype=tdt, device="cuda"); dev.fill_random(a, 0); b = a.clone()
    st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), npdt)
    for _ in range(reps): dev.stencil2d_tb(a, b, st, tb)
elif kind == "st2d":
    name, dt = sys.argv[2], sys.argv[3]; H = W = 8192
    tdt, npdt = (torch.float32, np.float32) if dt == "f32" else (torch.float64, np.float64)
    a = torch.empty((H, W), dtype=tdt, device="cuda"); dev.fill_random(a, 0); b = a.clone()
    st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), npdt)
    for _ in range(reps): dev.stencil2d_sweep(a, b, st)
elif kind == "st3dtb":
    name, dt, n = sys.argv[2], sys.argv[3], int(sys.argv[4])
    nz = int(sys.argv[5]) if len(sys.argv) > 5 else n
    tb = int(sys.argv[6]) if len(sys.argv) > 6 else 2
    tdt, npdt = (torch.float32, np.float32) if dt == "f32" else (torch.float64, np.float64)
    a = torch.empty((nz, n, n), dtype=tdt, device="cuda"); dev.fill_random(a, 0); b = a.clone()
    st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), npdt)
    for _ in range(reps): dev.stencil3d_tb(a, b, st, tb)
else:
    name, dt, n = sys.argv[2], sys.argv[3], int(sys.argv[4])
    tdt, npdt = (torch.float32, np.float32) if dt == "f32" else (torch.float64, np.float64)
    nz = int(sys.argv[5]) if len(sys.argv) > 5 else n
    a = torch.empty((nz, n, n), dtype=tdt, device="cuda"); dev.fill_random(a, 0); b = a.clone()
    st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), npdt)
    for _ in range(reps): dev.stencil3d_sweep(a, b, st)
torch.cuda.synchronize()
