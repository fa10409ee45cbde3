"""Small invocations of every kernel family for compute-sanitizer runs."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev

def grid(shape, dt=torch.float32, seed=1):
    a = torch.empty(shape, dtype=dt, device="cuda"); dev.fill_random(a, seed); return a

g = grid((96, 260)); o = torch.empty_like(g)
for K in (3, 7, 13, 20):
    dev.conv2d(g, o, np.ones((K, K), np.float32) / K)
a = grid((70, 132)); b = a.clone()
for name in ("2d5pt", "2d9pt", "2ds25pt", "2d121pt"):
    st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), np.float32)
    dev.stencil2d_sweep(a, b, st)
st = ssam.convert_stencil(ssam.make_benchmark_stencil("2d5pt"), np.float32)
dev.stencil2d_tb(a, b, st, 4)
a3 = grid((20, 40, 132)); b3 = a3.clone()
for name in ("3d7pt", "3d13pt", "3d27pt", "poisson"):
    st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), np.float32)
    dev.stencil3d_sweep(a3, b3, st)
st = ssam.convert_stencil(ssam.make_benchmark_stencil("3d7pt"), np.float32)
dev.stencil3d_tb(a3, b3, st, 2)
# star arms from shared memory (K >= 5), f32 and f64; 3D single-chain shapes; fp64 fused pair
for dt, npdt in ((torch.float32, np.float32), (torch.float64, np.float64)):
    a = grid((70, 132), dt); b = a.clone()
    for name in ("2d17pt", "2d21pt", "2ds25pt"):
        dev.stencil2d_sweep(a, b, ssam.convert_stencil(ssam.make_benchmark_stencil(name), npdt))
    a3 = grid((12, 24, 68), dt); b3 = a3.clone()
    for name in ("3d13pt", "poisson"):
        dev.stencil3d_sweep(a3, b3, ssam.convert_stencil(ssam.make_benchmark_stencil(name), npdt))
    dev.stencil3d_tb(a3, b3, ssam.convert_stencil(ssam.make_benchmark_stencil("3d7pt"), npdt), 2)
x = grid(100003); y = torch.empty_like(x)
dev.conv1d(x, y, np.ones(9, np.float32)); dev.scan(x, y)
for dt in (torch.float64, torch.int64):
    x = grid(70001, dt); y = torch.empty_like(x)
    dev.scan(x, y)
# the chunked scan across several L2 chunks (384 tiles) and a ragged tail
for dt, per in ((torch.float32, 8192), (torch.int64, 4096)):
    x = grid(1025 * per + 517, dt)
    y = torch.empty_like(x)
    dev.scan(x, y)
torch.cuda.synchronize()
print("sanitize workload done")
