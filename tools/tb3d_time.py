"""Time the fused Tb=2 kernel on the headline slab: python tools/tb3d_time.py [nz] [f32|f64]"""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
nz = int(sys.argv[1]) if len(sys.argv) > 1 else 514
f64 = len(sys.argv) > 2 and sys.argv[2] == "f64"
a = torch.empty((nz, 2048, 2048), dtype=torch.float64 if f64 else torch.float32, device="cuda"); dev.fill_random(a, 0)
b = a.clone()
st = ssam.convert_stencil(ssam.make_benchmark_stencil("3d7pt"), np.float64 if f64 else np.float32)
for _ in range(3): dev.stencil3d_tb(a, b, st, 2)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): dev.stencil3d_tb(a, b, st, 2)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print(os.environ.get("SSAM_B200_3D_TB_ZSEG", "default"), "f64" if f64 else "f32", f"{ms:.3f} ms  {2*2046*2046*(nz-2)/ms/1e6:.0f} GCells/s")
