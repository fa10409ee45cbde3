import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
name = sys.argv[1] if len(sys.argv) > 1 else "3d7pt"
n, nz = 2048, 514
a = torch.empty((nz, n, n), dtype=torch.float32, device="cuda"); dev.fill_random(a, 0); b = a.clone()
st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), np.float32)
dev.stencil3d_run(a, b, st, 4); torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); dev.stencil3d_run(a, b, st, 20); e.record(); torch.cuda.synchronize()
print(name, os.environ.get("SSAM_B200_3D_ZSEG", "auto"), round(n * n * nz * 20 / s.elapsed_time(e) / 1e6, 1), "GCells/s")
