"""Time stencil3d_run (the C-ABI ping-pong loop, as bench's kernel suite does):
python tools/run3d_time.py NAME DT N ITERS"""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
name, dt, n, iters = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
tdt, npdt = (torch.float32, np.float32) if dt == "f32" else (torch.float64, np.float64)
a = torch.empty((n, n, n), dtype=tdt, device="cuda"); dev.fill_random(a, 0); b = a.clone()
st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), npdt)
dev.stencil3d_run(a, b, st, iters); torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(3):
    s.record(); dev.stencil3d_run(a, b, st, iters); e.record(); torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
print(name, dt, n, iters, f"{n**3 * iters / best / 1e6:.1f} GCells/s")
