"""scan A/B under sustained load: python tools/scan_hot_ab.py lib.so ...
Each build in its own process: ~8 s of the headline-class 3D sweeps to bring
the GPU to its power-capped clock, then 2^28 fp32 / fp64 scans timed as the
bench suite does (2 warm-up calls, 5 timed)."""
import os, subprocess, sys
CODE = r'''
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
a = torch.empty((512, 1024, 1024), dtype=torch.float32, device="cuda"); dev.fill_random(a, 0)
b = a.clone()
st = ssam.convert_stencil(ssam.make_benchmark_stencil("3d7pt"), np.float32)
t0 = time.time()
while time.time() - t0 < 8:
    for _ in range(20): dev.stencil3d_tb(a, b, st, 2, 2, 510, 1, 511); a, b = b, a
    torch.cuda.synchronize()
del a, b; torch.cuda.empty_cache()
n = 1 << 28
out = []
for dt in (torch.float32, torch.float64):
    x = torch.empty(n, dtype=dt, device="cuda"); dev.fill_random(x, 0); y = torch.empty_like(x)
    for _ in range(2): dev.scan(x, y)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5): dev.scan(x, y)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    out.append(f"{str(dt)[6:]} {ms:.3f} ms {2*n*x.element_size()/ms/1e6:.0f} GB/s")
print(" | ".join(out))
'''
for rep in range(2):
    for lib in sys.argv[1:]:
        r = subprocess.run([sys.executable, "-c", CODE], env=dict(os.environ, SSAM_B200_LIB=lib),
                           capture_output=True, text=True)
        print(lib, r.stdout.strip() or r.stderr[-600:], flush=True)
