"""A/B of tb2d.cu build variants: python tools/tb2d_ab.py lib1.so lib2.so ...
Each variant in a fresh process (SSAM_B200_LIB), interleaved twice."""
import os
import subprocess
import sys

CODE = r'''
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
H = W = 8192
out = []
for dt, tdt, npdt in (("f32", torch.float32, np.float32), ("f64", torch.float64, np.float64)):
    a = torch.empty((H, W), dtype=tdt, device="cuda"); dev.fill_random(a, 0); b = torch.empty_like(a)
    for name, tb in (("2d5pt", 4), ("2d9pt", 2)):
        st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), npdt)
        dev.stencil2d_run(a, b, st, 8, tb); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); dev.stencil2d_run(a, b, st, 100, tb); e.record(); torch.cuda.synchronize()
        out.append(f"{name}/{dt}/tb{tb}={H*W*100/s.elapsed_time(e)/1e6:.0f}")
print(" ".join(out))
'''
for rep in range(2):
    for lib in sys.argv[1:]:
        env = dict(os.environ, SSAM_B200_LIB=lib)
        r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
        print(lib, r.stdout.strip() or r.stderr[-500:], flush=True)
