"""A/B of conv1d.cu variants: python tools/conv1d_ab.py lib.so ... (each in its own process).
GB/s = 2n bytes / time at n = 2^28; 'sum' is a float64 digest of one output to compare builds."""
import os, subprocess, sys
CODE = r'''
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1907_06154_b200 import device as dev
n = 1 << 28
out = []
for dt in (torch.float32, torch.float64):
    x = torch.empty(n, dtype=dt, device="cuda"); dev.fill_random(x, 0); y = torch.empty_like(x)
    for m in (3, 9, 32):
        w = np.linspace(-1, 1, m)
        for _ in range(3): dev.conv1d(x, y, w)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5): dev.conv1d(x, y, w)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 5
        dig = float(y.double().mul(torch.arange(n, device="cuda", dtype=torch.float64) % 977).sum())
        out.append(f"{str(dt)[6:]} m{m} {ms:.3f} ms {2*n*x.element_size()/ms/1e6:.0f} GB/s sum={dig:.17g}")
print(" | ".join(out))
'''
for rep in range(2):
    for lib in sys.argv[1:]:
        r = subprocess.run([sys.executable, "-c", CODE], env=dict(os.environ, SSAM_B200_LIB=lib),
                           capture_output=True, text=True)
        print(lib, r.stdout.strip() or r.stderr[-400:], flush=True)
