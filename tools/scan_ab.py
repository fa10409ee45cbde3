"""A/B of scan.cu variants: python tools/scan_ab.py lib.so ... (each in its own process)."""
import os, subprocess, sys
CODE = r'''
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1907_06154_b200 import device as dev
n = 1 << 28
out = []
for dt in (torch.float32, torch.float64):
    x = torch.empty(n, dtype=dt, device="cuda"); dev.fill_random(x, 0); y = torch.empty_like(x)
    for _ in range(3): dev.scan(x, y)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5): dev.scan(x, y)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    out.append(f"{str(dt)[6:]} {ms:.3f} ms {2*n*x.element_size()/ms/1e6:.0f} GB/s")
xi = torch.randint(-1000, 1000, (n + 12345,), dtype=torch.int64, device="cuda"); yi = torch.empty_like(xi)
dev.scan(xi, yi); out.append("int64 exact=" + str(bool(torch.equal(yi, torch.cumsum(xi, 0)))))
xf = torch.empty(n + 777, dtype=torch.float64, device="cuda"); dev.fill_random(xf, 1); yf = torch.empty_like(xf)
dev.scan(xf, yf); ref = torch.cumsum(xf, 0)
out.append("f64 max_abs=%.2e" % (yf - ref).abs().max().item())
print(" | ".join(out))
'''
for rep in range(2):
    for lib in sys.argv[1:]:
        r = subprocess.run([sys.executable, "-c", CODE], env=dict(os.environ, SSAM_B200_LIB=lib),
                           capture_output=True, text=True)
        print(lib, r.stdout.strip() or r.stderr[-400:], flush=True)
