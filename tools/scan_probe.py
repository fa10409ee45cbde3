import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1907_06154_b200 import device as dev
n = 1 << 28
for dt in (torch.float32, torch.float64, torch.int64):
    x = torch.empty(n, dtype=dt, device="cuda"); dev.fill_random(x, 0); y = torch.empty_like(x)
    for _ in range(3): dev.scan(x, y)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5): dev.scan(x, y)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(dt, os.environ.get("SSAM_B200_SCAN_NOLB"), f"{ms:.3f} ms  {2*n*x.element_size()/ms/1e6:.0f} GB/s")
    # copy reference
    s.record()
    for _ in range(5): y.copy_(x)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print("  copy", f"{ms:.3f} ms  {2*n*x.element_size()/ms/1e6:.0f} GB/s")
