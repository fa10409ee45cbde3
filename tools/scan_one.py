import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1907_06154_b200 import device as dev
n = 1 << 28
for dt in (torch.float32, torch.float64):
    x = torch.empty(n, dtype=dt, device="cuda"); dev.fill_random(x, 0); y = torch.empty_like(x)
    dev.scan(x, y); torch.cuda.synchronize()
