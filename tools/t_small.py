import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1907_06154_b200 import device as dev
K = int(sys.argv[1]); H = W = int(sys.argv[2]) if len(sys.argv) > 2 else 512
g = torch.empty((H, W), dtype=torch.float32, device="cuda"); dev.fill_random(g, 0)
o = torch.empty_like(g)
f = np.random.default_rng(1).uniform(-1, 1, (K, K)).astype(np.float32)
dev.conv2d(g, o, f); torch.cuda.synchronize(); print("ok", K, float(o.abs().sum()))
