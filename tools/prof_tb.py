import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
a = torch.empty((8192, 8192), dtype=torch.float32, device="cuda"); dev.fill_random(a, 0); b = a.clone()
st = ssam.convert_stencil(ssam.make_benchmark_stencil(sys.argv[1] if len(sys.argv) > 1 else "2d5pt"), np.float32)
for _ in range(3): dev.stencil2d_tb(a, b, st, 4)
torch.cuda.synchronize()
