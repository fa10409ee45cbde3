import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1907_06154_b200 import device as dev
from oracle import Oracle, max_rel_err
sys.path.insert(0, "tests")
from windows import conv2d_rows
orc = Oracle()
H = W = 8192
g = orc.random_grid((H, W), np.float32, 0)
gt = torch.from_numpy(g).cuda(); o = torch.empty_like(gt)
for K in (6, 8, 10, 12):
    f = orc.random_filter(K, K, np.float32, 1)
    dev.conv2d(gt, o, f)
    got = o.cpu().numpy()
    worst = 0
    for y0 in (0, 4000, 8192 - 64):
        want = conv2d_rows(orc, g, f, 0, y0, y0 + 64)
        worst = max(worst, max_rel_err(got[y0:y0 + 64], want))
    print(K, worst)
