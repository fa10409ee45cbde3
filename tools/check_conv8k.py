import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
from oracle import Oracle, max_rel_err
orc = Oracle()
for H, W in ((8192, 8192), (2048, 8192), (8192, 2048), (4096, 4096)):
    g = torch.empty((H, W), dtype=torch.float32, device="cuda"); dev.fill_random(g, 0)
    o = torch.empty_like(g)
    hin = g.cpu().numpy()
    for K in (5, 6, 7):
        f = orc.random_filter(K, K, np.float32, 1)
        for rep in range(2):
            o.fill_(1234.0)
            dev.conv2d(g, o, f); torch.cuda.synchronize()
            hout = o.cpu().numpy()
            want = orc.conv2d(hin[:64], f, 0)[:60]  # top band exact for rows < 64-3
            e = np.abs(hout[:60] - want) > 1e-4
            ys, xs = np.nonzero(e)
            # also check a middle band
            mid = orc.conv2d(hin[H//2-40:H//2+40], f, 0)[10:70]
            e2 = np.abs(hout[H//2-30:H//2+30] - mid) > 1e-4
            print(H, W, K, rep, "top bad", int(e.sum()), (ys.min(), ys.max(), xs.min(), xs.max()) if len(ys) else "", "mid bad", int(e2.sum()),
                  "n1234", int((hout == 1234.0).sum()))
