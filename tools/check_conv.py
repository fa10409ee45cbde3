import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1907_06154_b200 as ssam
from oracle import Oracle, max_rel_err
orc = Oracle()
for (H, W) in ((64, 256), (300, 512), (1024, 1024)):
    for dt in (np.float32, np.float64):
        g = orc.random_grid((H, W), dt, 0)
        bad = []
        for K in range(1, 21):
            f = orc.random_filter(K, K, dt, 1)
            e = max_rel_err(ssam.conv2d(g, f), orc.conv2d(g, f, 0))
            if e > (1e-5 if dt == np.float32 else 1e-12):
                got = ssam.conv2d(g, f); want = orc.conv2d(g, f, 0)
                err = np.abs(got - want) > 1e-3
                ys, xs = np.nonzero(err)
                bad.append((K, f"{e:.2g}", int(err.sum()), (ys.min(), ys.max(), xs.min(), xs.max()) if len(ys) else None))
        print(H, W, np.dtype(dt).name, "bad:", bad)
