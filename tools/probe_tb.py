import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
H, W = 16, 64
for dt in (np.float64, np.float32):
    g = np.arange(H * W, dtype=dt).reshape(H, W)
    offs = [(0, -1, 0), (-1, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 0)]
    for one in offs:
        st = ssam.Stencil("p", 2, 1, 0, [ssam.StencilTap(o, dt(1.0 if o == one else 0.0)) for o in offs])
        for tb in (2, 4):
            a = torch.from_numpy(g.copy()).cuda(); b = a.clone()
            dev.stencil2d_tb(a, b, st, tb)
            out = b.cpu().numpy()
            # which shift (sx, sy) explains interior cell (8, 8)?
            v = int(out[8, 8]); sy, sx = divmod(v, W); sy -= 8; sx -= 8
            print(np.dtype(dt).name, "tap", one, "tb", tb, "-> effective shift per run (dx,dy) =", (sx, sy),
                  "expected", (one[0] * tb, one[1] * tb))
