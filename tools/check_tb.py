import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
from oracle import Oracle, max_rel_err
orc = Oracle()
for name in ("2d5pt", "2d9pt"):
    for dt in (np.float32, np.float64):
        st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), dt)
        offs = [t.offset for t in st.taps]; cf = np.asarray([t.coeff for t in st.taps], dt)
        for (H, W) in ((64, 64), (256, 256), (260, 300), (40, 1024)):
            g = orc.random_grid((H, W), dt, 11)
            for tb in (2, 4):
                for iters in (tb, 2 * tb + 1):
                    a = torch.from_numpy(g).cuda(); b = a.clone()
                    got = dev.stencil2d_run(a, b, st, iters, tb=tb).cpu().numpy()
                    want = orc.stencil2d(g, offs, cf, st.order, iters)
                    e = max_rel_err(got, want)
                    if e > (1e-5 if dt == np.float32 else 1e-12):
                        bad = np.abs(got.astype(np.float64) - want) > 1e-4
                        ys, xs = np.nonzero(bad)
                        print("FAIL", name, np.dtype(dt).name, H, W, "tb", tb, "it", iters, f"{e:.3g}",
                              int(bad.sum()), "rows", ys.min(), ys.max(), "cols", xs.min(), xs.max(),
                              "first", list(zip(ys[:4], xs[:4])))
print("done")
