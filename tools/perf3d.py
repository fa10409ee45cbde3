import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
PEAK = 6538.6
def bench(fn, iters):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); fn(); e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e)
for (n, nz) in ((512, 512), (2048, 258)):
    for dt, tdt in (("f32", torch.float32), ("f64", torch.float64)):
        a = torch.empty((nz, n, n), dtype=tdt, device="cuda"); dev.fill_random(a, 0); b = a.clone()
        for name in ("3d7pt", "3d27pt", "poisson", "3d13pt"):
            st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), np.float32 if dt == "f32" else np.float64)
            it = 10
            ms = bench(lambda: dev.stencil3d_run(a, b, st, it), it)
            gc = n * n * nz * it / ms / 1e6
            sz = 4 if dt == "f32" else 8
            print(json.dumps({"k": f"{name}_{dt}_{n}x{nz}", "gcells": round(gc, 1), "frac": round(gc * 2 * sz / PEAK, 4)}))
        del a, b
