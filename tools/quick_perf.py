"""Quick per-kernel throughput probe (device-resident, CUDA events)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev

PEAK = 6538.6

def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best

res = []
H = W = 8192
g = torch.empty((H, W), dtype=torch.float32, device="cuda"); dev.fill_random(g, 0)
o = torch.empty_like(g)
for K in [int(k) for k in (sys.argv[1].split(",") if len(sys.argv) > 1 else "3,5,7,11,15,20".split(","))]:
    f = np.random.default_rng(1).uniform(-1, 1, (K, K)).astype(np.float32)
    ms = timeit(lambda: dev.conv2d(g, o, f))
    gc = H * W / ms / 1e6
    res.append(dict(k=f"conv{K}x{K}_f32", ms=ms, gcells=gc, gbs=gc * 8, frac=gc * 8 / PEAK,
                    tflops=gc * 2 * K * K / 1e3))
for dt, tdt in (("f32", torch.float32), ("f64", torch.float64)):
    a = torch.empty((H, W), dtype=tdt, device="cuda"); dev.fill_random(a, 0)
    b = torch.empty_like(a)
    for name in ("2d5pt", "2d9pt", "2ds25pt"):
        st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), np.float32 if dt == "f32" else np.float64)
        ms = timeit(lambda: dev.stencil2d_sweep(a, b, st))
        gc = H * W / ms / 1e6
        sz = 4 if dt == "f32" else 8
        res.append(dict(k=f"{name}_{dt}", ms=ms, gcells=gc, gbs=gc * 2 * sz, frac=gc * 2 * sz / PEAK))
    del a, b
n = 512
for dt, tdt in (("f32", torch.float32), ("f64", torch.float64)):
    a = torch.empty((n, n, n), dtype=tdt, device="cuda"); dev.fill_random(a, 0)
    b = torch.empty_like(a)
    for name in ("3d7pt", "3d13pt", "3d27pt", "poisson"):
        st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), np.float32 if dt == "f32" else np.float64)
        ms = timeit(lambda: dev.stencil3d_sweep(a, b, st))
        gc = n ** 3 / ms / 1e6
        sz = 4 if dt == "f32" else 8
        res.append(dict(k=f"{name}_{dt}_512", ms=ms, gcells=gc, gbs=gc * 2 * sz, frac=gc * 2 * sz / PEAK))
    del a, b
for r in res:
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}))
