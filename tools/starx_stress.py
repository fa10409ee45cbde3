"""Randomised parity of the 2D star paths (K = 4..6 stars on the FMA engine,
K >= 5 with the arms read from shared memory): random shapes and weights,
GPU sweeps vs the oracle (f32 1e-5, f64 1e-12).  python tools/starx_stress.py [N]"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
from oracle import Oracle, max_rel_err

orc = Oracle()
rng = np.random.default_rng(2026)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
worst = {np.float32: 0.0, np.float64: 0.0}
fails = 0
for it in range(N):
    K = int(rng.integers(4, 7))
    dt = np.float32 if rng.random() < 0.6 else np.float64
    H = int(rng.integers(2 * K + 1, 300))
    W = int(rng.integers(2 * K + 1, 700))
    if rng.random() < 0.7:
        W = (W + 3) // 4 * 4  # TMA-eligible rows
    taps = [ssam.StencilTap((0, 0, 0), float(rng.uniform(-1, 1)))]
    for i in range(1, K + 1):
        for o in ((-i, 0, 0), (i, 0, 0), (0, -i, 0), (0, i, 0)):
            taps.append(ssam.StencilTap(o, float(rng.uniform(-0.3, 0.3))))
    rng.shuffle(taps)
    st = ssam.Stencil(f"star{K}", 2, K, 0, taps)
    iters = int(rng.integers(1, 4))
    g = orc.random_grid((H, W), dt, it)
    a = torch.from_numpy(g).cuda()
    b = a.clone()
    for _ in range(iters):
        dev.stencil2d_sweep(a, b, st)
        a, b = b, a
    want = orc.stencil2d(g, [t.offset for t in st.taps], np.asarray([t.coeff for t in st.taps], dt),
                         K, iters)
    err = max_rel_err(a.cpu().numpy(), want)
    worst[dt] = max(worst[dt], err)
    tol = 1e-5 if dt == np.float32 else 1e-12
    if err > tol:
        fails += 1
        print("FAIL", K, np.dtype(dt).name, H, W, iters, err)
print(f"{N} random star cases, worst f32 {worst[np.float32]:.2e}, f64 {worst[np.float64]:.2e}, "
      f"fails {fails}")
print("STARX STRESS", "PASS" if fails == 0 else "FAIL")
