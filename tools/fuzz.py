"""Randomised parity sweep through the public API (host grids in, host grids
out) against the oracle: conv2d (any m x n <= 20, both boundaries, f32/f64/
int64, odd widths), stencil2d/3d (random tap sets of order 1..3 and catalog
stencils, random shapes and iteration counts), conv1d and scan.
python tools/fuzz.py [SECONDS] -- prints one summary line per family."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1907_06154_b200 as ssam
from oracle import Oracle, max_rel_err

orc = Oracle()
rng = np.random.default_rng(int(os.environ.get("FUZZ_SEED", "7")))
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
TOL = {np.dtype(np.float32): 1e-5, np.dtype(np.float64): 1e-12, np.dtype(np.int64): 0.0}
stats = {}


def note(fam, dt, err, case):
    s = stats.setdefault(fam, {"n": 0, "fail": 0, "worst": {}, "last": None})
    s["n"] += 1
    s["last"] = (np.dtype(dt).name, case, err)
    k = np.dtype(dt).name
    s["worst"][k] = max(s["worst"].get(k, 0.0), err)
    if err > TOL[np.dtype(dt)]:
        s["fail"] += 1
        print("FAIL", fam, k, case, err, flush=True)


def rand_dt():
    return [np.float32, np.float64, np.int64][int(rng.integers(0, 3))]


def rand_taps(dims, order):
    cells = [(dx, dy, dz) for dz in (range(-order, order + 1) if dims == 3 else [0])
             for dy in range(-order, order + 1) for dx in range(-order, order + 1)]
    n = int(rng.integers(1, min(len(cells), 40) + 1))
    pick = [cells[i] for i in rng.choice(len(cells), n, replace=False)]
    if not any(max(abs(c) for c in t) == order for t in pick):
        pick[0] = (order, 0, 0)
    return [ssam.StencilTap(t, float(rng.uniform(-0.3, 0.3))) for t in pick]


t_end = time.time() + budget
i = 0
while time.time() < t_end:
    i += 1
    fam = ["conv2d", "stencil2d", "stencil3d", "conv1d", "scan"][i % 5]
    dt = rand_dt()
    seed = int(rng.integers(0, 1 << 30))
    if fam == "conv2d":
        m, n = int(rng.integers(1, 21)), int(rng.integers(1, 21))
        p = 4
        H = int(rng.integers(n + p - 1, 300))
        W = int(rng.integers(32, 400))
        bnd = int(rng.integers(0, 2))
        g = orc.random_grid((H, W), dt, seed)
        f = orc.random_filter(m, n, dt, seed + 1)
        got = ssam.conv2d(g, f, ssam.KernelConfig(p=p, boundary=ssam.Boundary(bnd)))
        note(fam, dt, max_rel_err(got, orc.conv2d(g, f, bnd)), (H, W, m, n, bnd))
    elif fam in ("stencil2d", "stencil3d"):
        dims = 2 if fam == "stencil2d" else 3
        if rng.random() < 0.4:
            names = [s for s in ("2d5pt", "2d9pt", "2d13pt", "2d17pt", "2d21pt", "2ds25pt",
                                 "2d25pt", "2d64pt", "2d81pt", "2d121pt") if dims == 2] or \
                    ["3d7pt", "3d13pt", "3d27pt", "3d125pt", "poisson"]
            st = ssam.make_benchmark_stencil(names[int(rng.integers(0, len(names)))])
        else:
            order = int(rng.integers(1, 4))
            taps = rand_taps(dims, order)
            st = ssam.Stencil("fuzz", dims, order, 0, taps)
        st = ssam.convert_stencil(st, dt)
        k = st.order
        iters = int(rng.integers(1, 5))
        if dims == 2:
            shape = (int(rng.integers(2 * k + 1, 200)), int(rng.integers(max(32, 2 * k + 1), 300)))
        else:
            b = 128
            shape = (int(rng.integers(2 * k + 1, 24)), int(rng.integers(2 * k + 1, 40)),
                     int(rng.integers(max(32, 2 * k + 1), 140)))
        g = orc.random_grid(shape, dt, seed)
        offs = [t.offset for t in st.taps]
        cf = np.asarray([t.coeff for t in st.taps], dt)
        if dims == 2:
            got = ssam.stencil2d(g, st, ssam.KernelConfig(), iters)
            want = orc.stencil2d(g, offs, cf, k, iters)
        else:
            got = ssam.stencil3d(g, st, ssam.KernelConfig(p=2, b=128 if k < 2 else 256), iters)
            want = orc.stencil3d(g, offs, cf, k, iters)
        note(fam, dt, max_rel_err(got, want), (st.name, shape, iters))
        if rng.random() < 0.3:
            # the device-set path (slabs sharing device 0) must equal it bit for bit
            ndev = int(rng.integers(2, 5))
            cfg = ssam.KernelConfig() if dims == 2 else ssam.KernelConfig(p=2, b=128 if k < 2 else 256)
            multi, _ = ssam.stencil_multi(g, st, [0] * ndev, cfg, iters)
            note(fam + "_multi", dt, 0.0 if np.array_equal(multi, got) else float("inf"),
                 (st.name, shape, iters, ndev))
    elif fam == "conv1d":
        m = int(rng.integers(1, 33))
        nlen = int(rng.integers(32, 20000))
        bnd = int(rng.integers(0, 2))
        sig = orc.random_grid(nlen, dt, seed)
        f = orc.random_filter(m, 1, dt, seed + 1).reshape(-1)
        got = ssam.conv1d(sig, f, ssam.KernelConfig(boundary=ssam.Boundary(bnd)))
        note(fam, dt, max_rel_err(got, orc.conv1d(sig, f, bnd)), (nlen, m, bnd))
    else:
        nlen = 32 * int(rng.integers(1, 10000))  # the API takes whole lane_count tiles
        v = orc.random_grid(nlen, np.int64, seed)
        note(fam, np.int64, max_rel_err(ssam.scan(v), orc.scan(v)), (nlen,))
bad = 0
for fam, s in stats.items():
    bad += s["fail"]
    print(f"{fam:10s} cases {s['n']:5d}  fails {s['fail']}  worst " +
          ", ".join(f"{k} {v:.2e}" for k, v in sorted(s["worst"].items())) +
          f"  last case {s['last']}")
print("FUZZ", "PASS" if bad == 0 else "FAIL", f"({i} cases)")
