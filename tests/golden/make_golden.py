#!/usr/bin/env python3
"""Generate tests/golden/golden.json from the UNMODIFIED reference.

Run in the dev container (needs oracle/_ref/libssam_ref.so, built by
`make -C oracle` from /root/reference):

    python tests/golden/make_golden.py

Records, for every case in cases.py:
  * SHA-256 of the reference oracle's output (oracle.hpp:44-116) -- pins our
    C restatement bit-for-bit and is the integer-exact target of the GPU path;
  * SHA-256 of the reference's CPU SSAM output and its OpCounters
    (kernels.hpp:189-384) -- pins our closed-form counters;
  * SHA-256 of the reference's random streams (rng.hpp) and the full
    benchmark catalog (stencil_catalog.cpp) with exact hex coefficients.
The inputs are regenerated from seeds, so no large arrays are stored.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import cases as C  # noqa: E402
from oracle import Reference  # noqa: E402

NP = {"f32": np.float32, "f64": np.float64, "i64": np.int64}


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    ref = Reference()
    out: dict = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/proj",
                 "rng": {}, "filters": {}, "catalog": {}, "conv": {}, "stencil2d": {},
                 "stencil3d": {}, "conv1d": {}, "scan": {}}

    for dt in ("f32", "f64", "i64"):
        for seed in (0, 1, 11, 13, 1234, 4321):
            out["rng"][f"{dt}_{seed}"] = digest(ref.random_grid(4096, NP[dt], seed))
        for (m, n, seed) in ((3, 3, 1), (20, 20, 1), (5, 4, 10), (7, 1, 3)):
            out["filters"][f"{dt}_{m}x{n}_{seed}"] = digest(ref.random_filter(m, n, NP[dt], seed))

    for name in C.NAMES_2D + C.NAMES_3D:
        st = ref.benchmark_stencil(name)
        out["catalog"][name] = dict(dims=st["dims"], order=st["order"], fpp=st["fpp"],
                                    offsets=st["offsets"].tolist(),
                                    coeffs=[float(c).hex() for c in st["coeffs"]])

    def grid2(dt, w, h, seed):
        return ref.random_grid(w * h, NP[dt], seed).reshape(h, w)

    for tag, dt, w, h, m, n, gs, fs, bnd in C.conv_cases():
        g = grid2(dt, w, h, gs)
        f = ref.random_filter(m, n, NP[dt], fs)
        rc, want, _ = ref.conv2d(g, f, boundary=bnd, naive=True)
        assert rc == 0
        rc, got, cnt = ref.conv2d(g, f, boundary=bnd)
        assert rc == 0
        out["conv"][tag] = dict(oracle=digest(want), ssam=digest(got), counters=cnt.tolist())

    for tag, dt, w, h, name, gs, iters in C.stencil2d_cases():
        g = grid2(dt, w, h, gs)
        if name is None:
            s = C.INT_STENCIL_2D
            order, offs, cfs = s["order"], s["offsets"], s["coeffs"]
        else:
            st = ref.benchmark_stencil(name)
            order, offs, cfs = st["order"], st["offsets"], st["coeffs"]
        cf = np.asarray(cfs, dtype=np.float64).astype(NP[dt])
        rc, want, _ = ref.stencil2d(g, offs, cf, order, iters, naive=True)
        assert rc == 0
        rc, got, cnt = ref.stencil2d(g, offs, cf, order, iters)
        assert rc == 0, (tag, rc)
        out["stencil2d"][tag] = dict(oracle=digest(want), ssam=digest(got), counters=cnt.tolist())

    for tag, dt, nx, ny, nz, name, gs, iters in C.stencil3d_cases():
        g = ref.random_grid(nx * ny * nz, NP[dt], gs).reshape(nz, ny, nx)
        if name is None:
            s = C.INT_STENCIL_3D
            order, offs, cfs = s["order"], s["offsets"], s["coeffs"]
        else:
            st = ref.benchmark_stencil(name)
            order, offs, cfs = st["order"], st["offsets"], st["coeffs"]
        cf = np.asarray(cfs, dtype=np.float64).astype(NP[dt])
        rc, want, _ = ref.stencil3d(g, offs, cf, order, iters, naive=True)
        assert rc == 0
        b = max(256, 32 * (2 * order + 1))
        rc, got, cnt = ref.stencil3d(g, offs, cf, order, iters, p=2, b=b)
        assert rc == 0, (tag, rc)
        out["stencil3d"][tag] = dict(oracle=digest(want), ssam=digest(got), counters=cnt.tolist(),
                                     p=2, b=b)

    for tag, dt, n, m, ss, fs, bnd, lanes in C.conv1d_cases():
        sig = ref.random_grid(n, NP[dt], ss)
        f = ref.random_filter(m, 1, NP[dt], fs).reshape(-1)
        rc, want, _ = ref.conv1d(sig, f, boundary=bnd, lane_count=lanes, naive=True)
        assert rc == 0
        rc, got, cnt = ref.conv1d(sig, f, boundary=bnd, lane_count=lanes)
        assert rc == 0, (tag, rc)
        out["conv1d"][tag] = dict(oracle=digest(want), ssam=digest(got), counters=cnt.tolist())

    for tag, dt, n, seed, lanes in C.scan_cases():
        v = ref.random_grid(n, NP[dt], seed)
        rc, want, _ = ref.scan(v, lane_count=lanes, naive=True)
        assert rc == 0
        rc, got, cnt = ref.scan(v, lane_count=lanes)
        assert rc == 0, (tag, rc)
        out["scan"][tag] = dict(oracle=digest(want), ssam=digest(got), counters=cnt.tolist())

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("wrote", path)


if __name__ == "__main__":
    main()
