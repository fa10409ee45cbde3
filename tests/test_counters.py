"""Closed-form OpCounters equal what the reference's simulator counts (CPU only).

warp.hpp:12-28 makes OpCounters part of the kernel API; the drop-in fills
them analytically.  Checked against the golden counters of the
reference's CPU SSAM path (tests/golden/golden.json) and, when oracle/_ref is
present, against live reference runs over random configurations.
"""
import numpy as np

import cases as C
from oracle import Oracle


def _stencil_from(lib, name, spec):
    if name is None:
        return lib.Stencil("int", 2 if spec is C.INT_STENCIL_2D else 3, spec["order"], 0,
                           [lib.StencilTap(tuple(o), c)
                            for o, c in zip(spec["offsets"], spec["coeffs"])])
    return lib.make_benchmark_stencil(name)


def test_golden_conv_counters(lib, golden):
    for tag, dt, w, h, m, n, gs, fs, bnd in C.conv_cases():
        got = lib.counters_conv2d(w, h, m, n, lib.KernelConfig())
        assert list(got.as_tuple()) == golden["conv"][tag]["counters"], tag


def test_golden_stencil_counters(lib, golden):
    for tag, dt, w, h, name, gs, iters in C.stencil2d_cases():
        st = _stencil_from(lib, name, C.INT_STENCIL_2D)
        got = lib.counters_stencil2d(w, h, st, lib.KernelConfig(), iters)
        assert list(got.as_tuple()) == golden["stencil2d"][tag]["counters"], tag
    for tag, dt, nx, ny, nz, name, gs, iters in C.stencil3d_cases():
        st = _stencil_from(lib, name, C.INT_STENCIL_3D)
        rec = golden["stencil3d"][tag]
        got = lib.counters_stencil3d(nx, ny, nz, st, lib.KernelConfig(p=rec["p"], b=rec["b"]),
                                     iters)
        assert list(got.as_tuple()) == rec["counters"], tag


def test_conv_counters_closed_form_law(lib):
    """test_kernels_conv.cpp:88-103: 100x50, 3x3 -> 52 tiles."""
    c = lib.counters_conv2d(100, 50, 3, 3, lib.KernelConfig())
    tiles = 52
    assert c.as_tuple() == (tiles * 36, tiles * 8, tiles * 36, tiles * 32 * 6, 5000)


def test_counters_random_vs_reference(lib, ref):
    orc = Oracle()
    rng = np.random.default_rng(7)
    for _ in range(25):
        m, n = rng.integers(1, 21, size=2)
        p = int(rng.integers(1, 9))
        b = 32 * int(rng.integers(1, 7))
        w = int(rng.integers(32, 150))
        h = int(rng.integers(n + p - 1, 120))
        g = orc.random_grid((h, w), np.int64, 3)
        rc, _, cnt = ref.conv2d(g, np.ones((m, n), np.int64), p=p, b=b)
        assert rc == 0
        got = lib.counters_conv2d(w, h, int(m), int(n), lib.KernelConfig(p=p, b=b))
        assert list(got.as_tuple()) == cnt.tolist(), (m, n, p, b, w, h)
    for _ in range(20):
        k = int(rng.integers(0, 4))
        taps = {(0, 0, 0)}
        for _ in range(int(rng.integers(1, 7))):
            taps.add((int(rng.integers(-k, k + 1)), int(rng.integers(-k, k + 1)), 0))
        offs = sorted(taps)
        k = max(abs(c) for o in offs for c in o)
        p = int(rng.integers(1, 6))
        w = int(rng.integers(2 * k + 1, 120))
        h = int(rng.integers(2 * k + 1, 90))
        iters = int(rng.integers(1, 3))
        g = orc.random_grid((h, w), np.int64, 4)
        cf = np.ones(len(offs), np.int64)
        rc, _, cnt = ref.stencil2d(g, offs, cf, k, iters, p=p)
        assert rc == 0
        st = lib.Stencil("r", 2, k, 0, [lib.StencilTap(o, 1) for o in offs])
        got = lib.counters_stencil2d(w, h, st, lib.KernelConfig(p=p), iters)
        assert list(got.as_tuple()) == cnt.tolist(), (offs, p, w, h)
