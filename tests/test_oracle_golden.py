"""Pins the C oracle restatement (oracle/ssam_oracle.c) to the reference.

CPU only.  Three kinds of evidence:
  * the hand-computed fixtures frozen in proj/tests/test_oracle.cpp:19-129;
  * golden digests of the reference's own oracle.hpp / rng.hpp /
    stencil_catalog.cpp outputs (tests/golden/golden.json, made by
    tests/golden/make_golden.py from oracle/_ref);
  * when oracle/_ref is present, a direct side-by-side run.
"""
import hashlib

import numpy as np
import pytest

import cases as C

NP = {"f32": np.float32, "f64": np.float64, "i64": np.int64}


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def counting_grid(w, h):
    return (np.arange(w * h, dtype=np.int64) + 1).reshape(h, w)


# ---- proj/tests/test_oracle.cpp ---------------------------------------------

def test_conv_identity(orc):
    g = counting_grid(6, 5)
    assert np.array_equal(orc.conv2d(g, np.ones((1, 1), np.int64)), g)


def test_conv_constant_replicate(orc):
    g = np.full((8, 8), 3, np.int64)
    f = np.array([1, 2, 0, -1, 4, 2, 0, 1, 1], np.int64).reshape(3, 3)
    assert np.all(orc.conv2d(g, f, boundary=1) == 30)


def test_conv_hand_fixture(orc):
    g = counting_grid(4, 4)
    f = np.arange(1, 10, dtype=np.int64).reshape(3, 3)
    zero = orc.conv2d(g, f, 0)
    assert zero[1, 1] == 228 and zero[2, 2] == 453 and zero[0, 0] == 35 and zero[3, 3] == 371
    repl = orc.conv2d(g, f, 1)
    assert repl[0, 0] == 99 and repl[1, 1] == 228


def test_stencil2d_identity(orc):
    g = counting_grid(5, 5)
    for it in (1, 3):
        assert np.array_equal(orc.stencil2d(g, [(0, 0, 0)], [1], 0, it), g)


def test_stencil2d_convex_constant(orc):
    g = np.full((7, 7), 2.5)
    offs = [(0, 0, 0), (-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0)]
    out = orc.stencil2d(g, offs, [0.2] * 5, 1, 4)
    assert np.allclose(out, 2.5, rtol=1e-12)


def test_stencil2d_two_sweep_fixture(orc):
    y, x = np.mgrid[0:5, 0:5]
    g = (x + y).astype(np.int64)
    offs = [(0, 0, 0), (-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0)]
    out = orc.stencil2d(g, offs, [1, 2, 3, 4, 5], 1, 2)
    expect = np.array([[0, 1, 2, 3, 4], [1, 414, 615, 568, 5], [2, 675, 960, 927, 6],
                       [3, 512, 755, 610, 7], [4, 5, 6, 7, 8]])
    assert np.array_equal(out, expect)


def test_stencil3d_identity_and_ring(orc):
    g = np.arange(64, dtype=np.int64).reshape(4, 4, 4)
    assert np.array_equal(orc.stencil3d(g, [(0, 0, 0)], [1], 1, 2), g)
    out = orc.stencil3d(g, [(0, 0, 0), (0, 0, 1)], [1, 7], 1, 1)
    for z in range(4):
        for y in range(4):
            for x in range(4):
                inner = 1 <= x < 3 and 1 <= y < 3 and 1 <= z < 3
                want = g[z, y, x] + 7 * g[z + 1, y, x] if inner else g[z, y, x]
                assert out[z, y, x] == want


# ---- golden digests from the reference ---------------------------------------

@pytest.mark.parametrize("dt", ["f32", "f64", "i64"])
def test_rng_streams(orc, golden, dt):
    for seed in (0, 1, 11, 13, 1234, 4321):
        assert digest(orc.random_grid(4096, NP[dt], seed)) == golden["rng"][f"{dt}_{seed}"]
    for (m, n, seed) in ((3, 3, 1), (20, 20, 1), (5, 4, 10), (7, 1, 3)):
        key = f"{dt}_{m}x{n}_{seed}"
        assert digest(orc.random_filter(m, n, NP[dt], seed)) == golden["filters"][key]


def test_rng_offset_addressable(orc):
    """Index-addressable draws (device fill contract): stream[first:] == offset fill."""
    full = orc.random_grid(1000, np.float32, 7)
    part = orc.random_grid(400, np.float32, 7, first=600)
    assert np.array_equal(full[600:], part)


def test_catalog(orc, golden):
    assert orc.benchmark_names() == C.NAMES_2D + C.NAMES_3D
    for name, want in golden["catalog"].items():
        st = orc.benchmark_stencil(name)
        assert (st["dims"], st["order"], st["fpp"]) == (want["dims"], want["order"], want["fpp"])
        assert st["offsets"].tolist() == want["offsets"]
        assert [float(c).hex() for c in st["coeffs"]] == want["coeffs"]


def test_conv_oracle_digests(orc, golden):
    for tag, dt, w, h, m, n, gs, fs, bnd in C.conv_cases():
        g = orc.random_grid((h, w), NP[dt], gs)
        f = orc.random_filter(m, n, NP[dt], fs)
        assert digest(orc.conv2d(g, f, bnd)) == golden["conv"][tag]["oracle"], tag


def _taps(orc, name, spec):
    if name is None:
        return spec["order"], spec["offsets"], spec["coeffs"]
    st = orc.benchmark_stencil(name)
    return st["order"], st["offsets"], st["coeffs"]


def test_stencil2d_oracle_digests(orc, golden):
    for tag, dt, w, h, name, gs, iters in C.stencil2d_cases():
        g = orc.random_grid((h, w), NP[dt], gs)
        order, offs, cfs = _taps(orc, name, C.INT_STENCIL_2D)
        cf = np.asarray(cfs, dtype=np.float64).astype(NP[dt])
        assert digest(orc.stencil2d(g, offs, cf, order, iters)) == \
            golden["stencil2d"][tag]["oracle"], tag


def test_stencil3d_oracle_digests(orc, golden):
    for tag, dt, nx, ny, nz, name, gs, iters in C.stencil3d_cases():
        g = orc.random_grid((nz, ny, nx), NP[dt], gs)
        order, offs, cfs = _taps(orc, name, C.INT_STENCIL_3D)
        cf = np.asarray(cfs, dtype=np.float64).astype(NP[dt])
        assert digest(orc.stencil3d(g, offs, cf, order, iters)) == \
            golden["stencil3d"][tag]["oracle"], tag


def test_reference_simulator_agrees_on_ints(golden):
    """Integer mode: the reference's CPU SSAM path is bit-identical to its oracle."""
    for tag, rec in golden["conv"].items():
        if tag.startswith(("c1_", "unit_")):
            assert rec["oracle"] == rec["ssam"], tag
