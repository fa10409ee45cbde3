"""2D/3D stencils on the GPU vs the Jacobi oracle (run with -m gpu).

Mirrors proj/tests/test_kernels_stencil.cpp and acceptance criterion 2
(proj/tests/acceptance.cpp:76-114); full-size north-star configs
(8192^2 x 100 sweeps, 512^3) use the exact cone-windowed oracle.
"""
import hashlib

import numpy as np
import pytest

import cases as C
from oracle import Oracle, max_rel_err
from windows import sample_windows_2d, stencil2d_window

pytestmark = pytest.mark.gpu
NP = {"f32": np.float32, "f64": np.float64, "i64": np.int64}
TOL = {np.dtype(np.float32): 1e-5, np.dtype(np.float64): 1e-12, np.dtype(np.int64): 0.0}


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def mk(lib, dims, order, offsets, coeffs, dtype):
    t = np.dtype(dtype).type
    return lib.Stencil("t", dims, order, 0,
                       [lib.StencilTap(tuple(o), t(c)) for o, c in zip(offsets, coeffs)])


def taps_of(st):
    return [t.offset for t in st.taps], [t.coeff for t in st.taps]


# ---- 2D --------------------------------------------------------------------------

def test_identity_fixed_point(cuda_lib, orc):
    g = orc.random_grid((40, 64), np.int64, 1)
    st = mk(cuda_lib, 2, 0, [(0, 0, 0)], [1], np.int64)
    for it in (1, 3):
        assert np.array_equal(cuda_lib.stencil2d(g, st, cuda_lib.KernelConfig(), it), g)


def test_convex_combination_keeps_constants(cuda_lib):
    g = np.full((64, 64), 3.25)
    st = mk(cuda_lib, 2, 1, [(0, 0, 0), (-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0)],
            [0.2] * 5, np.float64)
    out = cuda_lib.stencil2d(g, st, cuda_lib.KernelConfig(), 4)
    assert np.allclose(out, 3.25, rtol=1e-12, atol=0)


def test_single_off_centre_taps(cuda_lib, orc):
    g = orc.random_grid((48, 64), np.int64, 7)
    for dx, dy in ((1, 0), (-1, 0), (0, 1), (0, -1), (1, -1)):
        st = mk(cuda_lib, 2, 1, [(dx, dy, 0)], [1], np.int64)
        out = cuda_lib.stencil2d(g, st, cuda_lib.KernelConfig(), 1)
        assert np.array_equal(out[1:47, 1:63], g[1 + dy:47 + dy, 1 + dx:63 + dx]), (dx, dy)


def test_int_stencil_bit_exact(cuda_lib, orc, golden):
    s = C.INT_STENCIL_2D
    st = mk(cuda_lib, 2, s["order"], s["offsets"], s["coeffs"], np.int64)
    g = orc.random_grid((52, 80), np.int64, 12)
    for it in (1, 2, 4):
        got = cuda_lib.stencil2d(g, st, cuda_lib.KernelConfig(), it)
        assert digest(got) == golden["stencil2d"][f"int_it{it}"]["oracle"]


@pytest.mark.parametrize("name", C.NAMES_2D)
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_criterion2_2d(cuda_lib, orc, name, dt):
    """All 10 2D benchmarks, 256^2 x 4 sweeps: f64 <= 1e-12, f32 <= 1e-5."""
    st = cuda_lib.convert_stencil(cuda_lib.make_benchmark_stencil(name), NP[dt])
    g = orc.random_grid((256, 256), NP[dt], 11)
    got = cuda_lib.stencil2d(g, st, cuda_lib.KernelConfig(), 4)
    offs, cfs = taps_of(st)
    want = orc.stencil2d(g, offs, np.asarray(cfs, NP[dt]), st.order, 4)
    assert max_rel_err(got, want) <= TOL[np.dtype(NP[dt])]


def test_ring_preserved_exactly(cuda_lib, orc):
    st = cuda_lib.make_benchmark_stencil("2d13pt")
    g = orc.random_grid((40, 72), np.float64, 5)
    out = cuda_lib.stencil2d(g, st, cuda_lib.KernelConfig(), 3)
    k = st.order
    ring = np.ones_like(g, dtype=bool)
    ring[k:-k, k:-k] = False
    assert np.array_equal(out[ring], g[ring])


def test_randomized_int_stencils(cuda_lib, orc):
    """test_kernels_stencil.cpp:217-253 style: random tap sets, bit-exact."""
    rng = np.random.default_rng(8192)
    for rep in range(25):
        k = int(rng.integers(0, 9))  # k > 6 exercises the direct-gather path
        taps = {(0, 0, 0): int(rng.integers(1, 6))}
        for _ in range(int(rng.integers(1, 7))):
            off = (int(rng.integers(-k, k + 1)), int(rng.integers(-k, k + 1)), 0)
            taps.setdefault(off, int(rng.integers(-9, 10)))
        offs = list(taps)
        k = max(abs(c) for o in offs for c in o)
        st = mk(cuda_lib, 2, k, offs, list(taps.values()), np.int64)
        w = int(rng.integers(2 * k + 1, 150))
        h = int(rng.integers(2 * k + 1, 100))
        it = int(rng.integers(1, 4))
        g = orc.random_grid((h, w), np.int64, int(rng.integers(1 << 62)))
        got = cuda_lib.stencil2d(g, st, cuda_lib.KernelConfig(p=int(rng.integers(1, 7))), it)
        want = orc.stencil2d(g, offs, np.asarray(list(taps.values()), np.int64), k, it)
        assert np.array_equal(got, want), (rep, offs, w, h, it)


@pytest.mark.parametrize("name", C.NORTH_STAR_2D)
@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_north_star_8192_100_sweeps(cuda_lib, orc, name, dt):
    """configs[2]: 8192^2, 100 sweeps, cone-windowed exact oracle at corners,
    edges and random interior points."""
    import torch
    from paper_1907_06154_b200 import device as dev
    H = W = 8192
    iters = 100
    st = cuda_lib.convert_stencil(cuda_lib.make_benchmark_stencil(name), NP[dt])
    tdt = torch.float32 if dt == "f32" else torch.float64
    a = torch.empty((H, W), dtype=tdt, device="cuda")
    b = torch.empty_like(a)
    dev.fill_random(a, 0)
    host_in = a.cpu().numpy()
    res = dev.stencil2d_run(a, b, st, iters)
    host_out = res.cpu().numpy()
    offs, cfs = taps_of(st)
    cf = np.asarray(cfs, NP[dt])
    worst = 0.0
    rng = np.random.default_rng(3)
    for (y0, y1, x0, x1) in sample_windows_2d(H, W, 16, rng, n_interior=2):
        want = stencil2d_window(orc, host_in, offs, cf, st.order, iters, y0, y1, x0, x1)
        worst = max(worst, max_rel_err(host_out[y0:y1, x0:x1], want))
    assert worst <= TOL[np.dtype(NP[dt])], worst


# ---- 3D --------------------------------------------------------------------------

def cfg3(lib, order):
    return lib.KernelConfig(p=2, b=max(256, 32 * (2 * order + 1)))


def test_3d_identity_and_constant(cuda_lib, orc):
    g = orc.random_grid((8, 16, 32), np.float64, 3)
    ident = mk(cuda_lib, 3, 0, [(0, 0, 0)], [1.0], np.float64)
    assert np.array_equal(cuda_lib.stencil3d(g, ident, cuda_lib.KernelConfig(p=2), 2), g)
    st = cuda_lib.make_benchmark_stencil("3d7pt")
    c = np.full((9, 12, 32), 1.5)
    out = cuda_lib.stencil3d(c, st, cuda_lib.KernelConfig(p=2, b=128), 2)
    assert np.allclose(out, 1.5, rtol=1e-12, atol=0)


def test_3d_out_of_plane_orientation(cuda_lib, orc):
    g = orc.random_grid((10, 12, 40), np.int64, 9)
    for dz in (-1, 1):
        st = mk(cuda_lib, 3, 1, [(0, 0, dz)], [1], np.int64)
        out = cuda_lib.stencil3d(g, st, cuda_lib.KernelConfig(p=2), 1)
        assert np.array_equal(out[1:9, 1:11, 1:39], g[1 + dz:9 + dz, 1:11, 1:39])


def test_3d_int_exact(cuda_lib, orc, golden):
    s = C.INT_STENCIL_3D
    st = mk(cuda_lib, 3, s["order"], s["offsets"], s["coeffs"], np.int64)
    g = orc.random_grid((9, 10, 36), np.int64, 31)
    got = cuda_lib.stencil3d(g, st, cuda_lib.KernelConfig(p=2), 2)
    assert digest(got) == golden["stencil3d"]["int3d"]["oracle"]


@pytest.mark.parametrize("name", C.NAMES_3D)
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_criterion2_3d(cuda_lib, orc, name, dt):
    """All 5 3D benchmarks, 64^3 x 2 sweeps (acceptance.cpp:95-108)."""
    st = cuda_lib.convert_stencil(cuda_lib.make_benchmark_stencil(name), NP[dt])
    g = orc.random_grid((64, 64, 64), NP[dt], 13)
    got = cuda_lib.stencil3d(g, st, cfg3(cuda_lib, st.order), 2)
    offs, cfs = taps_of(st)
    want = orc.stencil3d(g, offs, np.asarray(cfs, NP[dt]), st.order, 2)
    assert max_rel_err(got, want) <= TOL[np.dtype(NP[dt])]


def test_3d_unit_centre_identity(cuda_lib, orc):
    st = cuda_lib.make_benchmark_stencil("3d7pt")
    st = cuda_lib.Stencil(st.name, 3, 1, 0, [cuda_lib.StencilTap(t.offset, 1.0 if t.offset ==
                                                                (0, 0, 0) else 0.0)
                                             for t in st.taps])
    g = orc.random_grid((8, 10, 40), np.float64, 6)
    assert np.array_equal(cuda_lib.stencil3d(g, st, cuda_lib.KernelConfig(p=2), 3), g)


def test_3d_random_and_high_order(cuda_lib, orc):
    rng = np.random.default_rng(33)
    for rep in range(12):
        k = int(rng.integers(1, 4))  # k = 3 exercises the direct-gather path
        taps = {(0, 0, 0): 2}
        for _ in range(int(rng.integers(1, 8))):
            off = tuple(int(v) for v in rng.integers(-k, k + 1, size=3))
            taps.setdefault(off, int(rng.integers(-5, 6)))
        offs = list(taps)
        k = max(abs(c) for o in offs for c in o)
        st = mk(cuda_lib, 3, k, offs, list(taps.values()), np.int64)
        shape = tuple(int(v) for v in rng.integers(2 * k + 1, 30, size=3))
        g = orc.random_grid(shape, np.int64, rep)
        got = cuda_lib.stencil3d(g, st, cfg3(cuda_lib, k), 2)
        want = orc.stencil3d(g, offs, np.asarray(list(taps.values()), np.int64), k, 2)
        assert np.array_equal(got, want), (rep, offs, shape)


@pytest.mark.parametrize("name", C.NORTH_STAR_3D)
@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_north_star_512_cubed(cuda_lib, orc, name, dt):
    """configs[3]: 512^3, 10 sweeps; cone windows at a corner and the centre."""
    import torch
    from paper_1907_06154_b200 import device as dev
    n = 512
    iters = 10
    st = cuda_lib.convert_stencil(cuda_lib.make_benchmark_stencil(name), NP[dt])
    tdt = torch.float32 if dt == "f32" else torch.float64
    a = torch.empty((n, n, n), dtype=tdt, device="cuda")
    b = torch.empty_like(a)
    dev.fill_random(a, 0)
    offs, cfs = taps_of(st)
    cf = np.asarray(cfs, NP[dt])
    mg = st.order * iters
    wins = [(0, 12, 0, 12, 0, 12), (250, 262, 250, 262, 250, 262), (n - 12, n, 100, 112, n - 12, n)]
    inputs = []
    for z0, z1, y0, y1, x0, x1 in wins:
        zs, ys, xs = (slice(max(0, z0 - mg), min(n, z1 + mg)), slice(max(0, y0 - mg), min(n, y1 + mg)),
                      slice(max(0, x0 - mg), min(n, x1 + mg)))
        inputs.append((zs, ys, xs, a[zs, ys, xs].cpu().numpy()))
    res = dev.stencil3d_run(a, b, st, iters)
    worst = 0.0
    for (z0, z1, y0, y1, x0, x1), (zs, ys, xs, sub_in) in zip(wins, inputs):
        # oracle on the window-local grid: place it in a full-size frame view
        full = np.zeros((zs.stop - zs.start, ys.stop - ys.start, xs.stop - xs.start), NP[dt])
        full[...] = sub_in
        sub_out = orc.stencil3d(full, offs, cf, st.order, iters)
        want = sub_out[z0 - zs.start:z1 - zs.start, y0 - ys.start:y1 - ys.start,
                       x0 - xs.start:x1 - xs.start]
        got = res[z0:z1, y0:y1, x0:x1].cpu().numpy()
        worst = max(worst, max_rel_err(got, want))
    assert worst <= TOL[np.dtype(NP[dt])], worst


# ---- temporal blocking (2D) ------------------------------------------------------

@pytest.mark.parametrize("name", ["2d5pt", "2d9pt"])
@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_temporal_blocking_matches_sweeps(cuda_lib, orc, name, dt):
    """TB fused sweeps equal TB single sweeps BIT FOR BIT (one pinned chain per
    cell, engine2d.cuh star_row_chain) and the Jacobi oracle within
    tolerance, for every compiled depth and iteration counts that leave
    remainders."""
    import torch
    from paper_1907_06154_b200 import device as dev
    st = cuda_lib.convert_stencil(cuda_lib.make_benchmark_stencil(name), NP[dt])
    tdt = torch.float32 if dt == "f32" else torch.float64
    offs, cfs = taps_of(st)
    cf = np.asarray(cfs, NP[dt])
    tbmax = dev.stencil2d_tb_max(st, NP[dt])  # the automatic depth (2 or 4 here)
    assert tbmax >= 2
    for (H, W) in ((260, 300), (97, 1024)):
        g = orc.random_grid((H, W), NP[dt], 5)
        for iters in (1, 3, 8, 13):
            ref_a = torch.from_numpy(g).cuda()
            ref_b = ref_a.clone()
            single = dev.stencil2d_run(ref_a, ref_b, st, iters, tb=1).cpu().numpy()
            want = orc.stencil2d(g, offs, cf, st.order, iters)
            assert max_rel_err(single, want) <= TOL[np.dtype(NP[dt])]
            for tb in (2, 4, 8):
                if tb == 8 and st.order > 1:
                    continue  # compiled for order 1 only
                a = torch.from_numpy(g).cuda()
                b = a.clone()
                got = dev.stencil2d_run(a, b, st, iters, tb=tb).cpu().numpy()
                assert max_rel_err(got, want) <= TOL[np.dtype(NP[dt])], (H, W, iters, tb)
                assert np.array_equal(got, single), (H, W, iters, tb)
                ring = np.ones_like(g, dtype=bool)
                ring[st.order:-st.order, st.order:-st.order] = False
                assert np.array_equal(got[ring], g[ring])


@pytest.mark.parametrize("name,tbs", [("3d7pt", (2, 3, 4)), ("3d13pt", (2,)), ("poisson", (2,)),
                                      ("3d27pt", (2,))])
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_stencil3d_tb_bit_identical_to_single_sweeps(cuda_lib, orc, name, tbs, dt):
    """Temporal blocking (engine3d_pipe.cuh): Tb fused sweeps == Tb single sweeps,
    bit for bit, and == the oracle within tolerance; odd shapes and z-segments."""
    import torch
    from paper_1907_06154_b200 import device as dev
    st = cuda_lib.convert_stencil(cuda_lib.make_benchmark_stencil(name), dt)
    offs = [t.offset for t in st.taps]
    cf = np.asarray([t.coeff for t in st.taps], dt)
    tol = 1e-5 if dt == np.float32 else 1e-12
    for (nx, ny, nz) in ((132, 70, 37), (256, 97, 80), (64, 11, 9)):
        g = orc.random_grid((nz, ny, nx), dt, 21)
        for tb in tbs:
            a = torch.from_numpy(g).cuda()
            cur = a
            for _ in range(tb):
                nxt = cur.clone()
                dev.stencil3d_sweep(cur, nxt, st)
                cur = nxt
            f = a.clone()
            dev.stencil3d_tb(a, f, st, tb)
            assert torch.equal(f, cur), (name, tb, nx, ny, nz)
            want = orc.stencil3d(g, offs, cf, st.order, tb)
            assert max_rel_err(f.cpu().numpy(), want) <= tol, (name, tb, nx, ny, nz)
