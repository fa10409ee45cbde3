"""Edge shapes for the newer engines (-m gpu): the FMA conv engine on small /
odd images, the fused 3D pair on thin grids, conv1d / scan at their size
limits.  Oracle parity within the reference tolerances (int64 exact)."""
import numpy as np
import pytest

from oracle import max_rel_err

pytestmark = pytest.mark.gpu
TOL = {np.dtype(np.float32): 1e-5, np.dtype(np.float64): 1e-12, np.dtype(np.int64): 0.0}


@pytest.mark.parametrize("K", [6, 7, 11, 12, 13, 19, 20])
@pytest.mark.parametrize("shape", [(20, 32), (41, 64), (97, 132), (256, 260)])
def test_fma_conv_small_images(cuda_lib, orc, K, shape):
    h, w = shape
    if h < K:  # the reference needs H >= n + p - 1
        pytest.skip("shorter than one cache block")
    for dt in (np.float32, np.int64):
        g = orc.random_grid((h, w), dt, K * 7 + h)
        f = orc.random_filter(K, K, dt, K)
        cfg = cuda_lib.KernelConfig(p=1)
        got = cuda_lib.conv2d(g, f, cfg)
        assert max_rel_err(got, orc.conv2d(g, f, 0)) <= TOL[np.dtype(dt)], (K, shape, dt)


@pytest.mark.parametrize("shape", [(3, 3, 8), (4, 5, 16), (5, 3, 132), (7, 40, 260), (33, 17, 68)])
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_tb3d_thin_grids(cuda_lib, orc, shape, dt):
    import torch
    from paper_1907_06154_b200 import device as dev
    st = cuda_lib.convert_stencil(cuda_lib.make_benchmark_stencil("3d7pt"), dt)
    g = orc.random_grid(shape, dt, 3)
    a = torch.from_numpy(g).cuda()
    b, c, f = a.clone(), a.clone(), a.clone()
    dev.stencil3d_sweep(a, b, st)
    dev.stencil3d_sweep(b, c, st)
    dev.stencil3d_tb(a, f, st, 2)
    assert torch.equal(f, c), shape
    offs = [t.offset for t in st.taps]
    cf = np.asarray([t.coeff for t in st.taps], dt)
    for iters in (1, 2, 5):
        got = cuda_lib.stencil3d(g, st, cuda_lib.KernelConfig(p=2, b=128), iters)
        assert max_rel_err(got, orc.stencil3d(g, offs, cf, 1, iters)) <= TOL[np.dtype(dt)]


@pytest.mark.parametrize("n", [1, 31, 32, 4095, 4096, 4097, 65537, (1 << 20) + 7])
def test_scan_sizes_device(cuda_lib, orc, n):
    import torch
    from paper_1907_06154_b200 import device as dev
    v = np.random.default_rng(n).integers(-10**6, 10**6, n).astype(np.int64)
    x = torch.from_numpy(v).cuda()
    y = torch.empty_like(x)
    dev.scan(x, y)
    assert np.array_equal(y.cpu().numpy(), orc.scan(v))
    xf = torch.from_numpy(orc.random_grid(n, np.float32, n)).cuda()
    yf = torch.empty_like(xf)
    dev.scan(xf, yf)
    exact = np.cumsum(xf.cpu().numpy().astype(np.longdouble))
    scale = np.maximum(1.0, np.maximum.accumulate(np.abs(exact))).astype(np.float64)
    assert float(np.max(np.abs(yf.cpu().numpy().astype(np.longdouble) - exact) / scale)) <= 1e-5


@pytest.mark.parametrize("m", [1, 2, 17, 31, 32])
@pytest.mark.parametrize("n", [32, 33, 127, 4099])
def test_conv1d_limits(cuda_lib, orc, m, n):
    for dt in (np.int64, np.float64):
        sig = orc.random_grid(n, dt, m + n)
        f = orc.random_filter(m, 1, dt, m).reshape(-1)
        for bnd in (0, 1):
            got = cuda_lib.conv1d(sig, f, cuda_lib.KernelConfig(boundary=cuda_lib.Boundary(bnd)))
            assert max_rel_err(got, orc.conv1d(sig, f, bnd)) <= TOL[np.dtype(dt)], (m, n, bnd)


def test_star_arms_random_shapes(cuda_lib):
    """Random star stencils K = 4..6 (shuffled tap order, random weights) on
    random shapes, 1-3 sweeps: the FMA engine with the arms read from shared
    memory (K >= 5) and the chain (K = 4) within tolerance of the oracle."""
    import subprocess, sys, os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "tools/starx_stress.py", "60"], cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert "STARX STRESS PASS" in p.stdout, p.stdout[-2000:] + p.stderr[-2000:]


def test_public_api_fuzz(cuda_lib):
    """15 s of randomised public-API cases (conv2d any m x n with both
    boundaries, stencil2d/3d with random tap sets and catalog stencils,
    conv1d, scan; f32/f64/int64) against the oracle (tools/fuzz.py)."""
    import subprocess, sys, os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "tools/fuzz.py", "15"], cwd=root, capture_output=True,
                       text=True, timeout=600, env=dict(os.environ, FUZZ_SEED="11"))
    assert "FUZZ PASS" in p.stdout, p.stdout[-3000:] + p.stderr[-2000:]


@pytest.mark.parametrize("name,tb", [("3d7pt", 2), ("3d7pt", 3), ("3d13pt", 2), ("poisson", 2)])
def test_fused_ranges_outside_the_buffer(cuda_lib, name, tb):
    """ssam_b200_stencil3d_tb with output planes and ring bounds that lie
    outside the buffer (a slab passes its local ring bounds): the launch is
    clamped to the buffer's interior -- nothing outside the buffer is written
    (guard planes around it stay intact) and the result equals the in-range
    call away from the buffer's ends (launch_tb3d clamped only to
    the ring bounds)."""
    import torch
    from paper_1907_06154_b200 import device as dev
    st = cuda_lib.convert_stencil(cuda_lib.make_benchmark_stencil(name), np.float32)
    k = st.order
    nz, ny, nx = 24, 40, 128
    guard = 8
    big_in = torch.full((nz + 2 * guard, ny, nx), 7.0, dtype=torch.float32, device="cuda")
    a = big_in[guard:guard + nz]
    dev.fill_random(a, 3)
    big_out = torch.full_like(big_in, -5.0)
    b = big_out[guard:guard + nz]
    b.copy_(a)
    ref = a.clone()
    dev.stencil3d_tb(a, ref, st, tb)  # the in-range call
    # outputs requested far past both ends, ring bounds outside the buffer
    dev.stencil3d_tb(a, b, st, tb, -50, nz + 50, -40, nz + 40)
    assert torch.equal(big_out[:guard], torch.full_like(big_out[:guard], -5.0))
    assert torch.equal(big_out[guard + nz:], torch.full_like(big_out[guard + nz:], -5.0))
    # outputs are clamped to the buffer's interior [k, nz - k): its first /
    # last k planes are never written
    assert torch.equal(b[:k], a[:k]) and torch.equal(b[nz - k:], a[nz - k:])
    # away from the buffer's ends (beyond the fused cone) the declared ring
    # makes no difference: equal to the in-range call bit for bit
    c = 2 * k * tb
    assert torch.equal(b[c:nz - c], ref[c:nz - c])
