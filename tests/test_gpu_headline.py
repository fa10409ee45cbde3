"""Parity at the headline and full-size configurations, every cell (-m gpu).

BASELINE.json configs[4] at N = 1 exactly as bench.py runs it: 3d7pt fp32 on
the 2048 x 2048 x 512 grid held in the 2048 x 2048 x (512 + 2 Tb) slab (ghost
planes, > 2^31 elements per buffer), the product's fused depth, 100 sweeps
through the slab runner.  Checked
  * on EVERY cell against the direct-gather kernels (the oracle's tap order
    and double accumulation, oracle.hpp:77-116, on the GPU), max_rel <= 1e-5
    (acceptance.cpp:35-44), and
  * with the exact cone-windowed CPU oracle at global planes
    0, 1, 510, 511 (the slab elements past 2^31), corners and the centre.
configs[0..1]: conv2d 8192^2 K = 3..20, every cell against the gather kernel.
"""
import numpy as np
import pytest

from oracle import max_rel_err, max_abs_err

pytestmark = pytest.mark.gpu

NX = NY = 2048
NZ = 512
ITERS = 100


@pytest.fixture(scope="module")
def headline(cuda_lib):
    import torch
    from paper_1907_06154_b200 import device as dev
    from paper_1907_06154_b200.slab import SlabRunner, decompose, fill_slab
    st = cuda_lib.convert_stencil(cuda_lib.make_benchmark_stencil("3d7pt"), np.float32)
    tb = dev.stencil3d_tb_max(st, np.float32)
    slab = decompose(NZ, 1, 0, st.order, ghost=st.order * tb)
    a = torch.empty((slab.nz_local, NY, NX), dtype=torch.float32, device="cuda")
    assert a.numel() > 2 ** 31
    fill_slab(a, slab, NX, NY, seed=0)
    b = a.clone()
    rlo, rhi = slab.ring_bounds()
    runner = SlabRunner(
        slab, lambda c, n, zb, ze: dev.stencil3d_sweep(c, n, st, zb, ze),
        fused=(lambda c, n, zb, ze: dev.stencil3d_tb(c, n, st, tb, zb, ze, rlo, rhi))
        if tb > 1 else None, tb=tb)
    res = runner.run(a, b, ITERS)
    got = res[slab.local(0):slab.local(0) + NZ].clone()
    del a, b, res
    torch.cuda.empty_cache()
    yield st, tb, got
    del got
    torch.cuda.empty_cache()


def test_headline_every_cell_vs_gather(cuda_lib, headline):
    import torch
    from paper_1907_06154_b200 import device as dev
    st, tb, got = headline
    g0 = torch.empty((NZ, NY, NX), dtype=torch.float32, device="cuda")
    dev.fill_random(g0, 0)
    g1 = torch.empty_like(g0)
    want = dev.gather_run(g0, g1, st, ITERS)
    rel, ab = dev.max_rel_err(got, want)
    # the ring is carried bit for bit
    ring_in = torch.empty((2, NY, NX), dtype=torch.float32, device="cuda")
    dev.fill_random(ring_in[0], 0)
    dev.fill_random(ring_in[1], 0, first=(NZ - 1) * NX * NY)
    assert torch.equal(got[0], ring_in[0]) and torch.equal(got[NZ - 1], ring_in[1])
    del g0, g1, want, ring_in
    torch.cuda.empty_cache()
    assert rel <= 1e-5, (tb, rel, ab)


@pytest.mark.parametrize("z0,y0,x0", [(0, 0, 0), (1, 1000, 1000), (250, 1018, 1018),
                                      (499, 2036, 2036), (500, 0, 2036), (510, 500, 7)])
def test_headline_cone_windows(cuda_lib, orc, headline, z0, y0, x0):
    """Exact windowed oracle for 12^3 output windows (margin k * 100 sweeps)."""
    import torch
    from paper_1907_06154_b200 import device as dev
    st, tb, got = headline
    w = 12
    z1, y1, x1 = min(NZ, z0 + w), min(NY, y0 + w), min(NX, x0 + w)
    mg = st.order * ITERS
    zl, zh = max(0, z0 - mg), min(NZ, z1 + mg)
    yl, yh = max(0, y0 - mg), min(NY, y1 + mg)
    xl, xh = max(0, x0 - mg), min(NX, x1 + mg)
    # input sub-grid straight from the device generator (plane by plane)
    sub = torch.empty((zh - zl, NY, NX), dtype=torch.float32, device="cuda")
    dev.fill_random(sub, 0, first=zl * NX * NY)
    sub_in = sub[:, yl:yh, xl:xh].cpu().numpy()
    del sub
    offs = [t.offset for t in st.taps]
    cf = np.asarray([t.coeff for t in st.taps], np.float32)
    want = orc.stencil3d(sub_in, offs, cf, st.order, ITERS)[z0 - zl:z1 - zl, y0 - yl:y1 - yl,
                                                             x0 - xl:x1 - xl]
    have = got[z0:z1, y0:y1, x0:x1].cpu().numpy()
    assert max_rel_err(have, want) <= 1e-5, (z0, y0, x0, max_abs_err(have, want))


@pytest.mark.parametrize("K", list(range(3, 21)))
def test_conv_8192_every_cell_vs_gather(cuda_lib, orc, K):
    """configs[0..1]: every cell of 8192^2 fp32 K x K (both boundaries) against
    the direct-gather kernel (the oracle's order, double accumulation)."""
    import torch
    from paper_1907_06154_b200 import device as dev
    H = W = 8192
    g = torch.empty((H, W), dtype=torch.float32, device="cuda")
    dev.fill_random(g, 0)
    out = torch.empty_like(g)
    f = orc.random_filter(K, K, np.float32, 1)
    host_in = g.cpu().numpy()
    for bnd in (0, 1):
        dev.conv2d(g, out, f, boundary=bnd)
        want = np.empty_like(host_in)
        cuda_lib._raise(cuda_lib.lib.ssam_b200_gather_conv2d(
            0, host_in.ctypes.data, W, H, np.ascontiguousarray(f).ctypes.data, K, K, bnd,
            want.ctypes.data))
        rel, ab = dev.max_rel_err(out, torch.from_numpy(want).cuda())
        assert rel <= 1e-5, (K, bnd, rel, ab)


@pytest.mark.parametrize("name", ["2d5pt", "2d9pt", "2ds25pt"])
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_2d_8192_x100_every_cell_vs_gather(cuda_lib, name, dt):
    """configs[2]: 8192^2 x 100 sweeps as the product runs them (automatic
    temporal blocking), every cell against the direct-gather kernels."""
    import torch
    from paper_1907_06154_b200 import device as dev
    st = cuda_lib.convert_stencil(cuda_lib.make_benchmark_stencil(name), dt)
    tdt = torch.float32 if dt == np.float32 else torch.float64
    a = torch.empty((8192, 8192), dtype=tdt, device="cuda")
    dev.fill_random(a, 0)
    g0 = a.clone()
    got = dev.stencil2d_run(a, a.clone(), st, 100)
    want = dev.gather_run(g0, g0.clone(), st, 100)
    rel, ab = dev.max_rel_err(got, want)
    assert rel <= (1e-5 if dt == np.float32 else 1e-12), (name, rel, ab)


@pytest.mark.parametrize("name", ["3d7pt", "3d13pt", "3d27pt", "poisson"])
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_3d_512_x100_every_cell_vs_gather(cuda_lib, name, dt):
    """configs[3]: 512^3 x 100 sweeps as the product runs them (fused depth
    per shape), every cell against the direct-gather kernels."""
    import torch
    from paper_1907_06154_b200 import device as dev
    st = cuda_lib.convert_stencil(cuda_lib.make_benchmark_stencil(name), dt)
    tdt = torch.float32 if dt == np.float32 else torch.float64
    a = torch.empty((512, 512, 512), dtype=tdt, device="cuda")
    dev.fill_random(a, 0)
    g0 = a.clone()
    got = dev.stencil3d_run(a, a.clone(), st, 100)
    want = dev.gather_run(g0, g0.clone(), st, 100)
    rel, ab = dev.max_rel_err(got, want)
    assert rel <= (1e-5 if dt == np.float32 else 1e-12), (name, rel, ab)
