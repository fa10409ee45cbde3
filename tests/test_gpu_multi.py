"""One process, several devices (ssam_b200_stencil2d_multi / _3d_multi,
csrc/multi.cpp): slabs with k*Tb ghost planes, peer-copied halos overlapped
with the interior.  On a one-GPU box the slabs share device 0 (the peer copy
becomes a device copy; the event graph and every launch are the same), and
the result must equal the one-device entry point BIT FOR BIT and the oracle
within tolerance (N-GPU output bit-identical to 1-GPU)."""
import numpy as np
import pytest

from oracle import Oracle, max_rel_err

pytestmark = pytest.mark.gpu
TOL = {np.dtype(np.float32): 1e-5, np.dtype(np.float64): 1e-12, np.dtype(np.int64): 0.0}


@pytest.fixture(scope="module")
def orc():
    return Oracle()


@pytest.mark.parametrize("name", ["3d7pt", "3d13pt", "3d27pt", "poisson"])
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_multi_3d_bit_identical(cuda_lib, orc, name, dt):
    st = cuda_lib.convert_stencil(cuda_lib.make_benchmark_stencil(name), dt)
    offs = [t.offset for t in st.taps]
    cf = np.asarray([t.coeff for t in st.taps], dt)
    for (nx, ny, nz), iters, ndev in (((64, 40, 48), 5, 2), ((128, 33, 61), 7, 3),
                                      ((64, 16, 97), 4, 4), ((36, 20, 30), 3, 2),
                                      ((33, 21, 40), 5, 3)):  # unaligned rows: direct kernels
        g = orc.random_grid((nz, ny, nx), dt, 11)
        one = cuda_lib.stencil3d(g, st, None, iters)
        got, used = cuda_lib.stencil_multi(g, st, [0] * ndev, None, iters)
        assert used >= 2, (name, nx, ny, nz, ndev)
        assert np.array_equal(got, one), (name, nx, ny, nz, iters, ndev)
        want = orc.stencil3d(g, offs, cf, st.order, iters)
        assert max_rel_err(got, want) <= TOL[np.dtype(dt)]


@pytest.mark.parametrize("name", ["2d5pt", "2d9pt", "2ds25pt"])
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_multi_2d_bit_identical(cuda_lib, orc, name, dt):
    st = cuda_lib.convert_stencil(cuda_lib.make_benchmark_stencil(name), dt)
    offs = [t.offset for t in st.taps]
    cf = np.asarray([t.coeff for t in st.taps], dt)
    for (w, h), iters, ndev in (((256, 200), 9, 2), ((1024, 301), 13, 3), ((130, 150), 5, 4)):
        g = orc.random_grid((h, w), dt, 3)
        one = cuda_lib.stencil2d(g, st, None, iters)
        got, used = cuda_lib.stencil_multi(g, st, [0] * ndev, None, iters)
        assert used >= 2, (name, w, h, ndev)
        assert np.array_equal(got, one), (name, w, h, iters, ndev)
        want = orc.stencil2d(g, offs, cf, st.order, iters)
        assert max_rel_err(got, want) <= TOL[np.dtype(dt)]


def test_multi_int64_and_counters(cuda_lib, orc):
    st = cuda_lib.make_benchmark_stencil("3d7pt")
    ist = cuda_lib.Stencil("i", 3, 1, 0, [cuda_lib.StencilTap(t.offset, np.int64(i + 1))
                                          for i, t in enumerate(st.taps)])
    g = orc.random_grid((40, 24, 32), np.int64, 2)
    c1, c2 = cuda_lib.OpCounters(), cuda_lib.OpCounters()
    one = cuda_lib.stencil3d(g, ist, None, 3, counters=c1)
    got, used = cuda_lib.stencil_multi(g, ist, [0, 0, 0], None, 3, counters=c2)
    assert used == 3 and np.array_equal(got, one)
    assert c1.as_tuple() == c2.as_tuple()


def test_multi_clamps_slab_count(cuda_lib, orc):
    """A slab must own at least k*Tb planes: too many devices for the grid
    run fewer slabs, same result."""
    st = cuda_lib.convert_stencil(cuda_lib.make_benchmark_stencil("3d7pt"), np.float32)
    g = orc.random_grid((9, 16, 32), np.float32, 4)
    one = cuda_lib.stencil3d(g, st, None, 6)
    got, used = cuda_lib.stencil_multi(g, st, [0] * 8, None, 6)
    assert 1 <= used < 8 and np.array_equal(got, one)


def test_multi_rejects_bad_device(cuda_lib):
    st = cuda_lib.convert_stencil(cuda_lib.make_benchmark_stencil("3d7pt"), np.float32)
    g = np.zeros((16, 16, 16), np.float32)
    with pytest.raises(cuda_lib.InvalidArgument):
        cuda_lib.stencil_multi(g, st, [0, 4096])
    with pytest.raises(cuda_lib.InvalidArgument):
        cuda_lib.stencil_multi(g, st, [])


def test_multi_large_slabs(cuda_lib):
    """A larger grid (2048 x 512 x 256 f32, 4 slabs, 12 sweeps: fused pairs
    with the ghost exchange every round) through the device-set path equals
    the one-device call bit for bit."""
    st = cuda_lib.convert_stencil(cuda_lib.make_benchmark_stencil("3d7pt"), np.float32)
    g = cuda_lib.random_grid3d(2048, 512, 256, 7, np.float32)
    one = cuda_lib.stencil3d(g, st, None, 12)
    got, used = cuda_lib.stencil_multi(g, st, [0, 0, 0, 0], None, 12)
    assert used == 4 and np.array_equal(got, one)


def test_multi_headline_size(cuda_lib):
    """The headline grid (2048^2 x 512 f32, 2^31 cells) on 2 and 4 slabs, 12
    sweeps, equal to the one-device call bit for bit: at this size the
    buffers' initial device copies take milliseconds, so a halo copy ordered
    only after the neighbour's boundary launch would race them."""
    st = cuda_lib.convert_stencil(cuda_lib.make_benchmark_stencil("3d7pt"), np.float32)
    g = cuda_lib.random_grid3d(2048, 2048, 512, 0, np.float32)
    one = cuda_lib.stencil3d(g, st, None, 12)
    for n in (2, 4):
        got, used = cuda_lib.stencil_multi(g, st, [0] * n, None, 12)
        assert used == n and np.array_equal(got, one), n
