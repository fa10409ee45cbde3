"""conv2d on the GPU vs the oracle (run with -m gpu on a B200).

Mirrors proj/tests/test_kernels_conv.cpp and acceptance criterion 1
(proj/tests/acceptance.cpp:47-73); full-size fp32 parity at 8192^2 across the
K = 3..20 sweep uses the exact row-band oracle of tests/windows.py.
Tolerances (proj/tools/ssam_cli.cpp:48-55): int64 bit-exact, f64 <= 1e-12,
f32 <= 1e-5, all as max |got-want| / max(1, |want|).
"""
import hashlib

import numpy as np
import pytest

import cases as C
from oracle import Oracle, max_rel_err
from windows import conv2d_rows

pytestmark = pytest.mark.gpu
NP = {"f32": np.float32, "f64": np.float64, "i64": np.int64}
TOL = {np.dtype(np.float32): 1e-5, np.dtype(np.float64): 1e-12, np.dtype(np.int64): 0.0}


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_identity_filter(cuda_lib, orc):
    g = orc.random_grid((40, 64), np.int64, 1)
    assert np.array_equal(cuda_lib.conv2d(g, cuda_lib.Filter2D()), g)


def test_constant_times_weight_sum(cuda_lib):
    g = np.full((33, 64), 5, np.int64)
    f = np.array([2, 0, 1, -1, 3, 1, 0, 2, 2], np.int64).reshape(3, 3)
    out = cuda_lib.conv2d(g, f)
    assert np.all(out[1:32, 1:63] == 50)


def test_criterion1_int_bit_exact(cuda_lib, orc, golden):
    """acceptance.cpp:47-73 -- 10 seeds x 22 filters, 128^2, zero boundary."""
    for seed in range(10):
        g = orc.random_grid((128, 128), np.int64, seed)
        for m, n in C.CONV_INT_SHAPES:
            f = orc.random_filter(m, n, np.int64, seed * 1000 + m * 31 + n)
            got = cuda_lib.conv2d(g, f)
            want = orc.conv2d(g, f, 0)
            assert np.array_equal(got, want), (seed, m, n)
            tag = f"c1_s{seed}_{m}x{n}"
            if tag in golden["conv"]:
                assert digest(got) == golden["conv"][tag]["oracle"]


def test_unit_shapes_both_boundaries(cuda_lib, orc, golden):
    for tag, dt, w, h, m, n, gs, fs, bnd in C.conv_cases():
        if not tag.startswith("unit_"):
            continue
        g = orc.random_grid((h, w), NP[dt], gs)
        f = orc.random_filter(m, n, NP[dt], fs)
        cfg = cuda_lib.KernelConfig(boundary=cuda_lib.Boundary(bnd))
        got = cuda_lib.conv2d(g, f, cfg)
        assert digest(got) == golden["conv"][tag]["oracle"], tag


def test_f64_within_1e12(cuda_lib, orc):
    g = orc.random_grid((48, 96), np.float64, 9)
    f = orc.random_filter(5, 4, np.float64, 10)
    assert max_rel_err(cuda_lib.conv2d(g, f), orc.conv2d(g, f, 0)) < 1e-12


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_float_cases_vs_oracle(cuda_lib, orc, dt):
    for tag, cdt, w, h, m, n, gs, fs, bnd in C.conv_cases():
        if cdt != dt:
            continue
        g = orc.random_grid((h, w), NP[dt], gs)
        f = orc.random_filter(m, n, NP[dt], fs)
        got = cuda_lib.conv2d(g, f, cuda_lib.KernelConfig(boundary=cuda_lib.Boundary(bnd)))
        assert max_rel_err(got, orc.conv2d(g, f, bnd)) <= TOL[np.dtype(NP[dt])], tag


def test_randomized_configs_int(cuda_lib, orc):
    """test_kernels_conv.cpp:189-206 -- 30 random (w,h,m,n,p,b,boundary)."""
    rng = np.random.default_rng(4096)
    for _ in range(30):
        m, n = (int(v) for v in rng.integers(1, 21, size=2))
        p = int(rng.integers(1, 9))
        b = 32 * int(rng.integers(1, 7))
        bnd = int(rng.integers(0, 2))
        w = int(rng.integers(32, 201))
        h = int(rng.integers(n + p - 1, 151))
        g = orc.random_grid((h, w), np.int64, int(rng.integers(1 << 62)))
        f = orc.random_filter(m, n, np.int64, int(rng.integers(1 << 62)))
        cfg = cuda_lib.KernelConfig(p=p, b=b, boundary=cuda_lib.Boundary(bnd))
        assert np.array_equal(cuda_lib.conv2d(g, f, cfg), orc.conv2d(g, f, bnd)), (w, h, m, n)


@pytest.mark.parametrize("dt", [np.float32, np.float64, np.int64])
def test_unaligned_widths_all_shapes(cuda_lib, orc, dt):
    """Odd widths take the scalar load path; every (m, n) in 1..20 on both boundaries."""
    g = orc.random_grid((45, 97), dt, 77)
    for m in (1, 2, 3, 7, 12, 20):
        for n in (1, 4, 9, 20):
            f = orc.random_filter(m, n, dt, 100 * m + n)
            for bnd in (0, 1):
                got = cuda_lib.conv2d(g, f, cuda_lib.KernelConfig(boundary=cuda_lib.Boundary(bnd)))
                assert max_rel_err(got, orc.conv2d(g, f, bnd)) <= TOL[np.dtype(dt)], (m, n, bnd)


def test_lane_count_16(cuda_lib, orc):
    cfg = cuda_lib.KernelConfig(lane_count=16, b=32)
    g = orc.random_grid((24, 48), np.int64, 5)
    f = orc.random_filter(4, 3, np.int64, 6)
    assert np.array_equal(cuda_lib.conv2d(g, f, cfg), orc.conv2d(g, f, 0))


def test_counters_from_gpu_call(cuda_lib, orc):
    g = orc.random_grid((50, 100), np.int64, 3)
    f = orc.random_filter(3, 3, np.int64, 4)
    c = cuda_lib.OpCounters()
    cuda_lib.conv2d(g, f, cuda_lib.KernelConfig(), c)
    tiles = 52
    assert c.as_tuple() == (tiles * 36, tiles * 8, tiles * 36, tiles * 32 * 6, 5000)
    cuda_lib.conv2d(g, f, cuda_lib.KernelConfig(), c)  # accumulates
    assert c.global_stores == 10000


def test_deterministic(cuda_lib, orc):
    g = orc.random_grid((64, 128), np.float64, 17)
    f = orc.random_filter(4, 6, np.float64, 18)
    a = cuda_lib.conv2d(g, f, cuda_lib.KernelConfig(threads=1))
    b = cuda_lib.conv2d(g, f, cuda_lib.KernelConfig(threads=2, p=7, b=64))
    assert np.array_equal(a, b)


@pytest.mark.parametrize("K", list(range(3, 21)))
def test_f32_8192_sweep(cuda_lib, orc, K):
    """configs[0..1]: 8192^2 fp32, K x K, seeds (0, 1) as the CLI draws them;
    checked on row bands at the top, bottom and middle with the exact oracle."""
    import torch
    from paper_1907_06154_b200 import device as dev
    H = W = 8192
    g = torch.empty((H, W), dtype=torch.float32, device="cuda")
    dev.fill_random(g, 0)
    out = torch.empty_like(g)
    f = orc.random_filter(K, K, np.float32, 1)
    for bnd in (0, 1):
        dev.conv2d(g, out, f, boundary=bnd)
        torch.cuda.synchronize()
        host_in = g.cpu().numpy()
        host_out = out.cpu().numpy()
        worst = 0.0
        for y0, y1 in ((0, 24), (4090, 4106), (H - 24, H)):
            want = conv2d_rows(orc, host_in, f, bnd, y0, y1)
            worst = max(worst, max_rel_err(host_out[y0:y1], want))
        assert worst <= 1e-5, (K, bnd, worst)
    # the device generator is the reference's random_grid2d bit-for-bit
    assert np.array_equal(host_in[:2].reshape(-1), orc.random_grid(2 * W, np.float32, 0))
