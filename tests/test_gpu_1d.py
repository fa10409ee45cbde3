"""conv1d and scan on the GPU vs the oracle (run with -m gpu on a B200).

Mirrors proj/tests/test_kernels_conv.cpp:136-187, :210-221 and acceptance
criterion 3 (proj/tests/acceptance.cpp:116-135: 1000 random int64 scans of
1..127 tiles, exact).  Tolerances (ssam_cli.cpp:48-55): int64 bit-exact,
f64 <= 1e-12, f32 <= 1e-5 as max |got-want| / max(1, |want|).
"""
import hashlib

import numpy as np
import pytest

import cases as C
from oracle import max_rel_err

pytestmark = pytest.mark.gpu
NP = {"f32": np.float32, "f64": np.float64, "i64": np.int64}
TOL = {"f32": 1e-5, "f64": 1e-12, "i64": 0.0}


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_conv1d_identity_and_box(cuda_lib):
    ramp = np.arange(100, dtype=np.int64)
    assert np.array_equal(cuda_lib.conv1d(ramp, [1]), ramp)
    out = cuda_lib.conv1d(ramp, np.ones(5, np.int64))
    assert all(out[i] == 5 * i for i in range(2, 98))


def test_conv1d_golden(cuda_lib, orc, golden):
    for tag, dt, n, m, ss, fs, bnd, lanes in C.conv1d_cases():
        sig = orc.random_grid(n, NP[dt], ss)
        f = orc.random_filter(m, 1, NP[dt], fs).reshape(-1)
        cnt = cuda_lib.OpCounters()
        got = cuda_lib.conv1d(sig, f, cuda_lib.KernelConfig(boundary=cuda_lib.Boundary(bnd),
                                                            lane_count=lanes), cnt)
        if dt == "i64":
            assert digest(got) == golden["conv1d"][tag]["oracle"], tag
        else:
            assert max_rel_err(got, orc.conv1d(sig, f, bnd)) <= TOL[dt], tag
        assert list(cnt.as_tuple()) == golden["conv1d"][tag]["counters"], tag


def test_conv1d_random_vs_oracle(cuda_lib, orc):
    rng = np.random.default_rng(8)
    for dt in ("i64", "f32", "f64"):
        for _ in range(20):
            m = int(rng.integers(1, 33))
            n = int(rng.integers(32, 5000))
            bnd = int(rng.integers(0, 2))
            sig = orc.random_grid(n, NP[dt], int(rng.integers(1 << 40)))
            f = orc.random_filter(m, 1, NP[dt], int(rng.integers(1 << 40))).reshape(-1)
            got = cuda_lib.conv1d(sig, f, cuda_lib.KernelConfig(boundary=cuda_lib.Boundary(bnd)))
            assert max_rel_err(got, orc.conv1d(sig, f, bnd)) <= TOL[dt], (dt, n, m, bnd)


def test_conv1d_large(cuda_lib, orc):
    n = (1 << 22) + 3
    sig = orc.random_grid(n, np.float32, 1)
    f = orc.random_filter(9, 1, np.float32, 2).reshape(-1)
    assert max_rel_err(cuda_lib.conv1d(sig, f), orc.conv1d(sig, f, 0)) <= 1e-5


def test_scan_reference_cases(cuda_lib, orc):
    cnt = cuda_lib.OpCounters()
    out = cuda_lib.scan(np.ones(96, np.int64), 32, cnt)
    assert out.tolist() == list(range(1, 97))
    assert cnt.shuffles == 15
    alt = np.array([1 if i % 2 == 0 else -1 for i in range(64)], np.int64)
    assert cuda_lib.scan(alt).tolist() == [1 if i % 2 == 0 else 0 for i in range(64)]
    assert cuda_lib.scan(np.zeros(0, np.int64)).size == 0
    with pytest.raises(cuda_lib.InvalidArgument):
        cuda_lib.scan(np.ones(33, np.int64))
    v = np.random.default_rng(9).integers(-50, 50, 48).astype(np.int64)
    cnt = cuda_lib.OpCounters()
    assert np.array_equal(cuda_lib.scan(v, 16, cnt), orc.scan(v))
    assert cnt.shuffles == 12


def test_scan_golden(cuda_lib, orc, golden):
    for tag, dt, n, seed, lanes in C.scan_cases():
        v = orc.random_grid(n, NP[dt], seed)
        got = cuda_lib.scan(v, lanes)
        if dt == "i64":
            assert digest(got) == golden["scan"][tag]["oracle"], tag
        else:
            assert max_rel_err(got, orc.scan(v)) <= TOL[dt], tag


def test_scan_criterion3_property(cuda_lib, orc):
    """acceptance.cpp:116-135: 1000 random int64 inputs of 1..127 tiles, exact."""
    rng = np.random.default_rng(100)
    for _ in range(1000):
        tiles = int(rng.integers(1, 128))
        v = rng.integers(-1000000, 1000001, 32 * tiles).astype(np.int64)
        assert np.array_equal(cuda_lib.scan(v), orc.scan(v)), tiles


def test_scan_large_multi_tile(cuda_lib, orc):
    """Many tiles and L2 chunks: 2^24 + 32 elements (int64 exact, f64 / f32 within tolerance)."""
    n = (1 << 24) + 32
    v = np.random.default_rng(3).integers(-1 << 20, 1 << 20, n).astype(np.int64)
    assert np.array_equal(cuda_lib.scan(v), orc.scan(v))
    # Long floating prefix sums: every summation order (the oracle's serial
    # one included) carries ~sqrt(n) ulps of the largest partial sum seen so
    # far, so the per-element metric is taken against the running max |S|
    # and an extended-precision cumsum.
    for dt, tol in ((np.float64, 1e-12), (np.float32, 1e-5)):
        x = orc.random_grid(n, dt, 4)
        exact = np.cumsum(x.astype(np.longdouble))
        scale = np.maximum(1.0, np.maximum.accumulate(np.abs(exact))).astype(np.float64)
        got = cuda_lib.scan(x).astype(np.longdouble)
        assert float(np.max(np.abs(got - exact) / scale)) <= tol, dt


def test_scan_deterministic(cuda_lib, orc):
    """Chunked scan with fixed-order tile prefixes (scan.cu): repeated runs are
    bit-identical for floating point too, whatever the tile timing."""
    n = (1 << 22) + 96
    for dt in (np.float32, np.float64):
        x = orc.random_grid(n, dt, 12)
        first = cuda_lib.scan(x)
        for _ in range(4):
            assert np.array_equal(cuda_lib.scan(x), first)


def test_scan_chunk_boundaries(cuda_lib, orc):
    """Lengths around the L2-chunk edges of scan.cu (384 tiles of 4096 int64 /
    8192 fp32 elements): under one chunk, exactly one, a lane row over, two
    chunks less a row, ragged last tiles (lengths are lane_count multiples).  int64 exact; fp32 against the
    float64 prefix with the running-max scale."""
    rng = np.random.default_rng(21)
    for tiles, extra in ((383, 0), (384, 0), (384, 32), (385, -64), (768, -32), (769, 96)):
        n = tiles * 4096 + extra
        v = rng.integers(-1 << 30, 1 << 30, n).astype(np.int64)
        assert np.array_equal(cuda_lib.scan(v), orc.scan(v)), (tiles, extra)
    for tiles, extra in ((384, 0), (385, 160), (768, -32)):
        x = orc.random_grid(tiles * 8192 + extra, np.float32, 5)
        exact = np.cumsum(x.astype(np.float64))
        scale = np.maximum(1.0, np.maximum.accumulate(np.abs(exact)))
        assert float(np.max(np.abs(cuda_lib.scan(x) - exact) / scale)) <= 1e-5, tiles


def test_scan_device_unaligned_views():
    """Device scan on views whose base is off the 32-byte (64-bit) / 16-byte
    (fp32) vector alignment: the tiles take the scalar path, same results."""
    import torch
    from paper_1907_06154_b200 import device as dev
    n = 384 * 4096 + 4096 + 160
    g = torch.Generator().manual_seed(5)
    base = torch.randint(-1 << 30, 1 << 30, (n + 8,), generator=g, dtype=torch.int64).cuda()
    for off_in, off_out in ((1, 3), (2, 0), (0, 2), (4, 4)):
        x = base[off_in:off_in + n]
        y = torch.zeros(n + 8, dtype=torch.int64, device="cuda")[off_out:off_out + n]
        dev.scan(x, y)
        assert torch.equal(y, torch.cumsum(x, 0)), (off_in, off_out)
    xf = torch.rand(n + 8, generator=g, dtype=torch.float64).cuda()
    for off in (1, 2):
        x = xf[off:off + n]
        y = torch.empty(n + 8, dtype=torch.float64, device="cuda")[off:off + n]
        dev.scan(x, y)
        ref = torch.cumsum(x, 0)
        assert float(((y - ref).abs() / ref.abs().clamp_min(1)).max()) <= 1e-12, off
    x32 = torch.rand(n + 8, generator=g, dtype=torch.float32).cuda()[1:n + 1]
    y32 = torch.empty(n + 8, dtype=torch.float32, device="cuda")[1:n + 1]
    dev.scan(x32, y32)
    ref = torch.cumsum(x32.double(), 0)
    assert float(((y32.double() - ref).abs() / ref.abs().clamp_min(1)).max()) <= 1e-5


def test_conv1d_device_unaligned_views():
    """conv1d on views off the 32-byte vector alignment (scalar loads) equals
    the aligned run bit for bit, fp32 and fp64, zero and replicate edges."""
    import torch
    from paper_1907_06154_b200 import device as dev
    n = 100000
    g = torch.Generator().manual_seed(9)
    for dt in (torch.float32, torch.float64):
        base = torch.rand(n + 8, generator=g, dtype=dt).cuda()
        for m in (3, 9, 32):
            w = np.linspace(-1, 1, m)
            for bnd in (0, 1):
                ref_in = base[:n].clone()
                ref = torch.empty_like(ref_in)
                dev.conv1d(ref_in, ref, w, bnd)
                for off in (1, 2, 3):
                    x = base.clone()[off:off + n]
                    x.copy_(base[:n])
                    y = torch.empty(n + 8, dtype=dt, device="cuda")[off:off + n]
                    dev.conv1d(x, y, w, bnd)
                    assert torch.equal(y, ref), (dt, m, bnd, off)


def test_scan_device_in_place():
    """d_out == d_in (ssam_b200.h): every chunk's tiles are read before they
    are written, int64 exact, fp32 equal to the out-of-place result."""
    import torch
    from paper_1907_06154_b200 import device as dev
    n = 3 * 384 * 4096 + 4096 + 96
    g = torch.Generator().manual_seed(13)
    x = torch.randint(-1 << 30, 1 << 30, (n,), generator=g, dtype=torch.int64).cuda()
    want = torch.cumsum(x, 0)
    dev.scan(x, x)
    assert torch.equal(x, want)
    f = torch.rand(n, generator=g, dtype=torch.float32).cuda()
    ref = torch.empty_like(f)
    dev.scan(f, ref)
    dev.scan(f, f)
    assert torch.equal(f, ref)
