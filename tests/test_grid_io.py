"""SGRD grid files (proj/include/ssam/grid_io.hpp:14-158) through the C ABI.

CPU: host-buffer round trips, byte-identical files to the reference's own
writer (oracle/_ref), our reader on the reference's files, and the error
contract of proj/tests/test_grid_io.cpp:33-57 (bad magic, version, rank,
scalar type, truncation -> std::runtime_error; dims > 65535 ->
std::invalid_argument).  GPU (-m gpu): device buffers streamed through the
pinned staging path, including a payload larger than one 64 MiB chunk.
"""
import os

import numpy as np
import pytest


@pytest.fixture
def tmp(tmp_path):
    return lambda name: str(tmp_path / name)


def _grids(orc):
    return [orc.random_grid((17, 33), np.float64, 1), orc.random_grid((5, 6, 7), np.int64, 2),
            orc.random_grid(41, np.float32, 3), orc.random_grid((1, 65535), np.float32, 4)]


def test_round_trip_host(lib, orc, tmp):
    for i, g in enumerate(_grids(orc)):
        p = tmp(f"g{i}.sgrd")
        lib.write_grid(p, g)
        rank, dt, dims = lib.sgrd_info(p)
        assert rank == g.ndim and dt == g.dtype.type
        read = {1: lib.read_vector, 2: lib.read_grid2d, 3: lib.read_grid3d}[g.ndim]
        back = read(p, g.dtype)
        assert back.shape == g.shape and np.array_equal(back, g)


def test_files_identical_to_reference_writer(lib, orc, ref, tmp):
    for i, g in enumerate(_grids(orc)):
        ours, theirs = tmp(f"o{i}.sgrd"), tmp(f"r{i}.sgrd")
        lib.write_grid(ours, g)
        assert ref.sgrd_write(theirs, g) == 0
        assert open(ours, "rb").read() == open(theirs, "rb").read()
        rc, back = ref.sgrd_read(ours, g.dtype, g.ndim)
        assert rc == 0 and np.array_equal(back, g)


def test_error_contract(lib, orc, ref, tmp):
    g = orc.random_grid((4, 3), np.float64, 5)
    good = tmp("ok.sgrd")
    lib.write_grid(good, g)
    data = open(good, "rb").read()
    cases = {
        "magic": b"XGRD" + data[4:],
        "version": data[:4] + b"\x02" + data[5:],
        "short_header": data[:10],
        "truncated": data[:-3],
    }
    for name, blob in cases.items():
        p = tmp(name + ".sgrd")
        open(p, "wb").write(blob)
        with pytest.raises(lib.GridIOError):
            lib.read_grid2d(p, np.float64)
        assert ref.sgrd_read(p, np.float64, 2)[0] == 3, name  # std::runtime_error
    with pytest.raises(lib.GridIOError):      # scalar type mismatch
        lib.read_grid2d(good, np.float32)
    assert ref.sgrd_read(good, np.float32, 2)[0] == 3
    with pytest.raises(lib.GridIOError):      # rank mismatch
        lib.read_grid3d(good, np.float64)
    assert ref.sgrd_read(good, np.float64, 3)[0] == 3
    with pytest.raises(lib.GridIOError):      # missing file
        lib.read_grid2d(tmp("absent.sgrd"), np.float64)
    big = np.zeros(65536, np.float32)         # dims limit
    with pytest.raises(lib.InvalidArgument):
        lib.write_grid(tmp("big.sgrd"), big)
    assert ref.sgrd_write(tmp("bigr.sgrd"), big) == 1
    # both open (and truncate) the file before rejecting the dimensions
    assert os.path.exists(tmp("big.sgrd")) and os.path.getsize(tmp("big.sgrd")) == 0
    assert os.path.exists(tmp("bigr.sgrd")) and os.path.getsize(tmp("bigr.sgrd")) == 0
    # an unopenable path with oversize dims: the open failure wins (runtime_error)
    with pytest.raises(lib.GridIOError):
        lib.write_grid(tmp("no/such/dir/big.sgrd"), big)
    assert ref.sgrd_write(tmp("no/such/dir/bigr.sgrd"), big) == 3
    # a header with an empty dimension: Grid2D / Grid3D reject it (invalid_argument)
    for rank, dt, shape in ((2, np.float64, (4, 3)), (3, np.float64, (2, 3, 4))):
        src = tmp(f"z{rank}.sgrd")
        lib.write_grid(src, orc.random_grid(shape, dt, 1))
        blob = bytearray(open(src, "rb").read())
        blob[8:10] = b"\x00\x00"            # dims[0] = 0
        bad = tmp(f"zero{rank}.sgrd")
        open(bad, "wb").write(bytes(blob[:16]))
        read = lib.read_grid2d if rank == 2 else lib.read_grid3d
        with pytest.raises(lib.InvalidArgument):
            read(bad, dt)
        assert ref.sgrd_read(bad, dt, rank)[0] == 1


@pytest.mark.gpu
def test_device_round_trip(cuda_lib, orc, tmp):
    import torch
    from paper_1907_06154_b200 import device as dev
    # 3D f32 of 80 MiB: two staging chunks, the second partial
    nx, ny, nz = 1024, 640, 32
    a = torch.empty((nz, ny, nx), dtype=torch.float32, device="cuda")
    dev.fill_random(a, 7)
    p = tmp("dev.sgrd")
    dev.write_grid(p, a)
    assert os.path.getsize(p) == 16 + a.numel() * 4
    host = cuda_lib.read_grid3d(p, np.float32)
    assert np.array_equal(host, a.cpu().numpy())
    b = dev.read_grid(p)
    assert b.shape == a.shape and torch.equal(a, b)
    # reference-format reader on a small int64 grid written from the device
    g = orc.random_grid((9, 11), np.int64, 3)
    t = torch.from_numpy(g).cuda()
    dev.write_grid(tmp("i.sgrd"), t)
    assert np.array_equal(cuda_lib.read_grid2d(tmp("i.sgrd"), np.int64), g)
