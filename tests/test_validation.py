"""The drop-in's error contract equals the reference's (CPU only).

For every argument combination, the status the C ABI returns before touching
the GPU must name the exception the reference throws:
SSAM_ERR_INVALID_ARGUMENT <-> std::invalid_argument,
SSAM_ERR_LENGTH <-> std::length_error, SSAM_OK <-> no exception.
Anchors: proj/tests/test_kernels_conv.cpp:119-134,
proj/tests/test_kernels_stencil.cpp:108-123, :187-204, filter.hpp:76-94, :130-138.
"""
import ctypes
import itertools

import numpy as np
import pytest

from oracle import Oracle


def our_conv_status(lib, w, h, m, n, cfg):
    return lib.lib.ssam_b200_check_conv2d(w, h, m, n, ctypes.byref(cfg._c()))


def our_stencil_status(lib, dims, shape, order, offsets, coeffs, cfg, iters):
    st = lib.Stencil("t", dims, order, 0,
                     [lib.StencilTap(tuple(o), c) for o, c in zip(offsets, coeffs)])
    sa = lib._StencilArgs(st, np.int64)
    if len(shape) == 2:
        return lib.lib.ssam_b200_check_stencil2d(shape[1], shape[0], sa.ref,
                                                 ctypes.byref(cfg._c()), iters)
    return lib.lib.ssam_b200_check_stencil3d(shape[2], shape[1], shape[0], sa.ref,
                                             ctypes.byref(cfg._c()), iters)


# ---- the reference's own error-path tests ----------------------------------------

def test_conv_error_paths(lib):
    cfg = lib.KernelConfig()
    with pytest.raises(lib.InvalidArgument):
        lib.check_conv2d(16, 64, 3, 3, cfg)  # narrower than a warp
    with pytest.raises(lib.InvalidArgument):
        lib.check_conv2d(64, 4, 3, 3, cfg)  # shorter than one cache block
    with pytest.raises(lib.InvalidArgument):
        lib.check_conv2d(64, 64, 21, 3, cfg)
    with pytest.raises(lib.LengthError):
        lib.check_conv2d(64, 300, 3, 8, lib.KernelConfig(p=250))  # C = 257
    lib.check_conv2d(64, 64, 20, 20, cfg)


def test_stencil_error_paths(lib):
    cfg = lib.KernelConfig()
    st = lib.make_benchmark_stencil("2d5pt")
    with pytest.raises(lib.InvalidArgument):
        lib.check_stencil2d(2, 2, st, cfg, 1)
    with pytest.raises(lib.InvalidArgument):
        lib.check_stencil2d(64, 64, st, cfg, 0)
    dup = lib.Stencil("dup", 2, 1, 0, [lib.StencilTap((0, 0, 0), 1.0),
                                       lib.StencilTap((0, 0, 0), 2.0)])
    with pytest.raises(lib.InvalidArgument):
        lib.check_stencil2d(64, 64, dup, cfg, 1)
    with pytest.raises(lib.InvalidArgument):
        lib.check_stencil2d(64, 64, lib.make_benchmark_stencil("3d7pt"), cfg, 1)
    st13 = lib.make_benchmark_stencil("3d13pt")  # k = 2 needs 5 warps
    with pytest.raises(lib.InvalidArgument):
        lib.check_stencil3d(32, 12, 10, st13, lib.KernelConfig(p=2, b=128), 1)
    with pytest.raises(lib.InvalidArgument):
        lib.check_stencil3d(32, 12, 10, st, lib.KernelConfig(p=2, b=256), 1)
    with pytest.raises(lib.InvalidArgument):
        lib.check_stencil3d(32, 12, 3, st13, lib.KernelConfig(p=2, b=256), 1)
    lib.check_stencil3d(32, 12, 10, st13, lib.KernelConfig(p=2, b=256), 1)


# ---- exhaustive agreement with the reference -------------------------------------

def test_conv_status_matches_reference_sweep(lib, ref):
    orc = Oracle()
    g_cache = {}
    mismatches = []
    for (w, h), (m, n), p, b, lc in itertools.product(
            [(16, 40), (33, 9), (64, 64)], [(1, 1), (3, 3), (20, 5), (21, 3), (3, 21), (17, 17)],
            [0, 1, 4, 250], [0, 32, 48, 128], [1, 3, 16, 32, 64, 128]):
        cfg = lib.KernelConfig(p=p, b=b, lane_count=lc)
        ours = our_conv_status(lib, w, h, m, n, cfg)
        if (w, h) not in g_cache:
            g_cache[(w, h)] = orc.random_grid((h, w), np.int64, 1)
        f = np.ones((m, n), np.int64)
        rc, _, _ = ref.conv2d(g_cache[(w, h)], f, p=p, b=b, lane_count=lc)
        if rc != ours:
            mismatches.append(((w, h, m, n, p, b, lc), ours, rc))
    assert not mismatches, mismatches[:10]


STENCIL_CASES = [
    # (dims, shape, order, offsets, coeffs)
    (2, (40, 64), 1, [(0, 0, 0), (1, 0, 0)], [1, 2]),
    (2, (40, 64), 2, [(0, 0, 0), (1, 0, 0)], [1, 2]),            # order mismatch
    (2, (40, 64), 1, [(0, 0, 1)], [1]),                          # z offset in 2D
    (2, (40, 64), 1, [(0, 0, 0), (0, 0, 0)], [1, 2]),            # duplicate
    (2, (40, 64), 1, [(2, 0, 0)], [1]),                          # outside order
    (2, (2, 2), 1, [(0, 0, 0), (1, 0, 0)], [1, 2]),              # domain too small
    (2, (40, 64), 16, [(16, 0, 0)], [1]),                        # m = 33 > lanes
    (2, (40, 64), 0, [(0, 0, 0)], [1]),
    (3, (8, 12, 32), 1, [(0, 0, 0), (0, 0, 1)], [1, 2]),
    (3, (8, 12, 32), 2, [(0, 0, 2)], [1]),
    (3, (3, 12, 32), 2, [(0, 0, 2)], [1]),
    (1, (40, 64), 1, [(1, 0, 0)], [1]),                          # bad dims
]


@pytest.mark.parametrize("case", range(len(STENCIL_CASES)))
def test_stencil_status_matches_reference(lib, ref, case):
    dims, shape, order, offs, cfs = STENCIL_CASES[case]
    orc = Oracle()
    for kernel_dims in (2, 3):
        if len(shape) != kernel_dims:
            continue
        for p, b, lc, iters in itertools.product([0, 1, 2], [32, 128, 256], [16, 32], [0, 1]):
            cfg = lib.KernelConfig(p=p, b=b, lane_count=lc)
            ours = our_stencil_status(lib, dims, shape, order, offs, cfs, cfg, iters)
            g = orc.random_grid(shape, np.int64, 5)
            if kernel_dims == 2:
                rc, _, _ = ref.stencil2d(g, offs, np.asarray(cfs, np.int64), order, iters,
                                         dims=dims, p=p, b=b, lane_count=lc)
            else:
                rc, _, _ = ref.stencil3d(g, offs, np.asarray(cfs, np.int64), order, iters,
                                         dims=dims, p=p, b=b, lane_count=lc)
            assert rc == ours, (case, p, b, lc, iters, ours, rc)
