"""Golden case definitions shared by make_golden.py (generator) and the tests.

Every case is a small, seeded input drawn with the reference's own SplitMix64
conventions.  make_golden.py runs the UNMODIFIED reference (oracle/_ref) on
each case and records a SHA-256 of its output bytes (plus counters for the
reference's CPU SSAM path); the tests recompute the same cases with our C
restatement (oracle/) and, on the GPU, with the CUDA path.

Sources of the case lists (relative to /root/reference):
  CONV_INT_SHAPES ....... proj/tests/acceptance.cpp:49-54 (criterion 1)
  CONV_UNIT_SHAPES ...... proj/tests/test_kernels_conv.cpp:47-48
  stencil cases ......... proj/tests/acceptance.cpp:76-114 (criterion 2),
                          proj/tests/test_kernels_stencil.cpp:59-106, 155-185
  conv1d / scan cases ... proj/tests/test_kernels_conv.cpp:136-187, :210-221,
                          proj/tests/acceptance.cpp:116-135 (criterion 3)
"""
from __future__ import annotations

CONV_INT_SHAPES = [(k, k) for k in range(2, 21)] + [(3, 5), (5, 3), (2, 7)]
CONV_UNIT_SHAPES = [(2, 2), (3, 3), (5, 5), (8, 8), (13, 13), (20, 20), (3, 5), (5, 3), (2, 7),
                    (1, 4), (7, 1)]

NAMES_2D = ["2d5pt", "2d9pt", "2d13pt", "2d17pt", "2d21pt", "2ds25pt", "2d25pt", "2d64pt",
            "2d81pt", "2d121pt"]
NAMES_3D = ["3d7pt", "3d13pt", "3d27pt", "3d125pt", "poisson"]
NORTH_STAR_2D = ["2d5pt", "2d9pt", "2ds25pt"]
NORTH_STAR_3D = ["3d7pt", "3d13pt", "3d27pt", "poisson"]

# The integer stencil of test_kernels_stencil.cpp:62-65.
INT_STENCIL_2D = dict(order=2, offsets=[(0, 0, 0), (-1, 0, 0), (2, 0, 0), (0, -2, 0), (1, 1, 0),
                                        (-2, 2, 0)],
                      coeffs=[3, 2, -1, 4, 5, 1])
# test_kernels_stencil.cpp:172-175
INT_STENCIL_3D = dict(order=1, offsets=[(0, 0, 0), (1, 0, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)],
                      coeffs=[2, -3, 1, 4, 5])


def conv_cases():
    """(tag, dtype, w, h, m, n, grid_seed, filter_seed, boundary)."""
    cases = []
    # criterion 1: seeds 0..2 of the 10 (the rest are covered on the GPU by recomputation)
    for seed in range(3):
        for m, n in CONV_INT_SHAPES:
            cases.append((f"c1_s{seed}_{m}x{n}", "i64", 128, 128, m, n, seed,
                          seed * 1000 + m * 31 + n, 0))
    for bnd in (0, 1):
        for i, (m, n) in enumerate(CONV_UNIT_SHAPES):
            cases.append((f"unit_b{bnd}_{m}x{n}", "i64", 97, 61, m, n, 4200 + i, 5200 + i, bnd))
    cases.append(("f64_96x48_5x4", "f64", 96, 48, 5, 4, 9, 10, 0))
    for k in (3, 5, 11, 20):
        cases.append((f"f32_256_{k}x{k}", "f32", 256, 256, k, k, 0, 1, 0))
        cases.append((f"f32_256_{k}x{k}_repl", "f32", 256, 256, k, k, 0, 1, 1))
    return cases


def stencil2d_cases():
    """(tag, dtype, w, h, name_or_None, grid_seed, iters)."""
    cases = []
    for name in NAMES_2D:
        cases.append((f"{name}_f64", "f64", 256, 256, name, 11, 4))
        cases.append((f"{name}_f32", "f32", 256, 256, name, 11, 4))
    for it in (1, 2, 4):
        cases.append((f"int_it{it}", "i64", 80, 52, None, 12, it))
    return cases


def stencil3d_cases():
    """(tag, dtype, nx, ny, nz, name_or_None, grid_seed, iters)."""
    cases = []
    for name in NAMES_3D:
        cases.append((f"{name}_f64", "f64", 64, 64, 64, name, 13, 2))
        cases.append((f"{name}_f32", "f32", 64, 64, 64, name, 13, 2))
    cases.append(("int3d", "i64", 36, 10, 9, None, 31, 2))
    return cases


def conv1d_cases():
    """(tag, dtype, len, m, signal_seed, filter_seed, boundary, lane_count).
    Signal = random_grid stream of `len`, filter = random_filter(m, 1)."""
    cases = []
    for bnd in (0, 1):
        for m in (1, 2, 3, 9, 32):
            cases.append((f"i64_211_m{m}_b{bnd}", "i64", 211, m, 8 + m, 80 + m, bnd, 32))
        for m in (5, 16):
            cases.append((f"f32_4099_m{m}_b{bnd}", "f32", 4099, m, 3, 4, bnd, 32))
            cases.append((f"f64_4099_m{m}_b{bnd}", "f64", 4099, m, 3, 4, bnd, 32))
    cases.append(("i64_48_m7_l16", "i64", 48, 7, 5, 6, 0, 16))
    return cases


def scan_cases():
    """(tag, dtype, len, seed, lane_count)."""
    cases = []
    for tiles in (1, 3, 7, 128):
        cases.append((f"i64_t{tiles}", "i64", 32 * tiles, 55 + tiles, 32))
    cases.append(("i64_l16", "i64", 48, 9, 16))
    cases.append(("f64_4096", "f64", 4096, 2, 32))
    cases.append(("f32_4096", "f32", 4096, 2, 32))
    return cases
