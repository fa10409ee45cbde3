"""conv1d / scan (kernels.hpp:390-447): oracle, counters and error contract (CPU only).

* oracle: the hand fixtures of proj/tests/test_oracle.cpp:112-129 and the
  golden digests of the reference's conv1d_naive / scan_naive
  (tests/golden/golden.json, made by tests/golden/make_golden.py);
* counters: the closed forms against the reference simulator's tallies;
* errors: the C ABI's validation against the compiled reference for a
  sweep of (len, m, lane_count) -- std::invalid_argument <-> SSAM_ERR_INVALID_ARGUMENT.
"""
import hashlib
import itertools

import numpy as np
import pytest

import cases as C

NP = {"f32": np.float32, "f64": np.float64, "i64": np.int64}


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_oracle_fixtures(orc):
    """proj/tests/test_oracle.cpp:112-129."""
    s = orc.scan(np.ones(10, np.int64))
    assert s.tolist() == list(range(1, 11))
    ramp = np.arange(100, dtype=np.int64)
    assert orc.scan(ramp).tolist() == [i * (i + 1) // 2 for i in range(100)]
    c = orc.conv1d(ramp, np.ones(5, np.int64), 0)
    assert all(c[i] == 5 * i for i in range(2, 98))
    assert np.array_equal(orc.conv1d(ramp, np.ones(1, np.int64), 0), ramp)


def test_oracle_golden(orc, golden):
    for tag, dt, n, m, ss, fs, bnd, lanes in C.conv1d_cases():
        sig = orc.random_grid(n, NP[dt], ss)
        f = orc.random_filter(m, 1, NP[dt], fs).reshape(-1)
        assert digest(orc.conv1d(sig, f, bnd)) == golden["conv1d"][tag]["oracle"], tag
    for tag, dt, n, seed, lanes in C.scan_cases():
        v = orc.random_grid(n, NP[dt], seed)
        assert digest(orc.scan(v)) == golden["scan"][tag]["oracle"], tag


def test_reference_simulator_exact_on_ints(golden):
    for sec in ("conv1d", "scan"):
        for tag, rec in golden[sec].items():
            if tag.startswith("i64"):
                assert rec["oracle"] == rec["ssam"], (sec, tag)


def test_golden_counters(lib, golden):
    for tag, dt, n, m, ss, fs, bnd, lanes in C.conv1d_cases():
        got = lib.counters_conv1d(n, m, lib.KernelConfig(lane_count=lanes))
        assert list(got.as_tuple()) == golden["conv1d"][tag]["counters"], tag
    for tag, dt, n, seed, lanes in C.scan_cases():
        got = lib.counters_scan(n, lanes)
        assert list(got.as_tuple()) == golden["scan"][tag]["counters"], tag


def test_counters_vs_reference(lib, ref):
    rng = np.random.default_rng(7)
    for _ in range(60):
        lanes = int(2 ** rng.integers(1, 7))
        m = int(rng.integers(1, lanes + 1))
        n = int(rng.integers(lanes, 400))
        sig = rng.integers(-5, 5, n).astype(np.int64)
        f = rng.integers(-3, 3, m).astype(np.int64)
        rc, _, cnt = ref.conv1d(sig, f, lane_count=lanes)
        assert rc == 0
        assert list(lib.counters_conv1d(n, m, lib.KernelConfig(lane_count=lanes)).as_tuple()) \
            == cnt.tolist(), (n, m, lanes)
        t = int(rng.integers(0, 9))
        rc, _, cnt = ref.scan(np.ones(t * lanes, np.int64), lane_count=lanes)
        assert rc == 0
        assert list(lib.counters_scan(t * lanes, lanes).as_tuple()) == cnt.tolist()


def test_error_contract_vs_reference(lib, ref):
    import ctypes
    mism = []
    for n, m, lanes in itertools.product((0, 1, 2, 5, 16, 31, 32, 33, 64, 100),
                                         (-1, 0, 1, 2, 16, 31, 32, 33, 64, 65),
                                         (-4, 0, 1, 2, 3, 16, 32, 48, 64, 128)):
        sig = np.ones(n, np.int64)
        f = np.ones(max(m, 0), np.int64)
        if m < 0:
            want = 1  # the reference sizes the filter from the vector: m >= 0 always
        else:
            want, _, _ = ref.conv1d(sig, f, lane_count=lanes)
        got = lib.lib.ssam_b200_check_conv1d(n, m, ctypes.byref(
            lib.KernelConfig(lane_count=lanes)._c()))
        if (want, got) not in ((0, 0), (1, 1)):
            mism.append(("conv1d", n, m, lanes, want, got))
    for n, lanes in itertools.product((0, 1, 2, 16, 32, 48, 64, 96, 128),
                                      (1, 2, 3, 16, 32, 48, 64, 128)):
        want, _, _ = ref.scan(np.ones(n, np.int64), lane_count=lanes)
        got = lib.lib.ssam_b200_check_scan(n, lanes)
        if (want, got) not in ((0, 0), (1, 1)):
            mism.append(("scan", n, lanes, want, got))
    assert not mism, mism[:10]


def test_error_paths_of_reference_tests(lib):
    """proj/tests/test_kernels_conv.cpp:159-162, :184-186."""
    with pytest.raises(lib.InvalidArgument):
        lib.check_conv1d(10, 5)           # signal shorter than a warp
    with pytest.raises(lib.InvalidArgument):
        lib.check_conv1d(100, 33)         # filter wider than the warp
    with pytest.raises(lib.InvalidArgument):
        lib.check_scan(33, 32)            # ragged
    lib.check_scan(0, 32)                 # empty is fine
