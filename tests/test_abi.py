"""C-ABI library: loads without a GPU, exports every declared symbol, and
never computes on the CPU (CPU-only tests)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "ssam_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(ssam_b200_\w+)\s*\(", text)))


def test_header_and_exports_agree(lib):
    declared = declared_symbols()
    assert declared, "no declarations parsed"
    raw = ctypes.CDLL(lib.LIB_PATH)
    for name in declared:
        assert hasattr(raw, name), f"{name} declared in include/ssam_b200.h but not exported"
    assert sorted(lib.EXPORTED) == declared


def test_abi_version(lib):
    assert lib.lib.ssam_b200_abi_version() == 2


def test_default_config_matches_reference(lib):
    c = lib._Cfg()
    lib.lib.ssam_b200_default_config(ctypes.byref(c))
    assert (c.p, c.b, c.boundary, c.lane_count, c.threads) == (4, 128, 0, 32, 0)


def test_library_is_cuda_code(lib):
    """The shared object carries sm_100a SASS for the SSAM kernels."""
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", lib.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES", None) == "" or False,
                    reason="explicitly hidden devices")
def test_no_cpu_fallback_without_device(lib):
    if lib.device_available():
        pytest.skip("a device is present; covered by the GPU tests")
    g = np.zeros((64, 64), np.float32)
    with pytest.raises(lib.NoDevice):
        lib.conv2d(g, np.ones((3, 3), np.float32))
    with pytest.raises(lib.NoDevice):
        lib.stencil2d(g, lib.convert_stencil(lib.make_benchmark_stencil("2d5pt"), np.float32),
                      lib.KernelConfig(), 1)


def test_catalog_matches_golden(lib, golden):
    assert lib.benchmark_stencil_names() == list(golden["catalog"].keys()) or \
        sorted(lib.benchmark_stencil_names()) == sorted(golden["catalog"].keys())
    for name, want in golden["catalog"].items():
        st = lib.make_benchmark_stencil(name)
        assert (st.dims, st.order, st.fpp) == (want["dims"], want["order"], want["fpp"])
        assert [list(t.offset) for t in st.taps] == want["offsets"]
        assert [float(t.coeff).hex() for t in st.taps] == want["coeffs"]
    with pytest.raises(lib.InvalidArgument):
        lib.make_benchmark_stencil("2d7pt")


def test_peer_entry_points_refuse_without_device(lib):
    """The peer-halo and IPC entry points validate their arguments and fail with
    a status (never a CPU path) when no GPU is present."""
    if lib.device_available():
        pytest.skip("a device is present; covered by the GPU tests")
    ptr, h = ctypes.c_void_p(), ctypes.create_string_buffer(lib.IPC_HANDLE_BYTES)
    assert lib.lib.ssam_b200_ipc_alloc(0, ctypes.byref(ptr), h) == lib.SSAM_ERR_INVALID_ARGUMENT
    assert lib.lib.ssam_b200_ipc_alloc(1 << 20, ctypes.byref(ptr), h) != 0
    assert lib.lib.ssam_b200_ipc_open(None, ctypes.byref(ptr)) == lib.SSAM_ERR_INVALID_ARGUMENT
    st = lib.convert_stencil(lib.make_benchmark_stencil("3d7pt"), np.float32)
    sa = lib._StencilArgs(st, np.float32)
    halo = lib._PeerHalo()
    rc = lib.lib.ssam_b200_stencil3d_sweep_peer(7, None, None, 8, 8, 8, 0, 8, sa.ref,
                                                ctypes.byref(halo), None)
    assert rc == lib.SSAM_ERR_INVALID_ARGUMENT  # unknown dtype, checked first
    rc = lib.lib.ssam_b200_stencil3d_sweep_peer(0, None, None, 8, 8, 8, 0, 8, sa.ref,
                                                ctypes.byref(halo), None)
    assert rc != 0 and lib.lib.ssam_b200_last_error()


def test_multi_entry_points_validate_before_the_device(lib):
    """ssam_b200_stencil2d_multi / _3d_multi: the single-device checks come
    first (same statuses), then the device list; no CPU path."""
    if lib.device_available():
        pytest.skip("a device is present; covered by tests/test_gpu_multi.py")
    st = lib.convert_stencil(lib.make_benchmark_stencil("3d7pt"), np.float32)
    g = np.zeros((16, 16, 16), np.float32)
    with pytest.raises(lib.InvalidArgument):
        lib.stencil_multi(g, st, [0, 1], iters=0)  # iters < 1, as ssam::stencil3d
    st2 = lib.convert_stencil(lib.make_benchmark_stencil("2d5pt"), np.float32)
    with pytest.raises(lib.InvalidArgument):
        lib.stencil_multi(np.zeros((2, 64), np.float32), st2, [0])  # domain < 2k+1
    with pytest.raises(lib.NoDevice):
        lib.stencil_multi(g, st, [0, 1])
    sa = lib._StencilArgs(st, np.float32)
    rc = lib.lib.ssam_b200_stencil3d_multi(9, None, 8, 8, 8, sa.ref, None, 1, None, 0, None,
                                           None, None)
    assert rc == lib.SSAM_ERR_INVALID_ARGUMENT
