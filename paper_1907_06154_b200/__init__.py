"""paper_1907_06154_b200 -- B200-native SSAM engine (arXiv 1907.06154).

Python host mirror of the reference's kernel API (proj/include/ssam/kernels.hpp
:189 conv2d, :231 stencil2d, :283 stencil3d) over the C ABI in
include/ssam_b200.h.  Same names, same argument meaning, same error
behaviour: the reference's ``std::invalid_argument`` is :class:`InvalidArgument`
and ``std::length_error`` is :class:`LengthError` (both ``ValueError``).

All compute runs in libssam_b200.so on the GPU.  There is no CPU fallback:
importing fails loudly when the library is missing, and compute calls raise
:class:`NoDevice` without a CUDA device.

Grids are numpy arrays in the reference's layout: 2D ``(H, W)`` row-major
(``data[y*W + x]``, grid.hpp:11-28), 3D ``(nz, ny, nx)`` (grid.hpp:30-49);
dtypes float32, float64, int64 (T in {float, double, long long}).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from enum import IntEnum
from typing import List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "Boundary", "KernelConfig", "OpCounters", "Filter2D", "StencilTap", "Stencil",
    "InvalidArgument", "LengthError", "CudaError", "NoDevice",
    "conv2d", "stencil2d", "stencil3d", "make_benchmark_stencil", "benchmark_stencil_names",
    "is_3d_benchmark", "convert_stencil", "stencil_order_of", "random_grid2d", "random_grid3d",
    "device_available", "launch_count",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SSAM_B200_LIB") or os.path.join(_HERE, "libssam_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: the SSAM engine has no CPU fallback. Build it with "
        "`make -j` in the repo root (or __graft_entry__.build()).")

_lib = C.CDLL(LIB_PATH)

SSAM_OK, SSAM_ERR_INVALID_ARGUMENT, SSAM_ERR_LENGTH, SSAM_ERR_CUDA, SSAM_ERR_NO_DEVICE, \
    SSAM_ERR_OUT_OF_MEMORY, SSAM_ERR_RUNTIME = range(7)

_DT = {np.dtype(np.float32): 0, np.dtype(np.float64): 1, np.dtype(np.int64): 2}
_NP = {0: np.float32, 1: np.float64, 2: np.int64}


class InvalidArgument(ValueError):
    """The reference throws std::invalid_argument."""


class LengthError(ValueError):
    """The reference throws std::length_error (register cache C > 255)."""


class CudaError(RuntimeError):
    """CUDA runtime failure inside the engine."""


class NoDevice(RuntimeError):
    """No CUDA device: the engine never computes on the CPU."""


class OutOfMemory(CudaError):
    pass


class GridIOError(RuntimeError):
    """The reference throws std::runtime_error (grid_io.hpp readers / writers)."""


class _Cfg(C.Structure):
    _fields_ = [("p", C.c_int), ("b", C.c_int), ("boundary", C.c_int), ("lane_count", C.c_int),
                ("threads", C.c_int)]


class _Counters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in
                ("mads", "shuffles", "broadcast_reads", "global_loads", "global_stores")]


class _Stencil(C.Structure):
    _fields_ = [("dims", C.c_int), ("order", C.c_int), ("ntaps", C.c_int),
                ("offsets", C.c_void_p), ("coeffs", C.c_void_p)]


_p, _i, _u64, _sz = C.c_void_p, C.c_int, C.c_uint64, C.c_size_t
_PC, _PK, _PS = C.POINTER(_Cfg), C.POINTER(_Counters), C.POINTER(_Stencil)


def _sig(name, args, res=C.c_int):
    f = getattr(_lib, name)
    f.argtypes = args
    f.restype = res
    return f


_lib_last_error = _sig("ssam_b200_last_error", [], C.c_char_p)
_sig("ssam_b200_abi_version", [])
_sig("ssam_b200_device_count", [])
_sig("ssam_b200_default_config", [_PC], None)
_sig("ssam_b200_launch_count", [], C.c_uint64)
_sig("ssam_b200_conv2d", [_i, _p, _i, _i, _p, _i, _i, _PC, _p, _PK])
_sig("ssam_b200_stencil2d", [_i, _p, _i, _i, _PS, _PC, _i, _p, _PK])
_sig("ssam_b200_stencil3d", [_i, _p, _i, _i, _i, _PS, _PC, _i, _p, _PK])
_sig("ssam_b200_stencil2d_multi", [_i, _p, _i, _i, _PS, _PC, _i, C.POINTER(_i), _i, _p, _PK,
                                   C.POINTER(_i)])
_sig("ssam_b200_stencil3d_multi", [_i, _p, _i, _i, _i, _PS, _PC, _i, C.POINTER(_i), _i, _p, _PK,
                                   C.POINTER(_i)])
_sig("ssam_b200_check_conv2d", [_i, _i, _i, _i, _PC])
_sig("ssam_b200_check_stencil2d", [_i, _i, _PS, _PC, _i])
_sig("ssam_b200_check_stencil3d", [_i, _i, _i, _PS, _PC, _i])
_sig("ssam_b200_counters_conv2d", [_i, _i, _i, _i, _PC, _PK])
_sig("ssam_b200_counters_stencil2d", [_i, _i, _PS, _PC, _i, _PK])
_sig("ssam_b200_counters_stencil3d", [_i, _i, _i, _PS, _PC, _i, _PK])
_sig("ssam_b200_benchmark_count", [])
_sig("ssam_b200_benchmark_name", [_i], C.c_char_p)
_sig("ssam_b200_benchmark_stencil", [C.c_char_p, C.POINTER(_i), C.POINTER(_i), C.POINTER(_i),
                                     _p, _p, _i])
_sig("ssam_b200_conv2d_device", [_i, _p, _p, _i, _i, _i, _i, _p, _i, _i, _i, _p])
_sig("ssam_b200_stencil2d_sweep", [_i, _p, _p, _i, _i, _i, _i, _PS, _p])
_sig("ssam_b200_stencil2d_tb", [_i, _p, _p, _i, _i, _PS, _i, _p])
_sig("ssam_b200_stencil2d_tb_max", [_i, _PS])
_sig("ssam_b200_stencil2d_tb_range", [_i, _p, _p, _i, _i, _i, _i, _i, _i, _PS, _i, _p])
_sig("ssam_b200_stencil3d_sweep", [_i, _p, _p, _i, _i, _i, _i, _i, _PS, _p])
_sig("ssam_b200_stencil3d_tb", [_i, _p, _p, _i, _i, _i, _i, _i, _i, _i, _PS, _i, _p])
_sig("ssam_b200_stencil3d_tb_max", [_i, _PS])
_sig("ssam_b200_stencil2d_run", [_i, _p, _p, _i, _i, _PS, _i, _i, _p, C.POINTER(_p)])
_sig("ssam_b200_stencil3d_run", [_i, _p, _p, _i, _i, _i, _PS, _i, _p, C.POINTER(_p)])
_sig("ssam_b200_fill_random", [_i, _p, _sz, _u64, _u64, _p])
_sig("ssam_b200_max_rel_err", [_i, _p, _p, _sz, C.POINTER(C.c_double), C.POINTER(C.c_double),
                               _p])
_ll, _ull = C.c_longlong, C.c_ulonglong
_sig("ssam_b200_conv1d", [_i, _p, _ll, _p, _i, _PC, _p, _PK])
_sig("ssam_b200_scan", [_i, _p, _ull, _i, _p, _PK])
_sig("ssam_b200_check_conv1d", [_ll, _i, _PC])
_sig("ssam_b200_check_scan", [_ull, _i])
_sig("ssam_b200_counters_conv1d", [_ll, _i, _PC, _PK])
_sig("ssam_b200_counters_scan", [_ull, _i, _PK])
_sig("ssam_b200_conv1d_device", [_i, _p, _p, _i, _p, _i, _i, _p])
_sig("ssam_b200_scan_device", [_i, _p, _p, _sz, _p])
_sig("ssam_b200_sgrd_info", [C.c_char_p, C.POINTER(_i), C.POINTER(_i), _p])
_sig("ssam_b200_sgrd_read", [C.c_char_p, _i, _i, _p, _p, _sz, _i, _p])
_sig("ssam_b200_sgrd_write", [C.c_char_p, _i, _i, _p, _p, _i, _p])
_sig("ssam_b200_gather_conv2d", [_i, _p, _i, _i, _p, _i, _i, _i, _p])
_sig("ssam_b200_gather_stencil", [_i, _p, _i, _i, _i, _PS, _i, _p])
_sig("ssam_b200_gather_stencil_run", [_i, _p, _p, _i, _i, _i, _PS, _i, _p, C.POINTER(_p)])
_sig("ssam_b200_trim_cache", [])
_sig("ssam_b200_stencil_batch", [_i, _i, C.POINTER(_p), C.POINTER(_p), _i, _i, _i, _PS, _i, _i])


class _PeerHalo(C.Structure):
    _fields_ = [("lo", C.c_void_p), ("lo_shift", C.c_longlong), ("lo_end", C.c_int),
                ("hi", C.c_void_p), ("hi_shift", C.c_longlong), ("hi_begin", C.c_int)]


_PP = C.POINTER(_PeerHalo)
_sig("ssam_b200_stencil3d_sweep_peer", [_i, _p, _p, _i, _i, _i, _i, _i, _PS, _PP, _p])
_sig("ssam_b200_stencil3d_tb_peer", [_i, _p, _p, _i, _i, _i, _i, _i, _i, _i, _PS, _i, _PP, _p])
_sig("ssam_b200_ipc_alloc", [_sz, C.POINTER(_p), _p])
_sig("ssam_b200_ipc_free", [_p])
_sig("ssam_b200_ipc_open", [_p, C.POINTER(_p)])
_sig("ssam_b200_ipc_close", [_p])
_sig("ssam_b200_stream_write_u32", [_p, C.c_uint32, _p])
_sig("ssam_b200_stream_wait_u32", [_p, C.c_uint32, _p])
IPC_HANDLE_BYTES = 64

lib = _lib  # raw handle for device-level callers (bench.py, tests)

# Every symbol include/ssam_b200.h declares (checked by tests/test_abi.py).
EXPORTED = [
    "ssam_b200_abi_version", "ssam_b200_last_error", "ssam_b200_device_count",
    "ssam_b200_default_config", "ssam_b200_launch_count", "ssam_b200_conv2d",
    "ssam_b200_stencil2d_multi", "ssam_b200_stencil3d_multi", "ssam_b200_measure_latency",
    "ssam_b200_stencil2d", "ssam_b200_stencil3d", "ssam_b200_check_conv2d",
    "ssam_b200_check_stencil2d", "ssam_b200_check_stencil3d", "ssam_b200_counters_conv2d",
    "ssam_b200_counters_stencil2d", "ssam_b200_counters_stencil3d", "ssam_b200_benchmark_count",
    "ssam_b200_benchmark_name", "ssam_b200_benchmark_stencil", "ssam_b200_conv2d_device",
    "ssam_b200_stencil2d_sweep", "ssam_b200_stencil2d_tb", "ssam_b200_stencil2d_tb_max",
    "ssam_b200_stencil3d_sweep", "ssam_b200_stencil2d_run", "ssam_b200_stencil3d_run",
    "ssam_b200_fill_random", "ssam_b200_max_rel_err", "ssam_b200_conv1d", "ssam_b200_scan",
    "ssam_b200_check_conv1d", "ssam_b200_check_scan", "ssam_b200_counters_conv1d",
    "ssam_b200_counters_scan", "ssam_b200_conv1d_device", "ssam_b200_scan_device",
    "ssam_b200_sgrd_info", "ssam_b200_sgrd_read", "ssam_b200_sgrd_write",
    "ssam_b200_gather_conv2d", "ssam_b200_gather_stencil", "ssam_b200_stencil3d_tb",
    "ssam_b200_stencil3d_tb_max", "ssam_b200_stencil3d_sweep_peer", "ssam_b200_stencil3d_tb_peer",
    "ssam_b200_ipc_alloc", "ssam_b200_ipc_free", "ssam_b200_ipc_open", "ssam_b200_ipc_close",
    "ssam_b200_stream_write_u32", "ssam_b200_stream_wait_u32",
    "ssam_b200_stencil2d_tb_range", "ssam_b200_gather_stencil_run", "ssam_b200_trim_cache",
    "ssam_b200_stencil_batch",
]


def _raise(status: int) -> None:
    if status == SSAM_OK:
        return
    msg = (_lib_last_error() or b"").decode()
    if status == SSAM_ERR_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if status == SSAM_ERR_LENGTH:
        raise LengthError(msg)
    if status == SSAM_ERR_NO_DEVICE:
        raise NoDevice(msg)
    if status == SSAM_ERR_OUT_OF_MEMORY:
        raise OutOfMemory(msg)
    if status == SSAM_ERR_RUNTIME:
        raise GridIOError(msg)
    raise CudaError(f"status {status}: {msg}")


# ---------------------------------------------------------------------------
# Reference types (filter.hpp, warp.hpp)
# ---------------------------------------------------------------------------

class Boundary(IntEnum):
    """ssam::Boundary (filter.hpp:15)."""
    zero = 0
    replicate = 1


@dataclass
class KernelConfig:
    """ssam::KernelConfig (filter.hpp:117-139).  Validated like the reference;
    afterwards p, b, lane_count and threads are tuning hints the GPU may ignore."""
    p: int = 4
    b: int = 128
    boundary: Boundary = Boundary.zero
    lane_count: int = 32
    threads: int = 0

    kCacheCap = 255

    def warp_count(self) -> int:
        return self.b // self.lane_count

    def _c(self) -> _Cfg:
        return _Cfg(self.p, self.b, int(self.boundary), self.lane_count, self.threads)


@dataclass
class OpCounters:
    """ssam::OpCounters (warp.hpp:12-28); calls accumulate into it (+=)."""
    mads: int = 0
    shuffles: int = 0
    broadcast_reads: int = 0
    global_loads: int = 0
    global_stores: int = 0

    def _load(self) -> _Counters:
        return _Counters(self.mads, self.shuffles, self.broadcast_reads, self.global_loads,
                         self.global_stores)

    def _store(self, c: _Counters) -> None:
        self.mads, self.shuffles, self.broadcast_reads = c.mads, c.shuffles, c.broadcast_reads
        self.global_loads, self.global_stores = c.global_loads, c.global_stores

    def __iadd__(self, o: "OpCounters") -> "OpCounters":
        self.mads += o.mads
        self.shuffles += o.shuffles
        self.broadcast_reads += o.broadcast_reads
        self.global_loads += o.global_loads
        self.global_stores += o.global_stores
        return self

    def as_tuple(self):
        return (self.mads, self.shuffles, self.broadcast_reads, self.global_loads,
                self.global_stores)


class Filter2D:
    """ssam::Filter2D (filter.hpp:18-39): m taps across x, n along y,
    weights w[s*n + t] -- here an (m, n) array, w[s, t]."""

    def __init__(self, m: int = 1, n: int = 1, weights=None, dtype=np.float64):
        if m < 1 or n < 1:
            raise InvalidArgument("filter: taps must be >= 1")
        if weights is None:
            if (m, n) != (1, 1):
                raise InvalidArgument("filter: weight count does not match m x n")
            weights = [1]
        w = np.asarray(weights)
        if w.size != m * n:
            raise InvalidArgument("filter: weight count does not match m x n")
        self.m, self.n = m, n
        self.w = w.reshape(m, n).astype(w.dtype if w.dtype in _DT else dtype)

    def at(self, s: int, t: int):
        return self.w[s, t]

    def anchor_x(self) -> int:
        return (self.m - 1) // 2

    def anchor_y(self) -> int:
        return (self.n - 1) // 2


@dataclass
class StencilTap:
    offset: Tuple[int, int, int]
    coeff: float


@dataclass
class Stencil:
    """ssam::Stencil (filter.hpp:52-68)."""
    name: str = ""
    dims: int = 2
    order: int = 0
    fpp: int = 0
    taps: List[StencilTap] = field(default_factory=list)

    def offsets(self) -> np.ndarray:
        return np.asarray([t.offset for t in self.taps], dtype=np.int32).reshape(-1, 3)


def stencil_order_of(taps: Sequence[StencilTap]) -> int:
    return max((abs(c) for t in taps for c in t.offset), default=0)


class _StencilArgs:
    """Keeps the numpy buffers alive while the C struct points at them."""

    def __init__(self, st: Stencil, dtype):
        self.off = np.ascontiguousarray(st.offsets(), dtype=np.int32)
        if st.taps:
            vals = [t.coeff for t in st.taps]
            self.cf = np.ascontiguousarray(np.asarray(vals).astype(dtype))
        else:
            self.cf = np.zeros(1, dtype=dtype)
        self.s = _Stencil(st.dims, st.order, len(st.taps),
                          self.off.ctypes.data if len(st.taps) else None, self.cf.ctypes.data)

    @property
    def ref(self):
        return C.byref(self.s)


def convert_stencil(st: Stencil, dtype) -> Stencil:
    """convert_stencil<T> (filter.hpp:104-115): cast every coefficient to T."""
    t = np.dtype(dtype).type
    return Stencil(st.name, st.dims, st.order, st.fpp,
                   [StencilTap(tuple(x.offset), t(x.coeff)) for x in st.taps])


def make_benchmark_stencil(name: str) -> Stencil:
    """make_benchmark_stencil (stencil_catalog.cpp:81-112), double coefficients."""
    off = np.zeros((125, 3), dtype=np.int32)
    cf = np.zeros(125, dtype=np.float64)
    dims, order, fpp = _i(), _i(), _i()
    n = _lib.ssam_b200_benchmark_stencil(name.encode(), C.byref(dims), C.byref(order),
                                         C.byref(fpp), off.ctypes.data, cf.ctypes.data, 125)
    if n < 0:
        raise InvalidArgument(f"unknown stencil benchmark: {name}")
    taps = [StencilTap(tuple(int(v) for v in off[i]), float(cf[i])) for i in range(n)]
    return Stencil(name, dims.value, order.value, fpp.value, taps)


def benchmark_stencil_names() -> List[str]:
    return [_lib.ssam_b200_benchmark_name(i).decode()
            for i in range(_lib.ssam_b200_benchmark_count())]


def is_3d_benchmark(name: str) -> bool:
    return make_benchmark_stencil(name).dims == 3


# ---------------------------------------------------------------------------
# Kernel API (kernels.hpp:189 / :231 / :283)
# ---------------------------------------------------------------------------

def device_available() -> bool:
    return _lib.ssam_b200_device_count() > 0


def launch_count() -> int:
    return int(_lib.ssam_b200_launch_count())


def _grid(a: np.ndarray, ndim: int) -> np.ndarray:
    a = np.asarray(a)
    if a.ndim != ndim:
        raise InvalidArgument(f"expected a {ndim}D grid, got shape {a.shape}")
    if a.dtype not in _DT:
        raise InvalidArgument(f"unsupported dtype {a.dtype}; use float32, float64 or int64")
    return np.ascontiguousarray(a)


def _weights(filt, dtype) -> np.ndarray:
    w = filt.w if isinstance(filt, Filter2D) else np.asarray(filt)
    if w.ndim != 2:
        raise InvalidArgument("filter weights must be an (m, n) array")
    return np.ascontiguousarray(w.astype(dtype, copy=False))


def conv2d(grid: np.ndarray, filt, cfg: Optional[KernelConfig] = None,
           counters: Optional[OpCounters] = None) -> np.ndarray:
    """ssam::conv2d (kernels.hpp:189-225): true 2D convolution
    out(x,y) = sum_{s,t} in(x+ax-s, y+ay-t) w[s,t] with cfg.boundary."""
    g = _grid(grid, 2)
    w = _weights(filt, g.dtype)
    cfg = cfg or KernelConfig()
    out = np.empty_like(g)
    cnt = counters._load() if counters is not None else None
    st = _lib.ssam_b200_conv2d(_DT[g.dtype], g.ctypes.data, g.shape[1], g.shape[0],
                               w.ctypes.data, w.shape[0], w.shape[1], C.byref(cfg._c()),
                               out.ctypes.data, C.byref(cnt) if cnt is not None else None)
    _raise(st)
    if counters is not None:
        counters._store(cnt)
    return out


def stencil2d(grid: np.ndarray, st: Stencil, cfg: Optional[KernelConfig] = None, iters: int = 1,
              counters: Optional[OpCounters] = None) -> np.ndarray:
    """ssam::stencil2d (kernels.hpp:231-277): iters Jacobi sweeps; the ring of
    width st.order carries over unchanged."""
    g = _grid(grid, 2)
    cfg = cfg or KernelConfig()
    sa = _StencilArgs(st, g.dtype)
    out = np.empty_like(g)
    cnt = counters._load() if counters is not None else None
    s = _lib.ssam_b200_stencil2d(_DT[g.dtype], g.ctypes.data, g.shape[1], g.shape[0], sa.ref,
                                 C.byref(cfg._c()), iters, out.ctypes.data,
                                 C.byref(cnt) if cnt is not None else None)
    _raise(s)
    if counters is not None:
        counters._store(cnt)
    return out


def stencil3d(grid: np.ndarray, st: Stencil, cfg: Optional[KernelConfig] = None, iters: int = 1,
              counters: Optional[OpCounters] = None) -> np.ndarray:
    """ssam::stencil3d (kernels.hpp:283-384): iters 3D Jacobi sweeps."""
    g = _grid(grid, 3)
    cfg = cfg or KernelConfig(p=2, b=max(128, 32 * (2 * st.order + 1)))
    sa = _StencilArgs(st, g.dtype)
    out = np.empty_like(g)
    cnt = counters._load() if counters is not None else None
    nz, ny, nx = g.shape
    s = _lib.ssam_b200_stencil3d(_DT[g.dtype], g.ctypes.data, nx, ny, nz, sa.ref,
                                 C.byref(cfg._c()), iters, out.ctypes.data,
                                 C.byref(cnt) if cnt is not None else None)
    _raise(s)
    if counters is not None:
        counters._store(cnt)
    return out


class _Latency(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("t_shfl", "t_mad", "t_smem_read", "t_reg",
                                          "t_gmem_read", "t_gmem_write", "t_l2_read",
                                          "sm_clock_mhz")]


_sig("ssam_b200_measure_latency", [C.POINTER(_Latency)])

PROFILE_FIELDS = ("t_shfl", "t_mad", "t_smem_read", "t_reg", "t_gmem_read", "t_gmem_write")


def measure_latency_profile() -> dict:
    """ssam::LatencyProfile fields (perf_model.hpp:14-26) measured on the
    current device by csrc/latency.cu, in SM cycles (floats), plus t_l2_read
    and sm_clock_mhz."""
    r = _Latency()
    _raise(_lib.ssam_b200_measure_latency(C.byref(r)))
    return {n: getattr(r, n) for n, _ in _Latency._fields_}


def format_profile(name: str, prof: dict) -> str:
    """A profile file the reference's load_profile_file reads
    (perf_model.cpp:41-78): `name`, then one `field value` line per latency,
    values as integers (whole cycles) or `num/den` rationals."""
    lines = [f"name {name}"]
    for f in PROFILE_FIELDS:
        lines.append(f"{f} {max(1, int(round(prof[f])))}")
    return "\n".join(lines) + "\n"


def stencil_multi(grid: np.ndarray, st: Stencil, devices: Sequence[int],
                  cfg: Optional[KernelConfig] = None, iters: int = 1,
                  counters: Optional[OpCounters] = None):
    """ssam::stencil2d / stencil3d on several GPUs from this process
    (ssam_b200_stencil2d_multi / _3d_multi): slabs along the slowest axis,
    slab g on devices[g] (repeats allowed), halos by peer copies.  Returns
    (result, slabs actually used); the result equals stencil2d/3d bit for bit."""
    g = _grid(grid, st.dims)
    if cfg is None:
        cfg = KernelConfig() if st.dims == 2 else KernelConfig(p=2, b=max(128, 32 * (2 * st.order + 1)))
    sa = _StencilArgs(st, g.dtype)
    out = np.empty_like(g)
    devs = (_i * len(devices))(*devices)
    used = _i(0)
    cnt = counters._load() if counters is not None else None
    pk = C.byref(cnt) if cnt is not None else None
    if st.dims == 2:
        s = _lib.ssam_b200_stencil2d_multi(_DT[g.dtype], g.ctypes.data, g.shape[1], g.shape[0],
                                           sa.ref, C.byref(cfg._c()), iters, devs, len(devices),
                                           out.ctypes.data, pk, C.byref(used))
    else:
        nz, ny, nx = g.shape
        s = _lib.ssam_b200_stencil3d_multi(_DT[g.dtype], g.ctypes.data, nx, ny, nz, sa.ref,
                                           C.byref(cfg._c()), iters, devs, len(devices),
                                           out.ctypes.data, pk, C.byref(used))
    _raise(s)
    if counters is not None:
        counters._store(cnt)
    return out, used.value


def stencil_batch(grids, outs, st: Stencil, iters: int, depth: int = 0) -> None:
    """ssam_b200_stencil_batch: `iters` sweeps of each grid in `grids` into the
    matching `outs` entry, with host<->device copies overlapped across grids.
    Grids are numpy arrays or host tensors (pinned for the overlap) of one
    shape and dtype; 2D grids are (H, W), 3D (nz, ny, nx)."""
    if len(grids) != len(outs):
        raise InvalidArgument("stencil_batch: grids and outs differ in length")
    if not grids:
        return

    def info(a):
        if isinstance(a, np.ndarray):
            if not a.flags.c_contiguous:
                raise InvalidArgument("stencil_batch: grids must be C-contiguous")
            return a.ctypes.data, a.shape, np.dtype(a.dtype)
        return a.data_ptr(), tuple(a.shape), np.dtype(str(a.dtype).replace("torch.", ""))

    ins = [info(a) for a in grids]
    ots = [info(a) for a in outs]
    shape, dt = ins[0][1], ins[0][2]
    if any(i[1] != shape or i[2] != dt for i in ins + ots):
        raise InvalidArgument("stencil_batch: every grid needs the same shape and dtype")
    if dt not in _DT:
        raise InvalidArgument(f"unsupported dtype {dt}")
    if len(shape) == 2:
        (ny, nx), nz = shape, 1
    else:
        nz, ny, nx = shape
    sa = _StencilArgs(st, dt)
    n = len(grids)
    pin = (C.c_void_p * n)(*[i[0] for i in ins])
    pout = (C.c_void_p * n)(*[o[0] for o in ots])
    _raise(_lib.ssam_b200_stencil_batch(_DT[dt], n, C.cast(pin, C.POINTER(C.c_void_p)),
                                        C.cast(pout, C.POINTER(C.c_void_p)), nx, ny, nz, sa.ref,
                                        iters, depth))


def _vector(a) -> np.ndarray:
    a = np.asarray(a)
    if a.ndim != 1:
        raise InvalidArgument(f"expected a 1D signal, got shape {a.shape}")
    if a.dtype not in _DT:
        raise InvalidArgument(f"unsupported dtype {a.dtype}; use float32, float64 or int64")
    return np.ascontiguousarray(a)


def conv1d(signal, filt, cfg: Optional[KernelConfig] = None,
           counters: Optional[OpCounters] = None) -> np.ndarray:
    """ssam::conv1d (kernels.hpp:390-418): out(i) = sum_s in(i + (m-1)/2 - s) f[s]
    with cfg.boundary; m in [1, lane_count], len >= lane_count."""
    g = _vector(signal)
    f = np.ascontiguousarray(np.asarray(filt).astype(g.dtype, copy=False).reshape(-1))
    cfg = cfg or KernelConfig()
    out = np.empty_like(g)
    cnt = counters._load() if counters is not None else None
    st = _lib.ssam_b200_conv1d(_DT[g.dtype], g.ctypes.data, g.size, f.ctypes.data, f.size,
                               C.byref(cfg._c()), out.ctypes.data,
                               C.byref(cnt) if cnt is not None else None)
    _raise(st)
    if counters is not None:
        counters._store(cnt)
    return out


def scan(values, lane_count: int = 32, counters: Optional[OpCounters] = None) -> np.ndarray:
    """ssam::scan (kernels.hpp:422-447): inclusive prefix sum; the length must be a
    multiple of lane_count."""
    g = _vector(values)
    out = np.empty_like(g)
    cnt = counters._load() if counters is not None else None
    st = _lib.ssam_b200_scan(_DT[g.dtype], g.ctypes.data, g.size, lane_count, out.ctypes.data,
                             C.byref(cnt) if cnt is not None else None)
    _raise(st)
    if counters is not None:
        counters._store(cnt)
    return out


# -- SGRD grid files (grid_io.hpp:14-158) ---------------------------------------

def sgrd_info(path: str):
    """(rank, dtype, dims (d0, d1, d2) x-fastest) of an SGRD file."""
    rank, dt = C.c_int(), C.c_int()
    dims = np.zeros(3, dtype=np.int32)
    _raise(_lib.ssam_b200_sgrd_info(os.fsencode(path), C.byref(rank), C.byref(dt),
                                    dims.ctypes.data))
    return rank.value, _NP.get(dt.value), tuple(int(d) for d in dims)


def _read_sgrd(path: str, dtype, rank: int) -> np.ndarray:
    _, _, dims = sgrd_info(path)
    shape = tuple(dims[:rank][::-1])
    out = np.empty(shape, dtype=dtype)
    d = np.zeros(3, dtype=np.int32)
    _raise(_lib.ssam_b200_sgrd_read(os.fsencode(path), _DT[np.dtype(dtype)], rank, d.ctypes.data,
                                    out.ctypes.data, out.size, 0, None))
    return out


def read_grid2d(path: str, dtype=np.float64) -> np.ndarray:
    """ssam::read_grid2d<T> (grid_io.hpp:105-111) from a file: an (h, w) array."""
    return _read_sgrd(path, dtype, 2)


def read_grid3d(path: str, dtype=np.float64) -> np.ndarray:
    """ssam::read_grid3d<T> (grid_io.hpp:113-119): an (nz, ny, nx) array."""
    return _read_sgrd(path, dtype, 3)


def read_vector(path: str, dtype=np.float64) -> np.ndarray:
    """ssam::read_vector<T> (grid_io.hpp:121-127)."""
    return _read_sgrd(path, dtype, 1)


def write_grid(path: str, grid: np.ndarray) -> None:
    """ssam::write_grid_file (grid_io.hpp:129-134): rank = grid.ndim (x fastest)."""
    g = np.asarray(grid)
    if g.ndim not in (1, 2, 3) or g.dtype not in _DT:
        raise InvalidArgument("grid io: need a 1-3D float32/float64/int64 array")
    g = np.ascontiguousarray(g)
    dims = np.array(list(g.shape[::-1]) + [1] * (3 - g.ndim), dtype=np.int32)
    _raise(_lib.ssam_b200_sgrd_write(os.fsencode(path), _DT[g.dtype], g.ndim, dims.ctypes.data,
                                     g.ctypes.data, 0, None))


# -- validation / counters without a device ----------------------------------

def check_conv1d(length: int, m: int, cfg: Optional[KernelConfig] = None) -> None:
    _raise(_lib.ssam_b200_check_conv1d(length, m, C.byref((cfg or KernelConfig())._c())))


def check_scan(length: int, lane_count: int = 32) -> None:
    _raise(_lib.ssam_b200_check_scan(length, lane_count))


def counters_conv1d(length: int, m: int, cfg=None) -> OpCounters:
    c = _Counters()
    _raise(_lib.ssam_b200_counters_conv1d(length, m, C.byref((cfg or KernelConfig())._c()),
                                          C.byref(c)))
    o = OpCounters()
    o._store(c)
    return o


def counters_scan(length: int, lane_count: int = 32) -> OpCounters:
    c = _Counters()
    _raise(_lib.ssam_b200_counters_scan(length, lane_count, C.byref(c)))
    o = OpCounters()
    o._store(c)
    return o


def check_conv2d(w: int, h: int, m: int, n: int, cfg: Optional[KernelConfig] = None) -> None:
    _raise(_lib.ssam_b200_check_conv2d(w, h, m, n, C.byref((cfg or KernelConfig())._c())))


def check_stencil2d(w, h, st: Stencil, cfg=None, iters=1, dtype=np.float64) -> None:
    sa = _StencilArgs(st, dtype)
    _raise(_lib.ssam_b200_check_stencil2d(w, h, sa.ref, C.byref((cfg or KernelConfig())._c()),
                                          iters))


def check_stencil3d(nx, ny, nz, st: Stencil, cfg=None, iters=1, dtype=np.float64) -> None:
    sa = _StencilArgs(st, dtype)
    _raise(_lib.ssam_b200_check_stencil3d(nx, ny, nz, sa.ref,
                                          C.byref((cfg or KernelConfig())._c()), iters))


def counters_conv2d(w, h, m, n, cfg=None) -> OpCounters:
    c = _Counters()
    _raise(_lib.ssam_b200_counters_conv2d(w, h, m, n, C.byref((cfg or KernelConfig())._c()),
                                          C.byref(c)))
    o = OpCounters()
    o._store(c)
    return o


def counters_stencil2d(w, h, st: Stencil, cfg=None, iters=1) -> OpCounters:
    sa = _StencilArgs(st, np.float64)
    c = _Counters()
    _raise(_lib.ssam_b200_counters_stencil2d(w, h, sa.ref, C.byref((cfg or KernelConfig())._c()),
                                             iters, C.byref(c)))
    o = OpCounters()
    o._store(c)
    return o


def counters_stencil3d(nx, ny, nz, st: Stencil, cfg=None, iters=1) -> OpCounters:
    sa = _StencilArgs(st, np.float64)
    c = _Counters()
    _raise(_lib.ssam_b200_counters_stencil3d(nx, ny, nz, sa.ref,
                                             C.byref((cfg or KernelConfig())._c()), iters,
                                             C.byref(c)))
    o = OpCounters()
    o._store(c)
    return o


# -- synthetic inputs (generated on the device, grid.hpp:52-66 bit-for-bit) -----

def _device_fill_to_host(shape, dtype, seed: int) -> np.ndarray:
    import torch  # plumbing only: device memory
    if not torch.cuda.is_available():
        raise NoDevice("random grids are generated on the GPU")
    n = int(np.prod(shape))
    t = torch.empty(n, dtype={0: torch.float32, 1: torch.float64, 2: torch.int64}[_DT[np.dtype(dtype)]],
                    device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    _raise(_lib.ssam_b200_fill_random(_DT[np.dtype(dtype)], t.data_ptr(), n, seed, 0, s))
    return t.cpu().numpy().reshape(shape)


def random_grid2d(w: int, h: int, seed: int, dtype=np.float64) -> np.ndarray:
    return _device_fill_to_host((h, w), dtype, seed)


def random_grid3d(nx: int, ny: int, nz: int, seed: int, dtype=np.float64) -> np.ndarray:
    return _device_fill_to_host((nz, ny, nx), dtype, seed)


from . import device  # noqa: E402,F401  (device-resident API used by bench.py)
