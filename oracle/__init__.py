"""TEST INFRASTRUCTURE ONLY -- ctypes bindings for the CPU checkers.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the CPU baseline.  The product (``paper_1907_06154_b200``) never imports it.

* ``Oracle``    -- oracle/liboracle.so, our plain-C restatement of the
                   reference's oracle.hpp / rng.hpp / stencil_catalog.cpp.
* ``Reference`` -- oracle/_ref/libssam_ref.so, the unmodified reference
                   (kernels.hpp CPU SSAM simulator + oracle.hpp), compiled
                   from /root/reference by oracle/Makefile.

Parity of ``Oracle`` is pinned against the reference through
tests/golden/ (see tests/test_oracle_golden.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libssam_ref.so")

DTYPES = {np.dtype(np.float32): 0, np.dtype(np.float64): 1, np.dtype(np.int64): 2}
NP_OF = {0: np.float32, 1: np.float64, 2: np.int64}

_p = C.c_void_p
_i = C.c_int
_u64 = C.c_uint64


def dtype_code(dt) -> int:
    return DTYPES[np.dtype(dt)]


def build(quiet: bool = True) -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE, "-j4"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_p)


def _taps_arrays(offsets, coeffs, dt):
    off = np.ascontiguousarray(np.asarray(offsets, dtype=np.int32).reshape(-1, 3))
    cf = np.ascontiguousarray(np.asarray(coeffs, dtype=dt).reshape(-1))
    if off.shape[0] != cf.shape[0]:
        raise ValueError("offsets and coeffs disagree in length")
    return off, cf


class Oracle:
    """Our C restatement (oracle/ssam_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        lib = C.CDLL(path)
        lib.ssam_oracle_random_grid.argtypes = [_i, _p, C.c_size_t, _u64, _u64]
        lib.ssam_oracle_random_filter.argtypes = [_i, _p, C.c_size_t, _u64]
        lib.ssam_oracle_conv2d.argtypes = [_i, _p, _i, _i, _p, _i, _i, _i, _p]
        lib.ssam_oracle_stencil2d.argtypes = [_i, _p, _i, _i, _p, _p, _i, _i, _i, _p]
        lib.ssam_oracle_stencil3d.argtypes = [_i, _p, _i, _i, _i, _p, _p, _i, _i, _i, _p]
        lib.ssam_oracle_benchmark_stencil.argtypes = [C.c_char_p, C.POINTER(_i), C.POINTER(_i),
                                                      C.POINTER(_i), _p, _p, _i]
        lib.ssam_oracle_benchmark_name.restype = C.c_char_p
        lib.ssam_oracle_conv1d.argtypes = [_i, _p, _i, _p, _i, _i, _p]
        lib.ssam_oracle_scan.argtypes = [_i, _p, C.c_size_t, _p]
        self.lib = lib

    # -- generators (grid.hpp:52-66, filter.hpp:41-47) --------------------
    def random_grid(self, shape, dtype, seed: int, first: int = 0) -> np.ndarray:
        a = np.empty(shape, dtype=dtype)
        self.lib.ssam_oracle_random_grid(dtype_code(dtype), _ptr(a), a.size, seed, first)
        return a

    def random_filter(self, m: int, n: int, dtype, seed: int) -> np.ndarray:
        """Weights w[s*n+t] as an (m, n) array (filter.hpp:25)."""
        a = np.empty((m, n), dtype=dtype)
        self.lib.ssam_oracle_random_filter(dtype_code(dtype), _ptr(a), a.size, seed)
        return a

    # -- oracle.hpp ---------------------------------------------------------
    def conv2d(self, grid: np.ndarray, weights: np.ndarray, boundary: int = 0) -> np.ndarray:
        g = np.ascontiguousarray(grid)
        w = np.ascontiguousarray(weights, dtype=g.dtype)
        h_, w_ = g.shape
        m, n = w.shape
        out = np.empty_like(g)
        rc = self.lib.ssam_oracle_conv2d(dtype_code(g.dtype), _ptr(g), w_, h_, _ptr(w), m, n,
                                         boundary, _ptr(out))
        assert rc == 0
        return out

    def stencil2d(self, grid, offsets, coeffs, order: int, iters: int) -> np.ndarray:
        g = np.ascontiguousarray(grid)
        off, cf = _taps_arrays(offsets, coeffs, g.dtype)
        h_, w_ = g.shape
        out = np.empty_like(g)
        rc = self.lib.ssam_oracle_stencil2d(dtype_code(g.dtype), _ptr(g), w_, h_, _ptr(off),
                                            _ptr(cf), off.shape[0], order, iters, _ptr(out))
        assert rc == 0
        return out

    def stencil3d(self, grid, offsets, coeffs, order: int, iters: int) -> np.ndarray:
        g = np.ascontiguousarray(grid)
        off, cf = _taps_arrays(offsets, coeffs, g.dtype)
        nz, ny, nx = g.shape
        out = np.empty_like(g)
        rc = self.lib.ssam_oracle_stencil3d(dtype_code(g.dtype), _ptr(g), nx, ny, nz, _ptr(off),
                                            _ptr(cf), off.shape[0], order, iters, _ptr(out))
        assert rc == 0
        return out

    def conv1d(self, signal: np.ndarray, filt: np.ndarray, boundary: int = 0) -> np.ndarray:
        """oracle::conv1d_naive (oracle.hpp:61-73)."""
        g = np.ascontiguousarray(signal)
        f = np.ascontiguousarray(filt, dtype=g.dtype)
        out = np.empty_like(g)
        rc = self.lib.ssam_oracle_conv1d(dtype_code(g.dtype), _ptr(g), g.size, _ptr(f), f.size,
                                         boundary, _ptr(out))
        assert rc == 0
        return out

    def scan(self, values: np.ndarray) -> np.ndarray:
        """oracle::scan_naive (oracle.hpp:118-127)."""
        g = np.ascontiguousarray(values)
        out = np.empty_like(g)
        assert self.lib.ssam_oracle_scan(dtype_code(g.dtype), _ptr(g), g.size, _ptr(out)) == 0
        return out

    # -- stencil_catalog.cpp ------------------------------------------------
    def benchmark_names(self):
        n = self.lib.ssam_oracle_benchmark_count()
        return [self.lib.ssam_oracle_benchmark_name(i).decode() for i in range(n)]

    def benchmark_stencil(self, name: str):
        """Returns dict(dims, order, fpp, offsets (t,3) int32, coeffs (t,) float64)."""
        off = np.zeros((125, 3), dtype=np.int32)
        cf = np.zeros(125, dtype=np.float64)
        dims, order, fpp = _i(), _i(), _i()
        t = self.lib.ssam_oracle_benchmark_stencil(name.encode(), C.byref(dims), C.byref(order),
                                                   C.byref(fpp), _ptr(off), _ptr(cf), 125)
        if t < 0:
            raise KeyError(name)
        return dict(name=name, dims=dims.value, order=order.value, fpp=fpp.value,
                    offsets=off[:t].copy(), coeffs=cf[:t].copy())


class Reference:
    """The unmodified reference compiled into oracle/_ref/libssam_ref.so."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: build it with `make -C oracle` where "
                                    "/root/reference exists")
        lib = C.CDLL(path)
        lib.ssam_ref_conv2d.argtypes = [_i, _p, _i, _i, _p, _i, _i, _i, _i, _i, _i, _i, _p, _p, _i]
        lib.ssam_ref_stencil2d.argtypes = [_i, _p, _i, _i, _i, _i, _p, _p, _i, _i, _i, _i, _i,
                                           _i, _p, _p, _i]
        lib.ssam_ref_stencil3d.argtypes = [_i, _p, _i, _i, _i, _i, _i, _p, _p, _i, _i, _i, _i,
                                           _i, _i, _p, _p, _i]
        lib.ssam_ref_random_grid.argtypes = [_i, _p, _i, _u64]
        lib.ssam_ref_random_filter.argtypes = [_i, _p, _i, _i, _u64]
        lib.ssam_ref_benchmark_stencil.argtypes = [C.c_char_p, C.POINTER(_i), C.POINTER(_i),
                                                   C.POINTER(_i), _p, _p, _i]
        lib.ssam_ref_conv1d.argtypes = [_i, _p, _i, _p, _i, _i, _i, _p, _p, _i]
        lib.ssam_ref_scan.argtypes = [_i, _p, _i, _i, _p, _p, _i]
        lib.ssam_ref_sgrd_write.argtypes = [_i, C.c_char_p, _i, _p, _p]
        lib.ssam_ref_sgrd_read.argtypes = [_i, C.c_char_p, _i, _p, _p, C.c_longlong]
        lib.ssam_ref_profile.argtypes = [C.c_char_p, C.c_char_p, _i, _p, _i, _i, _p]
        self.lib = lib

    def max_threads(self) -> int:
        return self.lib.ssam_ref_max_threads()

    def random_grid(self, count: int, dtype, seed: int) -> np.ndarray:
        a = np.empty(count, dtype=dtype)
        assert self.lib.ssam_ref_random_grid(dtype_code(dtype), _ptr(a), count, seed) == 0
        return a

    def random_filter(self, m, n, dtype, seed) -> np.ndarray:
        a = np.empty((m, n), dtype=dtype)
        assert self.lib.ssam_ref_random_filter(dtype_code(dtype), _ptr(a), m, n, seed) == 0
        return a

    def benchmark_stencil(self, name: str):
        off = np.zeros((125, 3), dtype=np.int32)
        cf = np.zeros(125, dtype=np.float64)
        dims, order, fpp = _i(), _i(), _i()
        t = self.lib.ssam_ref_benchmark_stencil(name.encode(), C.byref(dims), C.byref(order),
                                                C.byref(fpp), _ptr(off), _ptr(cf), 125)
        if t < 0:
            raise KeyError(name)
        return dict(name=name, dims=dims.value, order=order.value, fpp=fpp.value,
                    offsets=off[:t].copy(), coeffs=cf[:t].copy())

    def conv2d(self, grid, weights, *, p=4, b=128, boundary=0, lane_count=32, threads=0,
               naive=False):
        """ssam::conv2d (naive=False) or oracle::conv2d_naive.  Returns (status, out, counters)."""
        g = np.ascontiguousarray(grid)
        w = np.ascontiguousarray(weights, dtype=g.dtype)
        out = np.zeros_like(g)
        cnt = np.zeros(5, dtype=np.uint64)
        h_, w_ = g.shape
        m, n = w.shape
        rc = self.lib.ssam_ref_conv2d(dtype_code(g.dtype), _ptr(g), w_, h_, _ptr(w), m, n, p, b,
                                      boundary, lane_count, threads, _ptr(out), _ptr(cnt),
                                      int(naive))
        return rc, out, cnt

    def stencil2d(self, grid, offsets, coeffs, order, iters, *, dims=2, p=4, b=128,
                  lane_count=32, threads=0, naive=False):
        g = np.ascontiguousarray(grid)
        off, cf = _taps_arrays(offsets, coeffs, g.dtype)
        out = np.zeros_like(g)
        cnt = np.zeros(5, dtype=np.uint64)
        h_, w_ = g.shape
        rc = self.lib.ssam_ref_stencil2d(dtype_code(g.dtype), _ptr(g), w_, h_, dims, order,
                                         _ptr(off), _ptr(cf), off.shape[0], p, b, lane_count,
                                         threads, iters, _ptr(out), _ptr(cnt), int(naive))
        return rc, out, cnt

    def stencil3d(self, grid, offsets, coeffs, order, iters, *, dims=3, p=2, b=None,
                  lane_count=32, threads=0, naive=False):
        g = np.ascontiguousarray(grid)
        off, cf = _taps_arrays(offsets, coeffs, g.dtype)
        if b is None:
            b = max(128, 32 * (2 * order + 1))
        out = np.zeros_like(g)
        cnt = np.zeros(5, dtype=np.uint64)
        nz, ny, nx = g.shape
        rc = self.lib.ssam_ref_stencil3d(dtype_code(g.dtype), _ptr(g), nx, ny, nz, dims, order,
                                         _ptr(off), _ptr(cf), off.shape[0], p, b, lane_count,
                                         threads, iters, _ptr(out), _ptr(cnt), int(naive))
        return rc, out, cnt

    def conv1d(self, signal, filt, *, boundary=0, lane_count=32, naive=False):
        """ssam::conv1d (kernels.hpp:390-418) or oracle::conv1d_naive -> (status, out, counters)."""
        g = np.ascontiguousarray(signal)
        f = np.ascontiguousarray(filt, dtype=g.dtype)
        out = np.zeros_like(g)
        cnt = np.zeros(5, dtype=np.uint64)
        rc = self.lib.ssam_ref_conv1d(dtype_code(g.dtype), _ptr(g), g.size, _ptr(f), f.size,
                                      boundary, lane_count, _ptr(out), _ptr(cnt), int(naive))
        return rc, out, cnt

    def scan(self, values, *, lane_count=32, naive=False):
        """ssam::scan (kernels.hpp:422-447) or oracle::scan_naive -> (status, out, counters)."""
        g = np.ascontiguousarray(values)
        out = np.zeros_like(g)
        cnt = np.zeros(5, dtype=np.uint64)
        rc = self.lib.ssam_ref_scan(dtype_code(g.dtype), _ptr(g), g.size, lane_count, _ptr(out),
                                    _ptr(cnt), int(naive))
        return rc, out, cnt

    def sgrd_write(self, path: str, a: np.ndarray) -> int:
        """ssam::write_grid_file (grid_io.hpp:129-134); rank = a.ndim, dims x-fastest."""
        a = np.ascontiguousarray(a)
        dims = np.array(list(a.shape[::-1]) + [1] * (3 - a.ndim), dtype=np.int32)
        return self.lib.ssam_ref_sgrd_write(dtype_code(a.dtype), path.encode(), a.ndim,
                                            _ptr(dims), _ptr(a))

    def sgrd_read(self, path: str, dtype, rank: int, cap: int = 1 << 24):
        """read_vector / read_grid2d / read_grid3d -> (status, array or None)."""
        dims = np.zeros(3, dtype=np.int32)
        buf = np.zeros(cap, dtype=dtype)
        rc = self.lib.ssam_ref_sgrd_read(dtype_code(dtype), path.encode(), rank, _ptr(dims),
                                         _ptr(buf), cap)
        if rc != 0:
            return rc, None
        shape = tuple(int(d) for d in dims[:rank][::-1])
        return 0, buf[:int(np.prod(shape))].reshape(shape).copy()


    def profile(self, name_or_path: str, m: int = 3, n: int = 3):
        """ssam::resolve_profile (perf_model.cpp:89-97) -> (status, name, six latencies,
        (latency_reg, latency_smem) at m x n)."""
        name = C.create_string_buffer(64)
        vals = np.zeros(6, dtype=np.float64)
        lat = np.zeros(2, dtype=np.float64)
        rc = self.lib.ssam_ref_profile(name_or_path.encode(), name, 64, _ptr(vals), m, n,
                                       _ptr(lat))
        return rc, name.value.decode(), vals, lat


def max_rel_err(got: np.ndarray, want: np.ndarray) -> float:
    """max_i |got-want| / max(1, |want|) -- proj/tests/acceptance.cpp:35-44."""
    g = np.asarray(got, dtype=np.float64)
    w = np.asarray(want, dtype=np.float64)
    if g.size == 0:
        return 0.0
    return float(np.max(np.abs(g - w) / np.maximum(1.0, np.abs(w))))


def max_abs_err(got, want) -> float:
    g = np.asarray(got, dtype=np.float64)
    w = np.asarray(want, dtype=np.float64)
    return float(np.max(np.abs(g - w))) if g.size else 0.0
