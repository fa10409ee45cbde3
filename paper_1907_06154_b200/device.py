"""Device-resident entry points (benchmarks, multi-GPU slabs).

torch supplies device memory and streams (plumbing); every computation is a
kernel in libssam_b200.so launched on the given (default: current) stream.
Tensors must be contiguous CUDA tensors of float32, float64 or int64.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Tuple

import numpy as np

from . import (_DT, _PeerHalo, _StencilArgs, _lib, _raise, InvalidArgument, Stencil)

_TORCH_DT = None


def _torch():
    import torch
    return torch


def _code(t) -> int:
    torch = _torch()
    m = {torch.float32: 0, torch.float64: 1, torch.int64: 2}
    if t.dtype not in m:
        raise InvalidArgument(f"unsupported dtype {t.dtype}")
    if not t.is_cuda or not t.is_contiguous():
        raise InvalidArgument("expected a contiguous CUDA tensor")
    return m[t.dtype]


def _np_dtype(code: int):
    return {0: np.float32, 1: np.float64, 2: np.int64}[code]


def _s(stream) -> int:
    torch = _torch()
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def conv2d(d_in, d_out, weights, boundary: int = 0, y_begin: int = 0,
           y_end: Optional[int] = None, stream=None) -> None:
    """conv2d over output rows [y_begin, y_end) of (H, W) tensors."""
    code = _code(d_in)
    H, W = d_in.shape
    w = np.ascontiguousarray(np.asarray(weights).astype(_np_dtype(code)))
    _raise(_lib.ssam_b200_conv2d_device(code, d_in.data_ptr(), d_out.data_ptr(), W, H, y_begin,
                                        H if y_end is None else y_end, w.ctypes.data,
                                        w.shape[0], w.shape[1], int(boundary), _s(stream)))


def stencil2d_sweep(d_in, d_out, st: Stencil, y_begin: int = 0, y_end: Optional[int] = None,
                    stream=None) -> None:
    code = _code(d_in)
    H, W = d_in.shape
    sa = _StencilArgs(st, _np_dtype(code))
    _raise(_lib.ssam_b200_stencil2d_sweep(code, d_in.data_ptr(), d_out.data_ptr(), W, H, y_begin,
                                          H if y_end is None else y_end, sa.ref, _s(stream)))


def stencil2d_tb(d_in, d_out, st: Stencil, tb: int, y_begin: Optional[int] = None,
                 y_end: Optional[int] = None, y_ring_lo: Optional[int] = None,
                 y_ring_hi: Optional[int] = None, stream=None) -> None:
    """tb fused 2D sweeps; with row bounds, only output rows [y_begin, y_end)
    and rows outside [y_ring_lo, y_ring_hi) kept as the global ring (row slabs)."""
    code = _code(d_in)
    H, W = d_in.shape
    sa = _StencilArgs(st, _np_dtype(code))
    if y_begin is None and y_end is None and y_ring_lo is None and y_ring_hi is None:
        _raise(_lib.ssam_b200_stencil2d_tb(code, d_in.data_ptr(), d_out.data_ptr(), W, H, sa.ref,
                                           tb, _s(stream)))
        return
    k = st.order
    _raise(_lib.ssam_b200_stencil2d_tb_range(
        code, d_in.data_ptr(), d_out.data_ptr(), W, H, k if y_begin is None else y_begin,
        H - k if y_end is None else y_end, k if y_ring_lo is None else y_ring_lo,
        H - k if y_ring_hi is None else y_ring_hi, sa.ref, tb, _s(stream)))


def stencil2d_tb_max(st: Stencil, dtype) -> int:
    sa = _StencilArgs(st, dtype)
    return int(_lib.ssam_b200_stencil2d_tb_max(_DT[np.dtype(dtype)], sa.ref))


def stencil2d_run(d_a, d_b, st: Stencil, iters: int, tb: int = 0, stream=None):
    """iters sweeps ping-ponging d_a/d_b; returns whichever holds the result."""
    code = _code(d_a)
    H, W = d_a.shape
    sa = _StencilArgs(st, _np_dtype(code))
    res = C.c_void_p()
    _raise(_lib.ssam_b200_stencil2d_run(code, d_a.data_ptr(), d_b.data_ptr(), W, H, sa.ref,
                                        iters, tb, _s(stream), C.byref(res)))
    return d_a if res.value == d_a.data_ptr() else d_b


def stencil3d_sweep(d_in, d_out, st: Stencil, z_begin: int = 0, z_end: Optional[int] = None,
                    stream=None, peer: Optional[_PeerHalo] = None) -> None:
    """One sweep over output planes [z_begin, z_end); `peer` (ssam_peer_halo)
    also stores the planes neighbours mirror into their buffers."""
    code = _code(d_in)
    nz, ny, nx = d_in.shape
    sa = _StencilArgs(st, _np_dtype(code))
    ze = nz if z_end is None else z_end
    if peer is None:
        _raise(_lib.ssam_b200_stencil3d_sweep(code, d_in.data_ptr(), d_out.data_ptr(), nx, ny, nz,
                                              z_begin, ze, sa.ref, _s(stream)))
    else:
        _raise(_lib.ssam_b200_stencil3d_sweep_peer(code, d_in.data_ptr(), d_out.data_ptr(), nx, ny,
                                                   nz, z_begin, ze, sa.ref, C.byref(peer),
                                                   _s(stream)))


def stencil3d_tb(d_in, d_out, st: Stencil, tb: int, z_begin: int = 0,
                 z_end: Optional[int] = None, z_ring_lo: Optional[int] = None,
                 z_ring_hi: Optional[int] = None, stream=None,
                 peer: Optional[_PeerHalo] = None) -> None:
    """tb fused 3D sweeps (order-1 stencils, tb = 2) writing planes [z_begin, z_end);
    planes outside [z_ring_lo, z_ring_hi) (default: the buffer's own ring) stay fixed."""
    code = _code(d_in)
    nz, ny, nx = d_in.shape
    sa = _StencilArgs(st, _np_dtype(code))
    k = st.order
    args = (code, d_in.data_ptr(), d_out.data_ptr(), nx, ny, nz, z_begin,
            nz if z_end is None else z_end, k if z_ring_lo is None else z_ring_lo,
            nz - k if z_ring_hi is None else z_ring_hi, sa.ref, tb)
    if peer is None:
        _raise(_lib.ssam_b200_stencil3d_tb(*args, _s(stream)))
    else:
        _raise(_lib.ssam_b200_stencil3d_tb_peer(*args, C.byref(peer), _s(stream)))


def stencil3d_tb_max(st: Stencil, dtype) -> int:
    sa = _StencilArgs(st, dtype)
    return int(_lib.ssam_b200_stencil3d_tb_max(_DT[np.dtype(dtype)], sa.ref))


def stencil3d_run(d_a, d_b, st: Stencil, iters: int, stream=None):
    code = _code(d_a)
    nz, ny, nx = d_a.shape
    sa = _StencilArgs(st, _np_dtype(code))
    res = C.c_void_p()
    _raise(_lib.ssam_b200_stencil3d_run(code, d_a.data_ptr(), d_b.data_ptr(), nx, ny, nz, sa.ref,
                                        iters, _s(stream), C.byref(res)))
    return d_a if res.value == d_a.data_ptr() else d_b


def gather_run(d_a, d_b, st: Stencil, iters: int, stream=None):
    """`iters` direct-gather sweeps (the oracle's summation order and arithmetic)
    on device buffers; returns whichever of d_a / d_b holds the result."""
    code = _code(d_a)
    if d_a.dim() == 2:
        (ny, nx), nz = d_a.shape, 1
    else:
        nz, ny, nx = d_a.shape
    sa = _StencilArgs(st, _np_dtype(code))
    res = C.c_void_p()
    _raise(_lib.ssam_b200_gather_stencil_run(code, d_a.data_ptr(), d_b.data_ptr(), nx, ny, nz,
                                             sa.ref, iters, _s(stream), C.byref(res)))
    return d_a if res.value == d_a.data_ptr() else d_b


def fill_random(t, seed: int, first: int = 0, stream=None) -> None:
    """SplitMix64 fill bit-identical to random_grid2d/3d (element i = draw first+i)."""
    _raise(_lib.ssam_b200_fill_random(_code(t), t.data_ptr(), t.numel(), seed, first,
                                      _s(stream)))


def max_rel_err(a, b, stream=None) -> Tuple[float, float]:
    """(max |a-b|/max(1,|b|), max |a-b|) reduced on the device."""
    rel, ab = C.c_double(), C.c_double()
    _raise(_lib.ssam_b200_max_rel_err(_code(a), a.data_ptr(), b.data_ptr(), a.numel(),
                                      C.byref(rel), C.byref(ab), _s(stream)))
    return rel.value, ab.value


def conv1d(d_in, d_out, weights, boundary: int = 0, stream=None) -> None:
    """conv1d of a 1D device signal (m <= 32)."""
    code = _code(d_in)
    w = np.ascontiguousarray(np.asarray(weights).astype(_np_dtype(code)).reshape(-1))
    _raise(_lib.ssam_b200_conv1d_device(code, d_in.data_ptr(), d_out.data_ptr(), d_in.numel(),
                                        w.ctypes.data, w.size, int(boundary), _s(stream)))


def scan(d_in, d_out, stream=None) -> None:
    """Inclusive prefix sum of a device tensor (flattened)."""
    code = _code(d_in)
    _raise(_lib.ssam_b200_scan_device(code, d_in.data_ptr(), d_out.data_ptr(), d_in.numel(),
                                      _s(stream)))


def read_grid(path: str, dtype=None, rank: Optional[int] = None, stream=None):
    """SGRD file -> a new CUDA tensor (payload streamed through pinned buffers)."""
    import os
    from . import sgrd_info, _DT
    torch = _torch()
    frank, fdt, dims = sgrd_info(path)
    rank = rank or frank
    dtype = np.dtype(dtype or fdt)
    shape = tuple(dims[:rank][::-1])
    tdt = {0: torch.float32, 1: torch.float64, 2: torch.int64}[_DT[dtype]]
    t = torch.empty(shape, dtype=tdt, device="cuda")
    d = np.zeros(3, dtype=np.int32)
    _raise(_lib.ssam_b200_sgrd_read(os.fsencode(path), _DT[dtype], rank, d.ctypes.data,
                                    t.data_ptr(), t.numel(), 1, _s(stream)))
    return t


def write_grid(path: str, t, stream=None) -> None:
    """A contiguous CUDA tensor (1-3D, x fastest) -> SGRD file."""
    import os
    code = _code(t)
    if t.dim() not in (1, 2, 3):
        raise InvalidArgument("grid io: need a 1-3D tensor")
    dims = np.array(list(t.shape[::-1]) + [1] * (3 - t.dim()), dtype=np.int32)
    _raise(_lib.ssam_b200_sgrd_write(os.fsencode(path), code, t.dim(), dims.ctypes.data,
                                     t.data_ptr(), 1, _s(stream)))
