"""Z-slab runs with the halo written by the sweep kernel over peer memory.

The NCCL transport (slab.py) computes the boundary planes, then runs a
send/recv pair per neighbour while the interior is computed.  Here there is
no exchange step: every rank's two slab buffers are CUDA IPC allocations
mapped into its neighbours' address spaces (NVLink P2P between GPUs of one
node, plain device memory when ranks share a GPU), and the z-streaming sweep
kernel stores each output row of a plane its neighbour mirrors twice -- into
its own buffer and straight into the neighbour's ghost slot
(ssam_b200_stencil3d_sweep_peer / _tb_peer, engine3d.cuh store_row3).  The
transfer rides on the kernel's own stores, tile by tile.

Ordering.  Sweep t of rank r writes neighbour buffers that the neighbour read
in its sweep t-1 (ping-pong parity), and reads ghosts the neighbours wrote in
their sweep t-1.  So every sweep waits, on the device, for the neighbours'
previous sweep, through generation flags: each rank owns two 32-bit words
(IPC memory, one per neighbour); after its sweep t a rank's stream writes
t+1 into the word each neighbour keeps for it (cuStreamWriteValue32, after
the sweep's peer stores are visible), and before sweep t+1 its stream waits
until both of its own words are >= t+1 (cuStreamWaitValue32).  No host
barrier per sweep: the host only enqueues, the GPU front end does the
waiting.  (SSAM_PEER_HOST_BARRIER=1 selects the previous protocol:
interprocess events made visible by a gloo barrier per sweep.)

Layout and decomposition are slab.py's (Slab, decompose, fill_slab): local
plane p is global plane z_first - ghost + p, ghost = k * Tb.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np
import torch
import torch.distributed as dist

from . import _PeerHalo, _raise, IPC_HANDLE_BYTES, Stencil, lib
from . import device as dev
from .slab import Slab

_TYPESTR = {torch.float32: "<f4", torch.float64: "<f8", torch.int64: "<i8"}


class _Cai:
    def __init__(self, ptr: int, shape, dtype):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": _TYPESTR[dtype],
                                         "data": (ptr, False), "version": 2, "strides": None}


class IpcBuffer:
    """A cudaMalloc'd slab buffer with its CUDA IPC handle; `.tensor` views it."""

    def __init__(self, shape, dtype: torch.dtype):
        nbytes = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
        ptr, h = C.c_void_p(), C.create_string_buffer(IPC_HANDLE_BYTES)
        _raise(lib.ssam_b200_ipc_alloc(nbytes, C.byref(ptr), h))
        self.ptr = ptr.value
        self.handle = h.raw
        self.tensor = torch.as_tensor(_Cai(self.ptr, shape, dtype), device="cuda")

    def free(self) -> None:
        if self.ptr:
            self.tensor = None
            _raise(lib.ssam_b200_ipc_free(self.ptr))
            self.ptr = 0


def _open(handle: bytes) -> int:
    ptr = C.c_void_p()
    _raise(lib.ssam_b200_ipc_open(C.create_string_buffer(handle, IPC_HANDLE_BYTES), C.byref(ptr)))
    return ptr.value


def peer_geometry(slab: Slab, nz_own_below: int, plane: int):
    """(lo_shift, lo_end, hi_shift, hi_begin) of ssam_peer_halo for this rank:
    my local planes z < lo_end are rank-1's top ghost planes at element offset
    + lo_shift (its local index = mine + nz_own of rank-1), planes z >= hi_begin
    rank+1's bottom ghosts at + hi_shift (its index = mine - my nz_own)."""
    own_lo = slab.local(slab.z_first)
    own_hi = own_lo + slab.nz_own
    return (nz_own_below * plane, own_lo + slab.ghost, -slab.nz_own * plane, own_hi - slab.ghost)


class PeerSlabRunner:
    """Jacobi sweeps on one rank's slab, halos stored by the kernel into the
    neighbours' buffers.  `group` must be a host-side (gloo) group; it carries
    the one-time handle exchange and the per-sweep barrier."""

    def __init__(self, slab: Slab, st: Stencil, nx: int, ny: int, dtype: torch.dtype,
                 group=None, tb: int = 1):
        if tb > 1 and slab.ghost < slab.order * tb:
            raise ValueError(f"Tb={tb} needs ghost >= {slab.order * tb}")
        self.slab, self.st, self.tb, self.group = slab, st, tb, group
        self.shape = (slab.nz_local, ny, nx)
        self.bufs = [IpcBuffer(self.shape, dtype), IpcBuffer(self.shape, dtype)]
        self.events = [torch.cuda.Event(interprocess=True) for _ in range(2)]
        # generation flags: word 0 written by rank-1, word 1 by rank+1
        self.flags = IpcBuffer((2,), torch.int64)
        self.flags.tensor.zero_()
        torch.cuda.synchronize()  # zeroed before any neighbour can signal
        self.host_barrier = os.environ.get("SSAM_PEER_HOST_BARRIER", "0") == "1"
        self.gen = 0
        dev_idx = torch.cuda.current_device()
        info = {"nz_own": slab.nz_own, "bufs": [b.handle for b in self.bufs],
                "flags": self.flags.handle,
                "events": [bytes(e.ipc_handle()) for e in self.events]}
        allinfo = [None] * slab.world
        dist.all_gather_object(allinfo, info, group=group)
        below = allinfo[slab.rank - 1]["nz_own"] if slab.rank > 0 else 0
        lo_shift, lo_end, hi_shift, hi_begin = peer_geometry(slab, below, nx * ny)
        self.opened = []
        self.nb_flags = []  # (address of my word in the neighbour's flags)
        self.nb_events = [[], []]
        self.halo = [_PeerHalo(), _PeerHalo()]
        for side, nb in ((0, slab.rank - 1), (1, slab.rank + 1)):
            if not 0 <= nb < slab.world:
                continue
            fptr = _open(allinfo[nb]["flags"])
            self.opened.append(fptr)
            # rank-1 keeps my word at index 1 (from its upper neighbour), rank+1 at 0
            self.nb_flags.append(fptr + (8 if side == 0 else 0))
            for j in range(2):
                ptr = _open(allinfo[nb]["bufs"][j])
                self.opened.append(ptr)
                h = self.halo[j]
                if side == 0:  # rank-1 mirrors my lowest `ghost` owned planes as its top ghosts
                    h.lo, h.lo_shift, h.lo_end = ptr, lo_shift, lo_end
                else:          # rank+1 mirrors my highest as its bottom ghosts
                    h.hi, h.hi_shift, h.hi_begin = ptr, hi_shift, hi_begin
                self.nb_events[j].append(
                    torch.cuda.Event.from_ipc_handle(dev_idx, allinfo[nb]["events"][j]))
        self._parity = 0

    @property
    def a(self) -> torch.Tensor:
        return self.bufs[0].tensor

    @property
    def b(self) -> torch.Tensor:
        return self.bufs[1].tensor

    def _publish(self, stream) -> None:
        """Signal the neighbours that the work queued so far is done and make
        the stream wait (on the device) until they signalled the same
        generation."""
        if not self.host_barrier:
            self.gen += 1
            sp = C.c_void_p(stream.cuda_stream)
            for addr in self.nb_flags:
                _raise(lib.ssam_b200_stream_write_u32(C.c_void_p(addr), self.gen, sp))
            s = self.slab
            for word, nb in ((0, s.rank - 1), (1, s.rank + 1)):
                if 0 <= nb < s.world:
                    _raise(lib.ssam_b200_stream_wait_u32(
                        C.c_void_p(self.flags.ptr + 8 * word), self.gen, sp))
            return
        p = self._parity
        self.events[p].record(stream)
        dist.barrier(group=self.group)
        for ev in self.nb_events[p]:
            stream.wait_event(ev)
        self._parity ^= 1

    def run(self, iters: int, stream=None) -> torch.Tensor:
        """iters sweeps from buffer a (input; b must hold a copy of it, ring and
        ghosts included).  Returns the buffer holding the final generation."""
        s = self.slab
        stream = stream or torch.cuda.current_stream()
        lo, hi = s.compute_range()
        rlo, rhi = s.ring_bounds()
        cur, nxt = 0, 1
        self._publish(stream)  # neighbours' buffers initialised before we write into them
        done = 0
        while done < iters:
            fused = self.tb > 1 and iters - done >= self.tb
            c, n = self.bufs[cur].tensor, self.bufs[nxt].tensor
            peer = self.halo[nxt] if s.world > 1 else None
            with torch.cuda.stream(stream):
                if fused:
                    dev.stencil3d_tb(c, n, self.st, self.tb, lo, hi, rlo, rhi, stream=stream,
                                     peer=peer)
                else:
                    dev.stencil3d_sweep(c, n, self.st, lo, hi, stream=stream, peer=peer)
            self._publish(stream)
            cur, nxt = nxt, cur
            done += self.tb if fused else 1
        return self.bufs[cur].tensor

    def __enter__(self) -> "PeerSlabRunner":
        return self

    def __exit__(self, *exc) -> None:
        self.close()

    def close(self) -> None:
        """Collective (every rank calls it): unmaps the neighbours' buffers and
        frees this rank's."""
        if not self.bufs:
            return
        torch.cuda.synchronize()
        dist.barrier(group=self.group)  # no neighbour still writes into our buffers
        for ptr in self.opened:
            _raise(lib.ssam_b200_ipc_close(ptr))
        self.opened = []
        dist.barrier(group=self.group)  # every mapping of our buffers is closed
        for b in self.bufs:
            b.free()
        self.flags.free()
        self.bufs = []
