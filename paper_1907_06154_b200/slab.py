"""Multi-GPU z-slab decomposition with halo exchange.

One process per GPU.  A 3D grid of nz_global planes (x fastest,
data[(z*ny + y)*nx + x], grid.hpp:30-49) is split along z -- the slowest
axis, so every slab and every halo is a contiguous run of planes.  Rank r
holds its owned planes plus `ghost` planes on each side:

    local plane p  <->  global plane z_first - ghost + p,   p in [0, nz_own + 2*ghost)

One sweep writes the owned planes that are interior to the GLOBAL domain
(the global ring of width k is never written, exactly as
oracle::stencil3d_naive leaves it), then the new boundary planes are swapped
with the neighbours: my lowest `ghost` owned planes go to rank-1's top ghost
slots, my highest to rank+1's bottom ghost slots.  That is the only exchange
the path has -- a pairwise neighbour send/recv, not a reduction.

Overlap (per sweep): the 2*ghost boundary planes are computed first, their
exchange runs on a communication stream while the interior planes are
computed, and the next sweep waits only for the receives.

Temporal blocking (Tb fused sweeps per step, ssam_b200_stencil3d_tb): with
ghost = k*Tb planes a rank can run Tb sweeps on its owned planes before it
needs its neighbours' new planes, so the exchange happens once per Tb sweeps
with the same plane count per message.  The global ring is passed to the
fused kernel in local plane coordinates (`ring_bounds`).

The exchange goes through torch.distributed (NCCL over NVLink on a B200 box,
gloo on CPU for tests).  The sweep itself is pluggable so the CPU tests can
drive the identical decomposition/exchange code with the oracle; in the
product it is the CUDA z-streaming kernel (ssam_b200_stencil3d_sweep).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Slab:
    rank: int
    world: int
    nz_global: int
    z_first: int   # first owned global plane
    nz_own: int
    ghost: int
    order: int

    @property
    def nz_local(self) -> int:
        return self.nz_own + 2 * self.ghost

    def local(self, z_global: int) -> int:
        return z_global - self.z_first + self.ghost

    def compute_range(self):
        """Local output planes of one sweep: owned ∩ global interior [k, nz-k)."""
        lo = max(self.z_first, self.order)
        hi = min(self.z_first + self.nz_own, self.nz_global - self.order)
        return self.local(lo), self.local(max(lo, hi))

    def ring_bounds(self):
        """Local plane range [lo, hi) of the GLOBAL interior (may lie outside the buffer)."""
        return self.local(self.order), self.local(self.nz_global - self.order)

    def boundary_ranges(self):
        """(low, high) boundary plane ranges whose results neighbours need."""
        lo, hi = self.compute_range()
        g = self.ghost
        low = (lo, min(hi, self.local(self.z_first) + g)) if self.rank > 0 else (lo, lo)
        top_own = self.local(self.z_first + self.nz_own)
        high = (max(lo, top_own - g), hi) if self.rank < self.world - 1 else (hi, hi)
        return low, high


def decompose(nz_global: int, world: int, rank: int, order: int, ghost: Optional[int] = None) -> Slab:
    """Even split of nz_global planes over world ranks (the first
    nz_global % world ranks own one extra plane)."""
    g = order if ghost is None else ghost
    base, extra = divmod(nz_global, world)
    nz_own = base + (1 if rank < extra else 0)
    z_first = rank * base + min(rank, extra)
    if nz_own < g:
        raise ValueError(f"slab of {nz_own} planes is thinner than the {g}-plane halo")
    return Slab(rank, world, nz_global, z_first, nz_own, g, order)


SweepFn = Callable[[torch.Tensor, torch.Tensor, int, int], None]  # (cur, nxt, z_begin, z_end)
# (cur, nxt, z_begin, z_end): `tb` fused sweeps writing nxt planes [z_begin, z_end)


class SlabRunner:
    """Runs Jacobi sweeps on one rank's slab with neighbour halo exchange."""

    def __init__(self, slab: Slab, sweep: SweepFn, group=None, comm_stream=None,
                 fused: Optional[SweepFn] = None, tb: int = 1):
        if tb > 1 and (fused is None or slab.ghost < slab.order * tb):
            raise ValueError(f"Tb={tb} needs a fused sweep and ghost >= {slab.order * tb}")
        self.slab = slab
        self.sweep = sweep
        self.fused = fused
        self.tb = tb
        self.group = group
        self.cuda = comm_stream is not None
        self.comm_stream = comm_stream

    def _staged(self, nxt: torch.Tensor) -> bool:
        """CUDA tensors over a host-only backend (gloo): stage halos through host memory."""
        return nxt.is_cuda and dist.get_backend(self.group) != "nccl"

    def _exchange_staged(self, nxt: torch.Tensor) -> None:
        s, g = self.slab, self.slab.ghost
        own_lo = s.local(s.z_first)
        own_hi = own_lo + s.nz_own
        ops, recvs = [], []
        if s.rank > 0:
            ops.append(dist.P2POp(dist.isend, nxt[own_lo:own_lo + g].cpu(), s.rank - 1, self.group))
            buf = torch.empty_like(nxt[own_lo - g:own_lo], device="cpu")
            ops.append(dist.P2POp(dist.irecv, buf, s.rank - 1, self.group))
            recvs.append((own_lo - g, buf))
        if s.rank < s.world - 1:
            ops.append(dist.P2POp(dist.isend, nxt[own_hi - g:own_hi].cpu(), s.rank + 1, self.group))
            buf = torch.empty_like(nxt[own_hi:own_hi + g], device="cpu")
            ops.append(dist.P2POp(dist.irecv, buf, s.rank + 1, self.group))
            recvs.append((own_hi, buf))
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        for z, buf in recvs:
            nxt[z:z + g].copy_(buf)

    def _exchange(self, nxt: torch.Tensor) -> list:
        s, g = self.slab, self.slab.ghost
        if s.world == 1 or g == 0:
            return []
        ops = []
        own_lo = s.local(s.z_first)
        own_hi = own_lo + s.nz_own
        if s.rank > 0:
            ops.append(dist.P2POp(dist.isend, nxt[own_lo:own_lo + g], s.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, nxt[own_lo - g:own_lo], s.rank - 1, self.group))
        if s.rank < s.world - 1:
            ops.append(dist.P2POp(dist.isend, nxt[own_hi - g:own_hi], s.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, nxt[own_hi:own_hi + g], s.rank + 1, self.group))
        return dist.batch_isend_irecv(ops)

    def step(self, cur: torch.Tensor, nxt: torch.Tensor, fused: bool = False) -> None:
        """One sweep (or self.tb fused sweeps) cur -> nxt including the halo
        exchange of nxt."""
        s = self.slab
        lo, hi = s.compute_range()
        (bl0, bl1), (bh0, bh1) = s.boundary_ranges()
        sweep = self.fused if fused else self.sweep
        if s.world == 1:
            sweep(cur, nxt, lo, hi)
            return
        # boundary planes first ...
        if bl1 > bl0:
            sweep(cur, nxt, bl0, bl1)
        if bh1 > max(bh0, bl1):  # thin slabs: the two boundary bands may touch
            sweep(cur, nxt, max(bh0, bl1), bh1)
        if self._staged(nxt):  # test mode: no overlap
            if bh0 > bl1:
                sweep(cur, nxt, bl1, bh0)
            self._exchange_staged(nxt)
        elif self.cuda:
            main = torch.cuda.current_stream()
            self.comm_stream.wait_stream(main)
            with torch.cuda.stream(self.comm_stream):
                reqs = self._exchange(nxt)
            # ... interior while the halo is in flight
            if bh0 > bl1:
                sweep(cur, nxt, bl1, bh0)
            for r in reqs:
                r.wait()
            main.wait_stream(self.comm_stream)
        else:
            reqs = self._exchange(nxt)
            if bh0 > bl1:
                sweep(cur, nxt, bl1, bh0)
            for r in reqs:
                r.wait()

    def run(self, a: torch.Tensor, b: torch.Tensor, iters: int) -> torch.Tensor:
        """iters sweeps; a holds the input, b must hold a copy of it (ring and
        ghosts).  Returns the buffer with the final generation."""
        cur, nxt = a, b
        done = 0
        while done < iters:
            fused = self.tb > 1 and iters - done >= self.tb
            self.step(cur, nxt, fused)
            cur, nxt = nxt, cur
            done += self.tb if fused else 1
        return cur


def fill_slab(t: torch.Tensor, slab: Slab, nx: int, ny: int, seed: int) -> None:
    """Fill a local slab buffer (owned + ghost planes) with the global
    random_grid3d stream: local plane p is global plane z_first - ghost + p,
    so every rank generates exactly its planes of the global grid."""
    from .device import fill_random
    plane = nx * ny
    z0 = slab.z_first - slab.ghost
    p0 = max(0, -z0)
    p1 = min(slab.nz_local, slab.nz_global - z0)
    if p1 > p0:
        fill_random(t[p0:p1].view(-1), seed, first=(z0 + p0) * plane)
    if p0 > 0:
        t[:p0].zero_()
    if p1 < slab.nz_local:
        t[p1:].zero_()


# ---------------------------------------------------------------------------
# 2D: row slabs ("z for 3D, y for 2D").  A (H, W) grid is the
# nz = H, ny = 1 case of the layout above -- rows are the planes -- so
# decompose / SlabRunner / fill_slab(t, slab, W, 1, seed) apply unchanged,
# with device.stencil2d_sweep(cur, nxt, st, y_begin, y_end) as the sweep.
# conv2d is a single pass over a read-only input: no exchange at all, each
# rank reads its rows plus the filter's halo rows.
# ---------------------------------------------------------------------------

def conv2d_halo(n: int) -> int:
    """Ghost rows a conv2d row slab needs for an n-row filter (anchor
    ay = (n-1)/2 above, n-1-ay below; oracle.hpp:40-56)."""
    return n - 1 - (n - 1) // 2


def replicate_outside(t: torch.Tensor, slab: Slab) -> None:
    """Ghost planes beyond the global domain take the nearest edge plane (the
    replicate boundary, clamp per axis: oracle.hpp:21-28)."""
    z0 = slab.z_first - slab.ghost
    p0 = max(0, -z0)
    p1 = min(slab.nz_local, slab.nz_global - z0)
    if p0 > 0:
        t[:p0].copy_(t[p0:p0 + 1].expand_as(t[:p0]))
    if p1 < slab.nz_local:
        t[p1:].copy_(t[p1 - 1:p1].expand_as(t[p1:]))


def conv2d_slab(d_in: torch.Tensor, d_out: torch.Tensor, weights, slab: Slab,
                boundary: int = 0, stream=None) -> None:
    """conv2d of this rank's owned rows.  d_in holds owned rows plus
    slab.ghost >= conv2d_halo(n) rows each side (fill_slab; zeros beyond the
    domain for the zero boundary, replicate_outside for replicate); the result
    lands in d_out's owned rows, equal to the one-GPU conv2d's."""
    from .device import conv2d
    n = np.asarray(weights).shape[1]
    if slab.ghost < conv2d_halo(n):
        raise ValueError(f"conv2d with {n} filter rows needs ghost >= {conv2d_halo(n)}")
    own_lo = slab.local(slab.z_first)
    conv2d(d_in, d_out, weights, boundary, own_lo, own_lo + slab.nz_own, stream=stream)
