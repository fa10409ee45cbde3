"""Peer-memory halo geometry (peer.peer_geometry) on CPU: the planes a rank's
kernel mirrors land in exactly its neighbours' ghost slots, at the same global
plane -- simulated with numpy over every decomposition of small grids."""
import numpy as np
import pytest

from paper_1907_06154_b200.peer import peer_geometry
from paper_1907_06154_b200.slab import decompose


@pytest.mark.parametrize("nzg,world,order,tb", [(20, 2, 1, 1), (23, 3, 1, 2), (31, 4, 2, 1),
                                                (9, 3, 1, 2), (40, 5, 2, 2)])
def test_mirrored_planes_fill_neighbour_ghosts(nzg, world, order, tb):
    plane = 6  # elements per plane (any)
    slabs = [decompose(nzg, world, r, order, ghost=order * tb) for r in range(world)]
    # every rank writes the global plane number into all of its owned planes ...
    bufs = [np.full((s.nz_local, plane), -1, np.int64) for s in slabs]
    for r, s in enumerate(slabs):
        below = slabs[r - 1].nz_own if r > 0 else 0
        lo_shift, lo_end, hi_shift, hi_begin = peer_geometry(s, below, plane)
        own_lo = s.local(s.z_first)
        for z in range(own_lo, own_lo + s.nz_own):
            g = s.z_first - s.ghost + z
            bufs[r][z] = g
            flat = z * plane
            # ... and mirrors the planes its neighbours keep as ghosts
            if r > 0 and z < lo_end:
                bufs[r - 1].reshape(-1)[flat + lo_shift:flat + lo_shift + plane] = g
            if r < world - 1 and z >= hi_begin:
                bufs[r + 1].reshape(-1)[flat + hi_shift:flat + hi_shift + plane] = g
    for r, s in enumerate(slabs):
        for z in range(s.nz_local):
            g = s.z_first - s.ghost + z
            if 0 <= g < nzg:
                assert (bufs[r][z] == g).all(), (r, z, g)  # ghosts hold the right global plane
            else:
                assert (bufs[r][z] == -1).all()             # outside the grid: untouched
