"""Multi-rank z-slab decomposition + halo exchange on CPU (gloo, world 2 and 3).

The SlabRunner drives the same decomposition, boundary-first ordering and
neighbour exchange it uses on B200s with NCCL; here the per-slab sweep is the
oracle (test infrastructure) so the result must equal the single-grid oracle
bit-for-bit.  A 1-GPU box cannot exercise NCCL across devices; this covers the
N > 1 host logic.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, shape, name, iters, q, tb=1):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        from oracle import Oracle
        from paper_1907_06154_b200.slab import SlabRunner, decompose
        import paper_1907_06154_b200 as ssam

        orc = Oracle()
        st = ssam.make_benchmark_stencil(name)
        offs = [t.offset for t in st.taps]
        cf = np.asarray([t.coeff for t in st.taps])
        nz, ny, nx = shape
        k = st.order
        slab = decompose(nz, world, rank, k, ghost=k * tb)
        full = orc.random_grid(shape, np.float64, 21)
        z0 = slab.z_first - slab.ghost
        local = np.zeros((slab.nz_local, ny, nx))
        for p in range(slab.nz_local):
            if 0 <= z0 + p < nz:
                local[p] = full[z0 + p]
        a = torch.from_numpy(local.copy())
        b = torch.from_numpy(local.copy())

        def sweep(cur, nxt, zb, ze):
            if ze <= zb:
                return
            sub = cur[zb - k:ze + k].numpy()
            out = orc.stencil3d(sub, offs, cf, k, 1)
            nxt[zb:ze] = torch.from_numpy(out[k:k + (ze - zb)])

        def fused(cur, nxt, zb, ze):
            # tb sweeps; sweep j writes [zb - k*(tb-1-j), ze + k*(tb-1-j)) of the
            # global interior -- what the fused kernel computes on the GPU
            rlo, rhi = slab.ring_bounds()
            src = cur
            for j in range(tb):
                w = k * (tb - 1 - j)
                dst = nxt if j == tb - 1 else src.clone()
                sweep(src, dst, max(zb - w, rlo), min(ze + w, rhi))
                src = dst

        res = SlabRunner(slab, sweep, fused=fused if tb > 1 else None, tb=tb).run(a, b, iters)
        own = res[slab.ghost:slab.ghost + slab.nz_own].numpy()
        q.put((rank, slab.z_first, own))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,name,tb", [(2, "3d7pt", 1), (3, "3d13pt", 1), (2, "3d27pt", 1),
                                           (2, "3d7pt", 2), (3, "poisson", 2)])
def test_slab_matches_global_oracle(world, name, tb):
    from oracle import Oracle
    import paper_1907_06154_b200 as ssam
    shape = (23, 11, 13)
    iters = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, name, iters, q, tb))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    orc = Oracle()
    st = ssam.make_benchmark_stencil(name)
    want = orc.stencil3d(orc.random_grid(shape, np.float64, 21), [t.offset for t in st.taps],
                         np.asarray([t.coeff for t in st.taps]), st.order, iters)
    got = np.zeros(shape)
    for _, z_first, own in parts:
        got[z_first:z_first + own.shape[0]] = own
    assert np.array_equal(got, want)


def test_decompose_covers_exactly_once():
    from paper_1907_06154_b200.slab import decompose
    for nz in (16, 23, 512 * 8 + 3):
        for world in (1, 2, 3, 8):
            for k in (1, 2):
                owned = []
                for r in range(world):
                    s = decompose(nz, world, r, k)
                    owned.extend(range(s.z_first, s.z_first + s.nz_own))
                    lo, hi = s.compute_range()
                    for p in range(lo, hi):
                        z = s.z_first - s.ghost + p
                        assert k <= z < nz - k
                assert owned == list(range(nz))
