"""2D row slabs on CPU (gloo, world 2 and 3; "y for 2D").

stencil2d: the SlabRunner's decomposition and neighbour exchange with the
oracle as the per-slab sweep, equal to the single-grid oracle bit for bit.
conv2d: each rank convolves its rows from owned + halo rows of the read-only
input (zero and replicate boundaries) -- no exchange -- equal to the
single-grid oracle.  The GPU twin is tests/test_gpu_slab.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

SHAPE = (29, 37)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _local_rows(full, slab):
    y0 = slab.z_first - slab.ghost
    local = np.zeros((slab.nz_local, full.shape[1]), full.dtype)
    for p in range(slab.nz_local):
        if 0 <= y0 + p < full.shape[0]:
            local[p] = full[y0 + p]
    return local


def _worker(rank, world, port, kind, arg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import Oracle
        from paper_1907_06154_b200.slab import (SlabRunner, conv2d_halo, decompose,
                                                replicate_outside)
        import paper_1907_06154_b200 as ssam

        orc = Oracle()
        full = orc.random_grid(SHAPE, np.float64, 5)
        if kind == "stencil":
            name, iters, tb = arg
            st = ssam.make_benchmark_stencil(name)
            offs = [t.offset for t in st.taps]
            cf = np.asarray([t.coeff for t in st.taps])
            k = st.order
            slab = decompose(SHAPE[0], world, rank, k, ghost=k * tb)
            a = torch.from_numpy(_local_rows(full, slab))
            b = a.clone()

            def sweep(cur, nxt, yb, ye):
                if ye <= yb:
                    return
                out = orc.stencil2d(cur[yb - k:ye + k].numpy(), offs, cf, k, 1)
                nxt[yb:ye] = torch.from_numpy(out[k:k + (ye - yb)])

            def fused(cur, nxt, yb, ye):
                # tb sweeps; sweep j writes [yb - k*(tb-1-j), ye + k*(tb-1-j)) of the global
                # interior -- what the fused row-range kernel computes on the GPU
                rlo, rhi = slab.ring_bounds()
                src = cur
                for j in range(tb):
                    w = k * (tb - 1 - j)
                    dst = nxt if j == tb - 1 else src.clone()
                    sweep(src, dst, max(yb - w, rlo), min(ye + w, rhi))
                    src = dst

            res = SlabRunner(slab, sweep, fused=fused if tb > 1 else None, tb=tb).run(a, b, iters)
        else:
            K, bnd = arg
            w = orc.random_filter(K, K, np.float64, K)
            slab = decompose(SHAPE[0], world, rank, 0, ghost=conv2d_halo(K))
            a = torch.from_numpy(_local_rows(full, slab))
            if bnd == 1:
                replicate_outside(a, slab)
            res = torch.from_numpy(orc.conv2d(a.numpy(), w, bnd))  # the per-slab conv
        own = res[slab.ghost:slab.ghost + slab.nz_own].numpy()
        q.put((rank, slab.z_first, own))
    finally:
        dist.destroy_process_group()


def _run(world, kind, arg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, arg, q))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.zeros(SHAPE)
    for _, y0, own in parts:
        got[y0:y0 + own.shape[0]] = own
    return got


@pytest.mark.parametrize("world,name,tb", [(2, "2d5pt", 1), (3, "2d9pt", 1), (2, "2ds25pt", 1),
                                           (2, "2d5pt", 4), (3, "2d9pt", 2)])
def test_stencil2d_row_slabs(world, name, tb):
    from oracle import Oracle
    import paper_1907_06154_b200 as ssam
    orc = Oracle()
    st = ssam.make_benchmark_stencil(name)
    iters = 2 * tb + 1 if tb > 1 else 3
    want = orc.stencil2d(orc.random_grid(SHAPE, np.float64, 5), [t.offset for t in st.taps],
                         np.asarray([t.coeff for t in st.taps]), st.order, iters)
    assert np.array_equal(_run(world, "stencil", (name, iters, tb)), want)


@pytest.mark.parametrize("world,K,bnd", [(2, 3, 0), (3, 7, 1), (2, 6, 1), (3, 9, 0)])
def test_conv2d_row_slabs(world, K, bnd):
    from oracle import Oracle
    orc = Oracle()
    w = orc.random_filter(K, K, np.float64, K)
    want = orc.conv2d(orc.random_grid(SHAPE, np.float64, 5), w, bnd)
    assert np.array_equal(_run(world, "conv", (K, bnd)), want)
