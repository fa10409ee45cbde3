"""N-rank 2D row-slab runs with the CUDA kernels vs one GPU, bit for bit.
Launch with torchrun; SSAM_BENCH_BACKEND=gloo lets the ranks share one GPU
(halos staged through host memory).  stencil2d sweeps (SlabRunner, rows are
the planes) and conv2d (no exchange, halo rows of the read-only input)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, torch.distributed as dist
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
from paper_1907_06154_b200.slab import (SlabRunner, conv2d_halo, conv2d_slab, decompose,
                                        fill_slab, replicate_outside)

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
dist.init_process_group(os.environ.get("SSAM_BENCH_BACKEND", "nccl"))
H, W = 203, 264
TD = {np.float32: torch.float32, np.float64: torch.float64, np.int64: torch.int64}
ok = True


def gather_rows(slab, res):
    own = res[slab.ghost:slab.ghost + slab.nz_own].cpu().numpy()
    parts = [None] * world
    dist.all_gather_object(parts, (slab.z_first, own))
    return parts


def report(tag, parts, want):
    global ok
    got = np.zeros_like(want)
    for y0, o in parts:
        got[y0:y0 + o.shape[0]] = o
    same = np.array_equal(got, want)
    ok &= same
    print(f"{tag} world={world}: identical to one GPU: {same}", flush=True)


for name, dt, iters in (("2d5pt", np.float32, 5), ("2d9pt", np.float64, 4),
                        ("2ds25pt", np.float32, 3), ("2d121pt", np.float32, 2),
                        ("2d5pt", np.int64, 3)):
    st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), dt)
    slab = decompose(H, world, rank, st.order)
    a = torch.empty((slab.nz_local, W), dtype=TD[dt], device="cuda")
    fill_slab(a, slab, W, 1, seed=7)
    b = a.clone()
    runner = SlabRunner(slab, lambda c, n, yb, ye: dev.stencil2d_sweep(c, n, st, yb, ye),
                        comm_stream=torch.cuda.Stream())
    parts = gather_rows(slab, runner.run(a, b, iters))
    if rank == 0:
        cur = torch.empty((H, W), dtype=TD[dt], device="cuda")
        dev.fill_random(cur, 7)
        nxt = cur.clone()
        for _ in range(iters):
            dev.stencil2d_sweep(cur, nxt, st)
            cur, nxt = nxt, cur
        report(f"stencil2d {name} {np.dtype(dt).name} x{iters}", parts, cur.cpu().numpy())

# fused 2D sweeps on row slabs (ghost = k*Tb, exchange once per Tb sweeps): vs the one-GPU
# sequence of whole-grid fused launches plus the single-sweep remainder
for name, dt in (("2d5pt", np.float32), ("2d9pt", np.float32), ("2d5pt", np.float64)):
    st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), dt)
    tb = dev.stencil2d_tb_max(st, dt)
    iters = 2 * tb + 1
    slab = decompose(H, world, rank, st.order, ghost=st.order * tb)
    a = torch.empty((slab.nz_local, W), dtype=TD[dt], device="cuda")
    fill_slab(a, slab, W, 1, seed=9)
    b = a.clone()
    rlo, rhi = slab.ring_bounds()
    runner = SlabRunner(slab, lambda c, n, yb, ye: dev.stencil2d_sweep(c, n, st, yb, ye),
                        comm_stream=torch.cuda.Stream(),
                        fused=lambda c, n, yb, ye: dev.stencil2d_tb(c, n, st, tb, yb, ye, rlo, rhi),
                        tb=tb)
    parts = gather_rows(slab, runner.run(a, b, iters))
    if rank == 0:
        cur = torch.empty((H, W), dtype=TD[dt], device="cuda")
        dev.fill_random(cur, 9)
        nxt = cur.clone()
        for j in range(iters // tb):
            dev.stencil2d_tb(cur, nxt, st, tb)
            cur, nxt = nxt, cur
        for j in range(iters % tb):
            dev.stencil2d_sweep(cur, nxt, st)
            cur, nxt = nxt, cur
        report(f"stencil2d {name} {np.dtype(dt).name} Tb={tb} x{iters}", parts, cur.cpu().numpy())

for K, bnd, dt in ((3, 0, np.float32), (7, 1, np.float32), (20, 0, np.float32),
                   (5, 1, np.float64), (4, 0, np.int64)):
    w = np.random.default_rng(K).uniform(-1, 1, (K, K)).astype(dt) if dt != np.int64 else \
        np.random.default_rng(K).integers(-5, 6, (K, K)).astype(dt)
    slab = decompose(H, world, rank, 0, ghost=conv2d_halo(K))
    a = torch.empty((slab.nz_local, W), dtype=TD[dt], device="cuda")
    fill_slab(a, slab, W, 1, seed=11)
    if bnd == 1:
        replicate_outside(a, slab)
    o = torch.zeros_like(a)
    conv2d_slab(a, o, w, slab, bnd)
    parts = gather_rows(slab, o)
    if rank == 0:
        full = torch.empty((H, W), dtype=TD[dt], device="cuda")
        dev.fill_random(full, 11)
        out = torch.empty_like(full)
        dev.conv2d(full, out, w, bnd)
        report(f"conv2d {K}x{K} boundary={bnd} {np.dtype(dt).name}", parts, out.cpu().numpy())
dist.destroy_process_group()
if rank == 0:
    print("SLAB2D CHECK", "PASS" if ok else "FAIL")
