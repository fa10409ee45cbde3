"""N-rank z-slab run with the CUDA sweep kernels vs one-GPU sweeps (bit-exact).
Launch with torchrun; SSAM_BENCH_BACKEND=gloo lets the ranks share one GPU
(halos staged through host memory).  Checks Tb = 1 and Tb = 2."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, torch.distributed as dist
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
from paper_1907_06154_b200.slab import SlabRunner, decompose, fill_slab

backend = os.environ.get("SSAM_BENCH_BACKEND", "nccl")
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
dist.init_process_group(backend)
nx, ny, nzg, iters = 264, 200, 61, 6
ok = True
for name in ("3d7pt", "poisson"):
    st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), np.float32)
    for tb in (1, 2):
        if tb == 2 and name != "3d7pt":
            continue
        slab = decompose(nzg, world, rank, st.order, ghost=st.order * tb)
        a = torch.empty((slab.nz_local, ny, nx), dtype=torch.float32, device="cuda")
        fill_slab(a, slab, nx, ny, seed=3)
        b = a.clone()
        rlo, rhi = slab.ring_bounds()
        runner = SlabRunner(
            slab, lambda c, n, zb, ze: dev.stencil3d_sweep(c, n, st, zb, ze),
            comm_stream=torch.cuda.Stream(),
            fused=(lambda c, n, zb, ze: dev.stencil3d_tb(c, n, st, 2, zb, ze, rlo, rhi)) if tb > 1 else None,
            tb=tb)
        res = runner.run(a, b, iters)
        own = res[slab.ghost:slab.ghost + slab.nz_own].cpu()
        parts = [None] * world
        dist.all_gather_object(parts, (slab.z_first, own.numpy()))
        if rank == 0:
            full = torch.empty((nzg, ny, nx), dtype=torch.float32, device="cuda")
            dev.fill_random(full, 3)
            ref = full.clone()
            out = dev.stencil3d_run(full, ref, st, iters)  # one GPU (fuses pairs for 3d7pt fp32)
            want = out.cpu().numpy()
            got = np.zeros_like(want)
            for z0, o in parts:
                got[z0:z0 + o.shape[0]] = o
            same = np.array_equal(got, want)
            ok &= same
            print(f"{name} tb={tb} world={world}: identical to one GPU: {same}", flush=True)
dist.destroy_process_group()
if rank == 0:
    print("SLAB CHECK", "PASS" if ok else "FAIL")
