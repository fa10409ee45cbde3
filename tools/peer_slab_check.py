"""N-rank z-slab runs with the peer-memory halo (peer.PeerSlabRunner) vs one-GPU
sweeps, bit for bit.  Launch with torchrun (gloo process group); ranks may
share one GPU (CUDA IPC within a device) or own one each (NVLink P2P)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, torch.distributed as dist
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
from paper_1907_06154_b200.peer import PeerSlabRunner
from paper_1907_06154_b200.slab import decompose, fill_slab

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
dist.init_process_group("gloo")
nx, ny, nzg = 264, 136, 47
TD = {np.float32: torch.float32, np.float64: torch.float64, np.int64: torch.int64}


def star3(k):
    taps = [ssam.StencilTap((0, 0, 0), 0.25)]
    for i in range(1, k + 1):
        for ax in range(3):
            for sgn in (-1, 1):
                o = [0, 0, 0]
                o[ax] = sgn * i
                taps.append(ssam.StencilTap(tuple(o), 0.125 / (i * 3)))
    return ssam.Stencil(f"star{k}", 3, k, 0, taps)


cases = [("3d7pt", np.float32, 1, 5), ("3d7pt", np.float32, 2, 7), ("3d7pt", np.float64, 2, 4),
         ("poisson", np.float32, 1, 5), ("3d27pt", np.float64, 1, 3), ("3d13pt", np.float32, 1, 4),
         ("3d125pt", np.float32, 1, 3), ("3d7pt", np.int64, 1, 4), ("star3", np.float32, 1, 3)]
ok = True
for name, dt, tb, iters in cases:
    base = star3(3) if name == "star3" else ssam.make_benchmark_stencil(name)
    st = ssam.convert_stencil(base, dt)
    slab = decompose(nzg, world, rank, st.order, ghost=st.order * tb)
    run = PeerSlabRunner(slab, st, nx, ny, TD[dt], tb=tb)
    fill_slab(run.a, slab, nx, ny, seed=5)
    run.b.copy_(run.a)
    res = run.run(iters)
    own = res[slab.ghost:slab.ghost + slab.nz_own].cpu().numpy()
    run.close()
    parts = [None] * world
    dist.all_gather_object(parts, (slab.z_first, own))
    if rank == 0:
        full = torch.empty((nzg, ny, nx), dtype=TD[dt], device="cuda")
        dev.fill_random(full, 5)
        cur, nxt = full, full.clone()
        for _ in range(iters):
            dev.stencil3d_sweep(cur, nxt, st)
            cur, nxt = nxt, cur
        want = cur.cpu().numpy()
        got = np.zeros_like(want)
        for z0, o in parts:
            got[z0:z0 + o.shape[0]] = o
        # interior owned planes; the global ring is identical by construction
        same = np.array_equal(got[st.order:nzg - st.order], want[st.order:nzg - st.order])
        ok &= same
        print(f"{name} {np.dtype(dt).name} tb={tb} iters={iters} world={world}: "
              f"identical to one GPU: {same}", flush=True)
dist.destroy_process_group()
if rank == 0:
    print("PEER SLAB CHECK", "PASS" if ok else "FAIL")
