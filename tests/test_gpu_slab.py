"""Multi-rank z-slab runs with the CUDA kernels (-m gpu, one B200).

tools/slab_check.py under torchrun: 2 and 3 ranks share the GPU
(SSAM_BENCH_BACKEND=gloo stages the halos through host memory), run 6 sweeps
with the product sweep kernel (Tb = 1) and the fused Tb = 2 kernel, and must
equal the one-GPU result bit for bit.  The NCCL transport itself needs
several GPUs; everything around it (decomposition, boundary-first ordering,
ghost planes, global ring in local coordinates, fused pairs) runs here.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world", [2, 3])
def test_slab_ranks_match_one_gpu(cuda_lib, world):
    env = dict(os.environ, SSAM_BENCH_BACKEND="gloo")
    port = str(29600 + world)
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
                        "--master-port", port, "tools/slab_check.py"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert "SLAB CHECK PASS" in p.stdout, p.stdout[-2000:] + p.stderr[-2000:]


@pytest.mark.parametrize("world", [2, 3])
def test_peer_halo_slabs_match_one_gpu(cuda_lib, world):
    """Peer-memory halo (peer.PeerSlabRunner): the sweep kernel stores the
    neighbours' ghost planes itself over CUDA IPC; 2 and 3 ranks share the GPU.
    fp32/fp64/int64, Tb 1 and 2, the halo-lane, aligned, dense-K2 and direct
    (order 3, pushed planes) kernels."""
    port = str(29650 + world)
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
                        "--master-port", port, "tools/peer_slab_check.py"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert "PEER SLAB CHECK PASS" in p.stdout, p.stdout[-2000:] + p.stderr[-2000:]


@pytest.mark.parametrize("world", [2, 3])
def test_row_slabs_2d_match_one_gpu(cuda_lib, world):
    """2D row slabs (y for 2D): stencil2d sweeps through SlabRunner
    and conv2d with read-only halo rows (zero and replicate boundaries), f32 /
    f64 / int64, equal to the one-GPU result bit for bit."""
    env = dict(os.environ, SSAM_BENCH_BACKEND="gloo")
    port = str(29700 + world)
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
                        "--master-port", port, "tools/slab2d_check.py"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert "SLAB2D CHECK PASS" in p.stdout, p.stdout[-2000:] + p.stderr[-2000:]
