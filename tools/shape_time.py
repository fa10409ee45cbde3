"""3D single sweeps at 512^3 of the named shapes (GCells/s): python tools/shape_time.py 3d13pt ..."""
import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import numpy as np, torch
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
from pipe_check import timed
out = []
for npdt, tdt in ((np.float32, torch.float32), (np.float64, torch.float64)):
    a = torch.empty((512, 512, 512), dtype=tdt, device="cuda"); dev.fill_random(a, 0); b = a.clone()
    for name in sys.argv[1:]:
        st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), npdt)
        k = st.order
        ms = timed(lambda: dev.stencil3d_sweep(a, b, st), 10)
        out.append(f"{name}/{np.dtype(npdt).name}={(512 - 2 * k) ** 3 / ms / 1e6:.0f}")
print(os.environ.get("SSAM_B200_LIB"), " ".join(out), flush=True)
