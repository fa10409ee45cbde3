"""A/B the 3D engines (each env config in its own process; knobs are read once).
Prints GCells/s per (stencil, dtype, shape) and whether the output is
bit-identical to the first config's.
  python tools/st3d_ab.py "SSAM_B200_3D_HALO=0" "SSAM_B200_3D_HALO=1" """
import json, os, subprocess, sys

CHILD = r'''
import sys, os, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1907_06154_b200 as ssam
from paper_1907_06154_b200 import device as dev
out = {}
for spec in sys.argv[1].split(","):
    name, dt, shape = spec.split(":")
    dims = [int(v) for v in shape.split("x")]
    tdt, npdt = (torch.float32, np.float32) if dt == "f32" else (torch.float64, np.float64)
    a = torch.empty(tuple(dims[::-1]), dtype=tdt, device="cuda"); dev.fill_random(a, 0)
    b = a.clone()
    st = ssam.convert_stencil(ssam.make_benchmark_stencil(name), npdt)
    sweep = dev.stencil3d_sweep if len(dims) == 3 else dev.stencil2d_sweep
    for _ in range(2): sweep(a, b, st)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(7):
        s.record(); sweep(a, b, st); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    iv = b.view(torch.int32) if dt == "f32" else b.view(torch.int64)
    ck = int(iv.to(torch.int64).sum().item()) & ((1 << 62) - 1)
    out[spec] = (int(np.prod(dims)) / best / 1e6, ck)
    del a, b
    torch.cuda.empty_cache()
print("RESULT " + json.dumps(out))
'''

DEFAULT = ",".join([f"{n}:{d}:512x512x512" for d in ("f32", "f64")
                    for n in ("3d7pt", "3d13pt", "3d27pt", "poisson")] +
                   ["3d7pt:f32:2048x2048x514"])

def run(env_s, specs):
    env = dict(os.environ)
    for kv in env_s.split():
        k, v = kv.split("=")
        env[k] = v
    try:
        r = subprocess.run([sys.executable, "-c", CHILD, specs], env=env, capture_output=True,
                           text=True, timeout=int(os.environ.get("AB_TIMEOUT", "200")))
    except subprocess.TimeoutExpired:
        print("TIMEOUT", env_s)
        return {}
    for line in r.stdout.splitlines():
        if line.startswith("RESULT "):
            return json.loads(line[7:])
    print(r.stdout[-2000:], r.stderr[-3000:])
    return {}

if __name__ == "__main__":
    specs = os.environ.get("SPECS", DEFAULT)
    cfgs = sys.argv[1:] or ["SSAM_B200_3D_HALO=0", "SSAM_B200_3D_HALO=1"]
    res = [run(c, specs) for c in cfgs]
    print(f"{'case':28s}" + "".join(f"{c[-26:]:>28s}" for c in cfgs))
    for sp in specs.split(","):
        row = f"{sp:28s}"
        for r in res:
            if sp in r:
                same = "=" if r[sp][1] == res[0].get(sp, (0, None))[1] else "X"
                row += f"{r[sp][0]:>26.1f} {same}"
            else:
                row += f"{'-':>28s}"
        print(row)
