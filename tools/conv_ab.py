"""A/B the conv2d engines over K (each config in its own process: the knobs are
read once).  Prints GCells/s per K and whether the output is bit-identical to
the first config's.   python tools/conv_ab.py "SSAM_B200_CONV_FMA=0" "SSAM_B200_CONV_FMA=3" ..."""
import json, os, subprocess, sys

CHILD = r'''
import sys, os, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1907_06154_b200 import device as dev
H = W = 8192
g = torch.empty((H, W), dtype=torch.float32, device="cuda"); dev.fill_random(g, 0)
o = torch.empty_like(g)
out = {}
for K in [int(k) for k in sys.argv[1].split(",")]:
    f = np.random.default_rng(K).uniform(-1, 1, (K, K)).astype(np.float32)
    for _ in range(2): dev.conv2d(g, o, f)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(7):
        s.record(); dev.conv2d(g, o, f); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    ck = int(o.view(torch.int32).to(torch.int64).mul(torch.arange(1, 8193, device="cuda").view(1, -1)).sum().item())
    out[K] = (H * W / best / 1e6, ck)
print("RESULT " + json.dumps(out))
'''

def run(env_s, ks):
    env = dict(os.environ)
    for kv in env_s.split():
        k, v = kv.split("=")
        env[k] = v
    r = subprocess.run([sys.executable, "-c", CHILD, ks], env=env, capture_output=True, text=True, timeout=int(os.environ.get("AB_TIMEOUT", "150")))
    for line in r.stdout.splitlines():
        if line.startswith("RESULT "):
            return {int(k): v for k, v in json.loads(line[7:]).items()}
    print(r.stdout[-2000:], r.stderr[-3000:])
    return {}

if __name__ == "__main__":
    ks = os.environ.get("KS", ",".join(str(k) for k in range(3, 21)))
    cfgs = sys.argv[1:] or ["SSAM_B200_CONV_FMA=0", "SSAM_B200_CONV_FMA=3"]
    res = [run(c, ks) for c in cfgs]
    print("K    " + "".join(f"{c[-28:]:>30s}" for c in cfgs))
    for K in [int(k) for k in ks.split(",")]:
        row = f"{K:<5d}"
        for r in res:
            if K in r:
                same = "=" if r[K][1] == res[0].get(K, (0, None))[1] else "X"
                row += f"{r[K][0]:>28.1f} {same}"
            else:
                row += f"{'-':>30s}"
        print(row)
