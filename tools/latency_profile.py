"""Measure the B200 LatencyProfile (perf_model.hpp:14-26) and write it in the
reference's profile-file format (perf_model.cpp:41-87).

    python tools/latency_profile.py [out.profile] [out.json]

Five runs of ssam_b200_measure_latency (csrc/latency.cu), median per field,
rounded to whole cycles.  The file loads with the reference's own
resolve_profile (SSAM_PROFILE_DIR=<dir> ... --profile B200), so its perf
model (latency_reg / latency_smem / compare_plans) can rank dataflows with
B200 numbers next to its built-in P100 and V100 profiles."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import paper_1907_06154_b200 as ssam

out_profile = sys.argv[1] if len(sys.argv) > 1 else "profiles/B200.profile"
out_json = sys.argv[2] if len(sys.argv) > 2 else "profiles/r02/latency_profile.json"
runs = [ssam.measure_latency_profile() for _ in range(5)]
med = {k: statistics.median(r[k] for r in runs) for k in runs[0]}
text = ssam.format_profile("B200", med)
with open(out_profile, "w") as fh:
    fh.write(text)
rec = {"median": med, "runs": runs, "profile_file": text,
       "method": "csrc/latency.cu: one warp, clock64 around 16384 chained ops "
                 "(fma.rn.f32; shfl.sync.idx; ld.shared pointer chase); global reads: "
                 "ld.global.cg chase of coalesced 128-byte lines, random over 256 MiB (HBM) "
                 "and 16 MiB (L2); writes: st.global.wt + fence.acq_rel.gpu per step"}
try:
    from oracle import Reference
    ref = Reference()
    cmp = {}
    for prof in ("P100", "V100", os.path.abspath(out_profile)):
        rc, name, vals, _ = ref.profile(prof)
        cmp[name or prof] = {"status": rc, "fields": vals.tolist(),
                             "latency_reg_smem": {f"{k}x{k}": ref.profile(prof, k, k)[3].tolist()
                                                  for k in (3, 5, 7, 11, 20)}}
    rec["reference_model"] = cmp
except Exception as exc:  # the checker library is optional on the box
    rec["reference_model"] = f"unavailable: {exc}"
os.makedirs(os.path.dirname(out_json), exist_ok=True)
with open(out_json, "w") as fh:
    json.dump(rec, fh, indent=1)
print(text, end="")
print(json.dumps(med))
