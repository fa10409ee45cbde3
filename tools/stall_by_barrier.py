"""Warp-stall samples of an ncu source page (--page source --csv --print-source
sass): the share at the branch after each mbarrier try_wait, per barrier
address, and the share per 4 KiB code region.  python tools/stall_by_barrier.py f.csv"""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    si, st, ad = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Address")
    tot, prev = 0, None
    bars, region = collections.Counter(), collections.Counter()
    for r in rows[2:]:
        if len(r) <= st:
            continue
        try:
            s = int(r[st])
        except ValueError:
            continue
        tot += s
        region[int(r[ad], 16) >> 12] += s
        src = r[si]
        if "TRYWAIT" in src:
            prev = src.split("[")[1].split("]")[0]
        elif "BRA" in src and prev:
            bars[prev] += s
            prev = None
        else:
            prev = None
    print(path)
    for b, s in bars.most_common(12):
        print(f"  wait {b:26s} {100 * s / tot:5.1f}%")
    base = min(region)
    print("  code regions (4 KiB from kernel start):",
          " ".join(f"{k - base}:{100 * v / tot:.0f}%" for k, v in sorted(region.items()) if v > tot * 0.01))
