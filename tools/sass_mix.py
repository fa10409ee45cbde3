"""Executed-instruction mix from an ncu source page (--page source --csv --print-source sass)."""
import csv, sys, collections, re

def mix(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    si, ei = hdr.index("Source"), hdr.index("Instructions Executed")
    c = collections.Counter()
    tot = 0
    for r in rows[2:]:
        if len(r) <= ei:
            continue
        try:
            n = int(r[ei])
        except ValueError:
            continue
        op = r[si].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", op).split()[0] if op else "?"
        c[op] += n
        tot += n
    print(f"{path}: {tot/1e6:.1f}M warp-instructions")
    for op, n in c.most_common(top):
        print(f"  {op:18s} {n/1e6:9.2f}M  {100*n/tot:5.1f}%")

if __name__ == "__main__":
    for p in sys.argv[1:]:
        mix(p)
