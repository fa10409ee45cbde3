"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import csv, sys, collections

def share(path):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr = rows[0]
    ki, vi = hdr.index('Kernel Name'), hdr.index('Metric Value')
    tot = collections.defaultdict(float); n = collections.Counter()
    for r in rows[1:]:
        v = float(r[vi].replace(',', '')) / 1000.0
        tot[r[ki]] += v; n[r[ki]] += 1
    s = sum(tot.values())
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{100*v/s:6.2f}%  n={n[k]:4d} mean={v/n[k]:10.1f}us  {k[:100]}")

if __name__ == '__main__':
    share(sys.argv[1])
