"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
mi = h.index("Metric Name") if "Metric Name" in h else None
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
tot = 0.0
seq = []
for r in rows[hi + 1:]:
    if len(r) <= vi or (mi is not None and r[mi] != "gpu__time_duration.sum"):
        continue
    v = float(r[vi].replace(",", ""))
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
    name = r[ki].split("(")[0].replace("void ", "")
    a = agg[name]
    a[0] += 1; a[1] += v; a[2] = max(a[2], v)
    tot += v
    seq.append((name, v))
print(f"{'kernel':48s} {'n':>5s} {'total ms':>9s} {'share':>6s} {'max us':>8s}")
for k, (n, v, mx) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:48]:48s} {n:5d} {v/1e3:9.3f} {100*v/tot:5.1f}% {mx:8.1f}")
print(f"total {tot/1e3:.3f} ms over {len(seq)} launches")
if len(sys.argv) > 2:
    for name, v in sorted(seq, key=lambda x: -x[1])[: int(sys.argv[2])]:
        print(f"  {name[:48]:48s} {v:9.1f} us")
