"""Per-launch (duration, grid, block) from an ncu --csv launch list with
gpu__time_duration.sum,launch__grid_size,launch__block_size; summary by kernel
and the launches of one kernel (substring filter) in order."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ii, ki, mi, vi, ui = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
L = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = L.setdefault(r[ii], {"name": r[ki].split("(")[0].replace("void ", "")})
    v = float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        d["us"] = v
    elif r[mi] == "launch__grid_size":
        d["grid"] = int(v)
    elif r[mi] == "launch__block_size":
        d["block"] = int(v)
agg = collections.defaultdict(lambda: [0, 0.0])
for d in L.values():
    a = agg[d["name"]]; a[0] += 1; a[1] += d.get("us", 0.0)
tot = sum(a[1] for a in agg.values())
for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{k[:50]:50s} {n:5d} {v/1e3:8.3f} ms {100*v/tot:5.1f}%")
print(f"total {tot/1e3:.3f} ms over {len(L)} launches")
for pat in sys.argv[2:]:
    print("--", pat)
    for d in L.values():
        if pat in d["name"]:
            print(f"   {d['name'][:40]:40s} {d.get('us',0):9.1f} us grid {d.get('grid')} block {d.get('block')}")
