"""Per-family DRAM traffic of one factorization from an ncu CSV capture
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum).
Writes a JSON {family: {launches, dram_bytes, dram_bytes_per_launch, ms}} that
bench.py reads to fill roofline.traffic.
  python scripts/ncu_traffic.py capture.csv out.json"""
import collections
import csv
import json
import sys

FAMILY = [("k_assemble", "assemble"), ("k_geqr", "geqrf"), ("k_larft", "geqrf"), ("k_zero_lower", "geqrf"),
          ("k_qrcp", "qrcp"), ("k_gather_R", "id_T"), ("k_gemm", "gemm"), ("k_getrf", "getrf"),
          ("k_getf2", "getrf"), ("k_laswp", "getrf"), ("k_pivot", "getrf"), ("k_trsm", "trsm"), ("k_apply_ipiv", "trsm"),
          ("k_gather", "move"), ("k_scatter", "move"), ("k_copy2d", "move"), ("k_schur", "move")]
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ui, idi = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                       h.index("Metric Unit"), h.index("ID"))
per = collections.defaultdict(dict)
names = {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    if r[mi].startswith("dram__bytes"):
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    else:
        v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(u, 1)
    per[r[idi]][r[mi]] = v
    names[r[idi]] = r[ki].split("(")[0].replace("void ", "")
fam = collections.defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0, "ms": 0.0, "kernels": collections.Counter()})
for i, m in per.items():
    nm = names[i]
    f = next((fa for pre, fa in FAMILY if pre in nm), None)
    if f is None:
        continue
    d = fam[f]
    d["launches"] += 1
    d["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    d["ms"] += m.get("gpu__time_duration.sum", 0.0)
    d["kernels"][nm.split("::")[-1].split("<")[0]] += 1
out = {f: {"launches": d["launches"], "dram_bytes": d["dram_bytes"],
           "dram_bytes_per_launch": d["dram_bytes"] / max(d["launches"], 1), "ms_serialised": d["ms"],
           "kernels": dict(d["kernels"])} for f, d in fam.items()}
json.dump({"source": sys.argv[1], "note": "one warm cfg2 factorization under ncu (cold caches, serialised)",
           "families": out}, open(sys.argv[2], "w"), indent=1)
for f, d in sorted(out.items(), key=lambda kv: -kv[1]["dram_bytes"]):
    print(f"{f:10s} launches {d['launches']:4d}  DRAM {d['dram_bytes']/1e6:9.2f} MB  per launch {d['dram_bytes_per_launch']/1e6:8.3f} MB  {d['ms_serialised']:7.3f} ms")
