"""Kernel timeline of one warm factorization (torch.profiler / CUPTI).

Prints the GPU-busy union, idle gaps and per-kernel start/end relative to the
factor() call, so the critical path (host bookkeeping vs. kernels) is visible.
  python scripts/timeline.py [cfg2] [factor|update] [out.json]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SKB_HOST_PROF", "trace")
import torch
from torch.profiler import ProfilerActivity, profile, record_function

from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
mode = sys.argv[2] if len(sys.argv) > 2 else "factor"
out = sys.argv[3] if len(sys.argv) > 3 else f"gpurun_out/timeline_{name}_{mode}.json"
wl = configs.by_name(name)
b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
fa = lambda: factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
for _ in range(3):
    f = fa()
if mode == "solve":
    import numpy as np
    X = torch.from_numpy(np.random.default_rng(5).standard_normal((f.dim, 256))).cuda()
    f.solve(X)
    f.solve(X)
    run = lambda: f.solve(X)
elif mode == "update":
    seq = configs.hole_move_sequence(b, 3)
    f = update(f, seq[0][2], seq[0][3])
    run = lambda: update(f, seq[1][2], seq[1][3])
    run()
elif mode != "solve":
    run = fa
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    with record_function("STEP"):
        r = run()
    torch.cuda.synchronize()
prof.export_chrome_trace(out)
ev = json.load(open(out))["traceEvents"]
step = [e for e in ev if e.get("name") == "STEP" and e.get("ph") == "X"][0]
t0, t1 = step["ts"], step["ts"] + step["dur"]
ks = sorted([e for e in ev if e.get("cat") == "kernel" and e.get("ph") == "X"], key=lambda e: e["ts"])
print(f"step wall {step['dur']/1e3:.2f} ms, {len(ks)} kernels")
busy, cur_s, cur_e = 0.0, None, None
gaps = []
for e in ks:
    s, d = e["ts"], e["ts"] + e["dur"]
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
            gaps.append((cur_e, s))
        cur_s, cur_e = s, d
    else:
        cur_e = max(cur_e, d)
if cur_e is not None:
    busy += cur_e - cur_s
first = ks[0]["ts"] if ks else t0
print(f"GPU busy union {busy/1e3:.2f} ms; first kernel at +{(first-t0)/1e3:.2f} ms; "
      f"last kernel end +{(cur_e-t0)/1e3:.2f} ms")
big = sorted(gaps, key=lambda g: g[0] - g[1])[:15]
print("largest idle gaps (start +ms, length ms):",
      " ".join(f"+{(a-t0)/1e3:.2f}:{(b_-a)/1e3:.2f}" for a, b_ in sorted(big)))
by_stream = {}
for e in ks:
    by_stream.setdefault(e["args"].get("stream"), []).append(e)
for s_, lst in by_stream.items():
    print(f"stream {s_}: {len(lst)} kernels, {sum(e['dur'] for e in lst)/1e3:.2f} ms")
if "-v" in sys.argv:
    hs = [e for e in ev if e.get("cat") == "user_annotation" and e.get("ph") == "X"
          and e.get("name") != "STEP"]
    rows = [(e["ts"], "K", e) for e in ks] + [(e["ts"], "H", e) for e in hs]
    for ts, kind, e in sorted(rows, key=lambda r: r[0]):
        if kind == "K":
            nm = e["name"].split("(")[0].replace("void ", "")[:40]
            print(f"  +{(ts-t0)/1e3:8.3f} {e['dur']/1e3:7.3f} s{e['args'].get('stream')} {nm} "
                  f"g{e['args'].get('grid')} b{e['args'].get('block')}")
        else:
            print(f"  +{(ts-t0)/1e3:8.3f} {e['dur']/1e3:7.3f} HOST {e['name']}")
