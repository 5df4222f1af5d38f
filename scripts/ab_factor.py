"""A/B timing of one factorization config under the current environment (knob sweeps).

usage: python scripts/ab_factor.py cfg3 [steps]  -> median / min ms and per-family device ms
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, _lib
from paper_2001_11619_b200 import skel as S
wl = configs.by_name(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
b = wl.boundary
b._skb_device = S.DeviceBoundary(b)
def step():
    t = build_tree(b.positions, wl.leaf_cap)
    return factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
for _ in range(3):
    f = step(); del f
ts = []
for _ in range(n):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    f = step(); torch.cuda.synchronize()
    ts.append(1e3 * (time.perf_counter() - t0)); del f
_lib.prof_enable(True); _lib.prof_read(reset=True)
f = step(); torch.cuda.synchronize(); del f
fam = _lib.prof_read(reset=True); _lib.prof_enable(False)
env = {k: v for k, v in os.environ.items() if k.startswith("SKB_")}
print(f"{env} {wl.name}: median {np.median(ts):.1f} min {min(ts):.1f} ms;",
      " ".join(f"{k}={v['ms']:.1f}" for k, v in sorted(fam.items(), key=lambda kv: -kv[1]['ms'])), flush=True)
