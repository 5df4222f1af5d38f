"""Host time per C-ABI entry point (Python + library host work) in warm factorizations."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, _lib
wl = configs.by_name(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
fa = lambda: factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
for _ in range(3):
    f = fa(); del f
_lib.CALL_TIMES = {}
reps = 5
for _ in range(reps):
    f = fa(); del f
tot = sum(v[1] for v in _lib.CALL_TIMES.values())
print(f"per factor: {1e3*tot/reps:.1f} ms in {sum(v[0] for v in _lib.CALL_TIMES.values())/reps:.0f} calls")
for k, (n, s_) in sorted(_lib.CALL_TIMES.items(), key=lambda kv: -kv[1][1]):
    print(f"   {k:26s} {n/reps:6.1f} calls {1e3*s_/reps:7.2f} ms  {1e6*s_/n:7.1f} us/call")
