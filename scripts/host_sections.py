"""Host time per pipeline section of warm factorizations (SKB_HOST_PROF=1)."""
import os, sys, time
os.environ["SKB_HOST_PROF"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor
from paper_2001_11619_b200 import skel as S
wl = configs.by_name(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
fa = lambda: factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
for _ in range(3):
    f = fa(); del f
reps = 5
S._HostTimer.acc.clear()
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(reps):
    f = fa(); del f
torch.cuda.synchronize()
print(f"wall per factor {1e3*(time.perf_counter()-t0)/reps:.1f} ms")
for k, v in sorted(S._HostTimer.acc.items(), key=lambda kv: -kv[1]):
    print(f"   {k:16s} {1e3*v/reps:7.2f} ms")
