"""Host time per factor() section (SKB_HOST_PROF=1), last of 4 cfg2 factorizations."""
import os, sys
os.environ.setdefault("SKB_HOST_PROF", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, skel
wl = configs.by_name(sys.argv[1] if len(sys.argv) > 1 else "cfg2"); b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
for i in range(4):
    skel._HostTimer.acc.clear()
    f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
    torch.cuda.synchronize()
print("factor %.2f ms" % (f.stats["factor_time"] * 1e3))
for k, v in sorted(skel._HostTimer.acc.items(), key=lambda x: -x[1]):
    print("  %-14s %8.3f ms" % (k, v * 1e3))
