"""One warm factor of a config (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
wl = configs.by_name(name)
t = build_tree(wl.boundary.positions, wl.leaf_cap)
f = factor(SystemSpec(), wl.boundary, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
torch.cuda.synchronize()
print("factor", f.stats["factor_time"])
