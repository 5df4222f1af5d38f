"""cProfile of one warm cfg2 factor (host-side overhead hunting)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor

wl = configs.by_name(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
t = build_tree(wl.boundary.positions, wl.leaf_cap)
for _ in range(2):
    f = factor(SystemSpec(), wl.boundary, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
del f
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
f = factor(SystemSpec(), wl.boundary, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
torch.cuda.synchronize()
pr.disable()
print("factor_time", f.stats["factor_time"])
st = pstats.Stats(pr)
st.sort_stats(sys.argv[2] if len(sys.argv) > 2 else "tottime").print_stats(45)
