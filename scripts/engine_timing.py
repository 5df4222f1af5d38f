import os, sys
sys.path.insert(0, os.getcwd())
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor
import torch
wl = configs.by_name("cfg2"); b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
for i in range(4):
    if i == 3: print("=== last run", file=sys.stderr, flush=True)
    f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
    torch.cuda.synchronize()
