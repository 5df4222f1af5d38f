"""Repeat cfg2 factor + solve and compare bitwise across runs (engine race hunt)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor
from paper_2001_11619_b200 import skel as S
wl = configs.cfg2()
b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
rhs = wl.extra["rhs"]
ref = None
bad = 0
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for i in range(n):
    f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
    x = f.solve(rhs)
    if ref is None:
        ref = x
    elif not np.array_equal(x, ref):
        bad += 1
        print("run", i, "differs", np.linalg.norm(x - ref) / np.linalg.norm(ref))
    del f
print(os.environ.get("SKB_ENGINE_VARIANT", "default"), "mismatching runs:", bad, "of", n - 1)
