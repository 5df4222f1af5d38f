"""Median hole-move update time on cfg2 (engine lead from SKB_ENGINE_LEAD)."""
import gc, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update
wl = configs.cfg2(); b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
seq = configs.hole_move_sequence(b, 14)
ts = []
for i, (h, d, nb, rp) in enumerate(seq):
    gc.collect()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = update(f, nb, rp)
    torch.cuda.synchronize()
    if i >= 2:
        ts.append((time.perf_counter() - t0) * 1e3)
print(os.environ.get("SKB_ENGINE_LEAD", "default"), "update ms median %.2f" % np.median(ts), " ".join("%.1f" % x for x in ts))
