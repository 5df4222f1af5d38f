"""Median wall time of cfg2 hole-move updates (moves 3..N) under the current environment."""
import gc, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update
wl = configs.cfg2(); b = wl.boundary
f = factor(SystemSpec(), b, build_tree(b.positions, wl.leaf_cap), wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
seq = configs.hole_move_sequence(b, n)
ts = []
for i, (h, d, nb, rp) in enumerate(seq):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = update(f, nb, rp)
    torch.cuda.synchronize()
    if i >= 3:
        ts.append((time.perf_counter() - t0) * 1e3)
env = {k: v for k, v in os.environ.items() if k.startswith("SKB_")}
print(f"{env} update ms median {np.median(ts):.2f} min {min(ts):.2f} max {max(ts):.2f}", flush=True)
