"""Stage breakdown + timings of factor / solve / update on one config (GPU box)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update
from paper_2001_11619_b200 import skel as S

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
wl = configs.by_name(name)
b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
print(name, "nodes", b.n_nodes, "boxes", len(t.lev), "depth", t.depth, flush=True)
f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
print("warm factor", f.stats["factor_time"], "k/level", f.stats["k_per_level"], flush=True)
times = []
for _ in range(2):
    f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
    times.append(f.stats["factor_time"])
print("factor s", times, "unknowns/s", f.dim / min(times), flush=True)
S._Prof.enabled = True
S._Prof.reset()
f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
S._Prof.enabled = False
tot = sum(S._Prof.acc.values())
for k, v in sorted(S._Prof.acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:16s} {v*1e3:9.2f} ms  {100*v/tot:5.1f}%")
print("profiled factor", f.stats["factor_time"])
rng = np.random.default_rng(0)
for nr in (1, 16):
    X = torch.from_numpy(rng.standard_normal((f.dim, nr))).cuda()
    f.solve(X)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        f.solve(X)
    torch.cuda.synchronize()
    print(f"solve nrhs={nr}: {(time.perf_counter()-t0)/3*1e3:.2f} ms", flush=True)
if b.n_holes:
    seq = configs.hole_move_sequence(b, 3)
    cur = f
    for h, d, nb, rep in seq:
        torch.cuda.synchronize()
        cur = update(cur, nb, rep)
        print(f"update hole {h}: {cur.stats['update_time']*1e3:.1f} ms, dirty {cur.stats['n_dirty']}/{cur.stats['n_boxes']}", flush=True)
print("max mem GB", torch.cuda.max_memory_allocated() / 1e9)
