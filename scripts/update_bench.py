"""cfg4: successive hole moves on cfg2; time update(), check update == refactor bitwise."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
check_every = int(sys.argv[2]) if len(sys.argv) > 2 else 5
wl = configs.cfg2()
b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
rhs = wl.extra["rhs"]
seq = configs.hole_move_sequence(b, steps)
times, dirty, same = [], [], []
cur = f
for s, (h, d, nb, rep) in enumerate(seq):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cur = update(cur, nb, rep)
    torch.cuda.synchronize()
    times.append(1e3 * (time.perf_counter() - t0))
    dirty.append(cur.stats["n_dirty"])
    if (s + 1) % check_every == 0:
        t2 = build_tree(nb.positions, wl.leaf_cap, root_box=(t.root_center, t.root_half_width))
        fr = factor(SystemSpec(), nb, t2, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
        same.append(bool(np.array_equal(fr.solve(rhs), cur.solve(rhs))))
        del fr
out = {"steps": steps, "update_ms_mean": float(np.mean(times[1:])), "update_ms_median": float(np.median(times)),
       "update_ms_first": times[0], "n_dirty_mean": float(np.mean(dirty)),
       "n_boxes": cur.stats["n_boxes"], "update_equals_refactor_bitwise": same,
       "factor_ms": 1e3 * f.stats["factor_time"]}
print(json.dumps(out))
