"""The cfg4 test sequence: 6 updates, then refactor; checks xr against a second refactor."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update
wl = configs.cfg2()
b = wl.boundary
rhs = wl.extra["rhs"]
t = build_tree(b.positions, wl.leaf_cap)
f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    cur = f
    for s, (h, d, nb, rep) in enumerate(configs.hole_move_sequence(b, 6)):
        cur = update(cur, nb, rep)
    t2 = build_tree(nb.positions, wl.leaf_cap, root_box=(f.tree.root_center, f.tree.root_half_width))
    xu = cur.solve(rhs)
    xs = []
    for r in range(3):
        fr = factor(SystemSpec(), nb, t2, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
        xs.append(fr.solve(rhs))
        xs.append(fr.solve(rhs))
        del fr
    print("trial", trial, "xu-xr", [float(np.abs(xu - x).max()) for x in xs], flush=True)
