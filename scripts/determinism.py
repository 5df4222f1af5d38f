"""Repeat factor + solve on the same input and report bitwise differences."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
wl = configs.by_name(name)
b = wl.boundary
seq = configs.hole_move_sequence(b, 6)
nb = seq[5][2]
rhs = wl.extra["rhs"] if "rhs" in wl.extra else np.ones(2 * b.n_nodes + 3 * b.n_holes)
t = build_tree(b.positions, wl.leaf_cap)
t2 = build_tree(nb.positions, wl.leaf_cap, root_box=(t.root_center, t.root_half_width))
for bb, tt, lab in ((b, t, "base"), (nb, t2, "moved")):
    xs, ks = [], []
    for r in range(reps):
        f = factor(SystemSpec(), bb, tt, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
        xs.append(f.solve(rhs))
        ks.append({L.lev: (L.k.copy(), L.batch.perm.copy()) for L in f.levels})
        del f
    for r in range(1, reps):
        d = np.abs(xs[r] - xs[0]).max()
        lv = [lev for lev in ks[0] if not (np.array_equal(ks[0][lev][0], ks[r][lev][0])
                                          and np.array_equal(ks[0][lev][1], ks[r][lev][1]))]
        print(lab, "rep", r, "max|dx|", d, "levels with different skeletons", lv, flush=True)
