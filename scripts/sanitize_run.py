"""Small factor/update/solve run for compute-sanitizer (memcheck / racecheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update
for name in (sys.argv[1:] or ["mini"]):
    wl = configs.by_name(name)
    b = wl.boundary
    t = build_tree(b.positions, wl.leaf_cap)
    f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
    rhs = np.ones(f.dim)
    x = f.solve(rhs)
    seq = configs.hole_move_sequence(b, 2) if b.n_holes else []
    for (h, d, nb, rep) in seq:
        f = update(f, nb, rep)
    if seq:
        x2 = f.solve(rhs)
    print(name, "ok", float(np.abs(x).max()), flush=True)
