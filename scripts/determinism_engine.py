"""Repeat cfg2 factor + solve and compare bitwise across runs (engine race hunt)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2001_11619_b200 import _lib
if os.environ.get("SKB_LIB"):          # compare another build of the library
    _lib.load(os.environ["SKB_LIB"])
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

# update chains: the same 6 hole moves twice, solves compared bitwise per step
if len(sys.argv) > 2:
    from paper_2001_11619_b200 import update
    seq = configs.hole_move_sequence(b, 6)
    runs = []
    for rep in range(int(sys.argv[2])):
        cur = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
        xs = []
        for (h, d, nb, rp) in seq:
            cur = update(cur, nb, rp)
            xs.append(cur.solve(rhs))
        runs.append(xs)
    ubad = sum(not np.array_equal(a, c) for xs in runs[1:] for a, c in zip(xs, runs[0]))
    print("update chains: mismatching steps:", ubad, "of", 6 * (len(runs) - 1))
