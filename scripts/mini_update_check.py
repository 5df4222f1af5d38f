"""Repeat the mini-holes update == refactor check (tests/test_gpu_parity.py)
N times in one process; report mismatches and which of update / refactor moved.
SKB_LIB selects another build of the library."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2001_11619_b200 import _lib
if os.environ.get("SKB_LIB"):
    _lib.load(os.environ["SKB_LIB"])
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update
from paper_2001_11619_b200.geometry import MoveHole, apply_perturbation
wl = configs.mini_holes()
b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
nb, rep = apply_perturbation(b, [MoveHole(2, translation=(0.1, -0.05))])
rhs = np.random.default_rng(3).standard_normal(2 * nb.n_nodes + 3 * nb.n_holes)
t2 = build_tree(nb.positions, wl.leaf_cap, root_box=(t.root_center, t.root_half_width))
ref_u = ref_r = None
bad = nu = nr = 0
N = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for it in range(N):
    f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
    xu = update(f, nb, rep).solve(rhs)
    xr = factor(SystemSpec(), nb, t2, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor).solve(rhs)
    if ref_u is None:
        ref_u, ref_r = xu, xr
    nu += not np.array_equal(xu, ref_u)
    nr += not np.array_equal(xr, ref_r)
    bad += not np.array_equal(xu, xr)
print(f"{os.environ.get('SKB_LIB', 'current')}: update!=refactor {bad}/{N}; update moved {nu}, refactor moved {nr}")
