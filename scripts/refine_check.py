"""Does one step of iterative refinement with the compressed apply() reduce the
exact-operator residual on the ill-conditioned cfg3?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, system_matvec
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
wl = configs.by_name(name)
b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
rng = np.random.default_rng(1)
rhs = np.concatenate([rng.standard_normal(2 * b.n_nodes), np.zeros(3 * b.n_holes)])
x = f.solve(rhs)
res = lambda v: np.linalg.norm(system_matvec(SystemSpec(), b, v) - rhs) / np.linalg.norm(rhs)
print("plain solve residual", res(x))
for it in range(3):
    r = rhs - f.apply(x)
    print(f"  compressed residual before step {it}: {np.linalg.norm(r)/np.linalg.norm(rhs):.3e}")
    x = x + f.solve(r)
    print(f"refined {it+1}: exact residual {res(x):.3e}")
