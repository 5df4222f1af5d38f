"""Repeatability of factor() on the engine and the Python loop (debug)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor
from paper_2001_11619_b200 import skel
wl = getattr(configs, sys.argv[1])()
b = wl.boundary
rhs = np.random.default_rng(11).standard_normal(2 * b.n_nodes + 3 * b.n_holes)
res = {}
for on in (False, True, False, True):
    skel._ENGINE_ON = on
    t = build_tree(b.positions, wl.leaf_cap)
    f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
    x = f.solve(rhs)
    sk = {k: f.factors[k].skel_dofs for k in f.factors.keys()}
    T = {k: f.factors[k].T for k in f.factors.keys()}
    res.setdefault(on, []).append((x, sk, T, f))
for on in (False, True):
    a, c = res[on]
    print("engine" if on else "python", "repeat solve equal:", np.array_equal(a[0], c[0]))
a, c = res[False][0], res[True][0]
print("python vs engine solve equal:", np.array_equal(a[0], c[0]))
dk = [k for k in a[1] if not np.array_equal(a[1][k], c[1][k])]
dT = [k for k in a[2] if not np.array_equal(a[2][k], c[2][k])]
print("skel diffs", dk[:10], "T diffs", len(dT), dT[:10])
for k in dT[:3]:
    L = [L for L in a[3].levels if k in L.keys][0]
    j = L.keys.index(k)
    bt = L.batch
    print(k, "nB", bt.nB[j], "k", bt.k[j], "rows?", getattr(bt, "_rows", None), "maxdiff", np.abs(a[2][k]-c[2][k]).max())
