import sys; sys.path.insert(0,'/root/repo')
import numpy as np
from oracle import skel_oracle as O
from paper_2001_11619_b200 import configs, build_tree, factor, SystemSpec
from paper_2001_11619_b200 import skel as S
S.PIVOT_RATIO_FLOOR = 2e-2; O.PIVOT_FLOOR = 2e-2
wl = configs.mini_holes()
t = build_tree(wl.boundary.positions, wl.leaf_cap)
f = factor(SystemSpec(), wl.boundary, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
ref = O.factor_full(wl.boundary, wl.leaf_cap, wl.tol, wl.proxy_count, wl.proxy_factor)
ratio = {}
for L in f.levels:
    for bi, key in enumerate(L.keys):
        ratio[key] = (L.batch.ratio[bi], L.batch.info[bi], int(L.k[bi]), int(L.batch.nB[bi]))
for k in sorted(ref.boxes):
    kg = len(f.factors[k].S_loc); kr = len(ref.boxes[k].S)
    if kg != kr or not np.array_equal(f.factors[k].skel_dofs, ref.boxes[k].skel):
        print(k, "gpu k", kg, "ref k", kr, "gpu ratio/info/k/nB", ratio[k], "ref ratio", ref.boxes[k].lu.pivot_ratio)
