"""Incremental vs full augmentation sweep in update(): compare UH / PsiV / UH_div / schur (debug)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update
from paper_2001_11619_b200 import skel as S
from paper_2001_11619_b200.geometry import MoveHole, apply_perturbation
wl = configs.mini_holes()
b = wl.boundary
f = factor(SystemSpec(), b, build_tree(b.positions, wl.leaf_cap), wl.tol, proxy_count=wl.proxy_count,
           proxy_factor=wl.proxy_factor)
nb, rep = apply_perturbation(b, [MoveHole(2, translation=(0.1, -0.05))])
out = {}
for inc in (False, True):
    S._INC_SWEEP = inc
    fu = update(f, nb, rep)
    torch.cuda.synchronize()
    out[inc] = (fu.UH.cpu().numpy(), fu.PsiV.cpu().numpy(), fu.UH_div.cpu().numpy(), fu.top.cpu().numpy(), fu)
names = ["UH", "PsiV", "UH_div", "top"]
for i, nm in enumerate(names):
    a, c = out[False][i], out[True][i]
    bad = np.argwhere(a != c)
    print(nm, "equal" if len(bad) == 0 else f"{len(bad)} entries differ; max {np.abs(a - c).max():.3e}; rows {np.unique(bad[:, 0])[:20]} cols {np.unique(bad[:, 1])[:20]}")
fu = out[True][4]
t = fu.tree
dm = np.zeros(len(t.lev), bool)
dk = fu.stats["dirty"]
for L in fu.levels:
    for j, i in enumerate(L.idx):
        pass
# which box owns differing rows (as eliminated / skeleton rows)
a, c = out[False][0], out[True][0]
rows = np.unique(np.argwhere(a != c)[:, 0])
own = {}
for L in fu.levels:
    for j in range(len(L.idx)):
        rd = L.rd[L.rd_off[j]:L.rd_off[j + 1]]
        for r in rd:
            own[int(r)] = (L.lev, int(L.idx[j]), t.key(int(L.idx[j])) in dk)
print("owners of differing UH rows (lev, box, dirty):", sorted({own.get(int(r), "root") for r in rows}, key=str)[:20])
