"""Find the first level/box where two engine factorizations of cfg2 differ."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor
wl = configs.cfg2()
b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)

from paper_2001_11619_b200.skel import _fetch
def snap(f):
    out = {}
    for L in f.levels:
        for bi, key in enumerate(L.keys):
            bf = f.factors[key]
            r = int(L.r[bi])
            out[("LU",) + tuple(key)] = _fetch(L.P["LU"][bi], r, r).copy()
            out[key] = (L.lev, bf.skel_dofs.copy(), bf.T.copy(), bf.Xss_mod.copy(), bf.X_rr.copy(),
                        bf.X_sr.copy(), bf.X_rs_div.copy())
    return out, f.top.cpu().numpy().copy()

from paper_2001_11619_b200 import skel as SK
if os.environ.get("REF_PY"):
    SK._ENGINE_ON = False
ref, reftop = snap(factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor))
SK._ENGINE_ON = os.environ.get("SKB_ENGINE", "1") != "0"
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    cur, top = snap(factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor))
    diffs = {}
    for key, val in ref.items():
        if key[0] == "LU":
            if not np.array_equal(val, cur[key]):
                print("   LU differs for", key[1:])
            continue
        (lev, sk, T, X, R, SR, RSD) = val
        l2, sk2, T2, X2, R2, SR2, RSD2 = cur[key]
        kind = None
        if not np.array_equal(sk, sk2): kind = "skel"
        elif not np.array_equal(T, T2): kind = "T"
        elif not np.array_equal(R, R2): kind = "Xrr"
        elif not np.array_equal(SR, SR2): kind = "Xsr"
        elif not np.array_equal(RSD, RSD2): kind = "Xrsdiv"
        elif not np.array_equal(X, X2): kind = "Xss"
        if kind:
            diffs.setdefault(lev, []).append((key, kind))
    for key, kinds in [(k, v) for lv_ in diffs for (k, v) in diffs[lv_]][:0]:
        pass
    if diffs:
        lv = max(diffs)
        key0, kind0 = diffs[lv][0]
        if kind0 == "Xrsdiv":
            A0, A1 = ref[key0][6], cur[key0][6]
            d = np.abs(A0 - A1)
            rr, cc = np.nonzero(d)
            print(f"   {key0}: shape {A0.shape}, {len(rr)} entries differ, rows {sorted(set(rr.tolist()))[:12]}, "
                  f"cols {sorted(set(cc.tolist()))[:12]}, max rel {d.max() / np.abs(A0).max():.2e}")
        print(f"run {it}: differing levels {sorted(diffs, reverse=True)}; deepest level {lv}: {diffs[lv][:6]} ({len(diffs[lv])} boxes)")
    else:
        print(f"run {it}: identical factors; top equal {np.array_equal(top, reftop)}")
