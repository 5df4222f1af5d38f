"""Locate run-to-run differences of engine update chains: per step, per level,
per box: skeleton (k, perm) and a hash of every factor block."""
import ctypes, hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update

cudart = ctypes.CDLL("libcudart.so") if os.path.exists("/usr/local/cuda/lib64/libcudart.so") else None
if cudart is None:
    import glob
    cudart = ctypes.CDLL(glob.glob("/usr/local/cuda/lib64/libcudart.so*")[0])
SZ = {"T": lambda k, r: k * r, "Xrr": lambda k, r: r * r, "LU": lambda k, r: r * r,
      "Xsr": lambda k, r: k * r, "Xrsdiv": lambda k, r: r * k, "Xss": lambda k, r: k * k}


def snap(f):
    torch.cuda.synchronize()
    out = {}
    for L in f.levels:
        for j, i in enumerate(L.idx):
            k, r = int(L.k[j]), int(L.r[j])
            ent = [int(k)]
            for fld, fn in SZ.items():
                n = fn(k, r)
                buf = np.empty(max(n, 1), np.float64)
                if n:
                    cudart.cudaMemcpy(ctypes.c_void_p(buf.ctypes.data), ctypes.c_void_p(int(L.P[fld][j])),
                                      ctypes.c_size_t(8 * n), 2)
                ent.append(hashlib.md5(buf[:n].tobytes()).hexdigest()[:8])
            out[(L.lev, int(i))] = ent
    return out


wl = configs.cfg2()
b = wl.boundary
t = build_tree(b.positions, wl.leaf_cap)
rhs = wl.extra["rhs"]
seq = configs.hole_move_sequence(b, 6)
chains = []
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    cur = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
    ch = []
    for (h, d, nb, rp) in seq:
        cur = update(cur, nb, rp)
        ch.append((snap(cur), cur.solve(rhs), getattr(cur, "stats", {}).get("dirty")))
    chains.append(ch)
for rep in range(1, len(chains)):
    for s, ((a, xa, da), (c, xc, dc)) in enumerate(zip(chains[0], chains[rep])):
        if np.array_equal(xa, xc):
            continue
        diffs = [(key, a[key], c.get(key)) for key in sorted(a) if a[key] != c.get(key)]
        print(f"chain {rep} step {s}: solve differs; {len(diffs)} boxes differ; first:")
        for key, ea, ec in diffs[:6]:
            flds = [n for n, u, v in zip(["k"] + list(SZ), ea, ec) if u != v]
            print("   level/box", key, "fields", flds)
print("done")
