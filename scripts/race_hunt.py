"""Race localisation for engine update chains (debug tool).

Runs the same cfg2 hole-move chain many times from ONE base factorization and
compares, per step, the solve (bitwise), the factor blocks of the top levels
and -- with SKB_ENGINE_SNAP=<level> -- that level's ID stacks after assembly /
pre-reduction / QRCP.  Prints one JSON summary line.
  python scripts/race_hunt.py CHAINS MOVES
"""
import ctypes, hashlib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update, _lib

SZ = {"T": lambda k, r: k * r, "Xrr": lambda k, r: r * r, "LU": lambda k, r: r * r,
      "Xsr": lambda k, r: k * r, "Xrsdiv": lambda k, r: r * k, "Xss": lambda k, r: k * k}
lib = _lib.load()
from paper_2001_11619_b200 import skel as S


def h(a):
    return hashlib.md5(np.ascontiguousarray(a).tobytes()).hexdigest()[:10]


def fetch(addr, n):
    return S._fetch(int(addr), 1, n)


def snap_factors(f, maxlev):
    torch.cuda.synchronize()
    out = {}
    for L in f.levels:
        if L.lev > maxlev:
            continue
        for j, i in enumerate(L.idx):
            k, r = int(L.k[j]), int(L.r[j])
            ent = [k, h(L.batch.perm[L.batch.act_off[j]:L.batch.act_off[j + 1]])]
            for fld, fn in SZ.items():
                ent.append(h(fetch(L.P[fld][j], fn(k, r))))
            out[(int(L.lev), int(i))] = ent
    return out


def snaps():
    res = []
    for w in range(3):
        n = lib.skb_debug_snap(w, None, 0)
        if n < 0:
            res.append(None)
            continue
        buf = np.empty(max(n, 1))
        lib.skb_debug_snap(w, buf.ctypes.data, n)
        res.append(h(buf[:n]))
    return res


def main():
    chains, moves = int(sys.argv[1]), int(sys.argv[2])
    maxlev = int(os.environ.get("RACE_MAXLEV", "3"))
    wl = configs.cfg2()
    b = wl.boundary
    t = build_tree(b.positions, wl.leaf_cap)
    rhs = wl.extra["rhs"]
    seq = configs.hole_move_sequence(b, moves)
    mk = lambda: factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count,
                        proxy_factor=wl.proxy_factor)
    base = mk()
    x0 = base.solve(rhs)
    fbad = 0
    for _ in range(3):
        fb = mk()
        fbad += not np.array_equal(fb.solve(rhs), x0)
        del fb
    runs = []
    for rep in range(chains):
        cur = base
        ch = []
        for (hole, d, nb, rp) in seq:
            cur = update(cur, nb, rp)
            sn = snaps()
            ch.append((cur.solve(rhs), snap_factors(cur, maxlev), sn))
        runs.append(ch)
    bad = []
    for rep in range(1, chains):
        for s, ((xa, fa, sa), (xc, fc, sc)) in enumerate(zip(runs[0], runs[rep])):
            if np.array_equal(xa, xc):
                if sa != sc:
                    bad.append({"chain": rep, "step": s, "solve_same": True, "snap_same": [u == v for u, v in zip(sa, sc)]})
                continue
            diffs = []
            for key in sorted(fa):
                if fa[key] != fc.get(key):
                    flds = [n for n, u, v in zip(["k", "perm"] + list(SZ), fa[key], fc[key]) if u != v]
                    diffs.append([key[0], key[1], flds])
            bad.append({"chain": rep, "step": s, "rel": float(np.linalg.norm(xa - xc) / np.linalg.norm(xa)),
                        "snap_same": [u == v for u, v in zip(sa, sc)], "boxes": diffs[:8]})
    print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith(("SKB_", "CUDA_LAUNCH"))},
                      "factor_mismatch": fbad, "steps": moves * (chains - 1),
                      "mismatch_steps": sum(1 for x in bad if not x.get("solve_same")),
                      "details": bad[:12]}), flush=True)


if __name__ == "__main__":
    main()
