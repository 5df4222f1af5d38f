"""Process-parallel driver of the CPU oracle -- TEST INFRASTRUCTURE / CPU REFERENCE ARM ONLY.

Same rules as ``skel_oracle``: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (cpu_baseline leg, ``--impl reference``) may use it.

The reference parallelises a level over a thread pool (``workers``,
``skel.py:354-357``; BLAS pinned to one thread, ``skel.py:441``).  Under the GIL
that pool does not scale (cfg2: 4.9 s at 1 worker, 6.0 s at 8 in this
container), so "all the host threads it can use" is realised here with forked
worker processes running the *same* per-box code:

* compression: the boxes of one level are independent (skel.py:340-361); each
  level forks a pool that inherits the pass state (active sets, children's
  factors) and returns the per-box ``BoxOut``;
* ``_finish_top``: H columns and the level sweeps run on the workers over
  anonymous shared mappings of UH / PsiV / UH_div (boxes of one level touch
  disjoint rows); the q x q Schur contributions come back and are added in box
  order, as the serial loop does.

Every per-box NumPy/LAPACK call is the serial oracle's, so the result is
bitwise the serial oracle's (``tests/test_oracle_golden.py``).
"""

from __future__ import annotations

import mmap
import multiprocessing as mp
import os
import time

import numpy as np
from threadpoolctl import threadpool_limits

from . import skel_oracle as O

_STATE: dict = {}          # inherited by forked workers


def _ctx():
    return mp.get_context("fork")


def _compress(key):
    return _STATE["pass"].compress(key)


def _shared(shape):
    n = int(np.prod(shape)) * 8
    mm = mmap.mmap(-1, max(n, 8), flags=mmap.MAP_SHARED, prot=mmap.PROT_READ | mmap.PROT_WRITE)
    a = np.frombuffer(mm, dtype=np.float64, count=int(np.prod(shape))).reshape(shape)
    return a, mm


def _aug_cols(ids):
    s = _STATE
    for i in ids:
        O._aug_column(s["points"], s["centers"][i], i, s["UH"])
    return len(ids)


def _sweep(key):
    s = _STATE
    part = s["pass"]._sweep_box(key, s["UH"], s["PsiV"], s["UH_div"])
    nz = np.flatnonzero(np.any(part != 0.0, axis=1))   # rows that are all +-0 add nothing
    return nz, part[nz]


def _order(p, keys):
    """Largest boxes first (load balance); results are put back by key."""
    cost = []
    for k in keys:
        bx = p.tree.boxes[k]
        n = len(p.active[k]) if k in p.active else 0
        cost.append(-(n * n))
    return [keys[i] for i in np.argsort(cost, kind="stable")]


def run(p: "O._Pass", procs: int):
    """_Pass.run with the boxes of every level compressed on ``procs`` processes."""
    t = p.tree
    for k, bx in t.boxes.items():
        if bx.leaf:
            p.active[k] = p.leaf_dofs(bx)
    sweep = []
    for lev in range(t.depth, 0, -1):
        keys = t.levels[lev]
        for k in keys:
            bx = t.boxes[k]
            if not bx.leaf:
                p.active[k] = np.concatenate([p.out[c].skel for c in bx.kids])
        todo = _order(p, list(keys))
        if procs > 1 and len(todo) > 1:
            _STATE["pass"] = p
            with _ctx().Pool(min(procs, len(todo))) as pool:
                outs = pool.map(_compress, todo, chunksize=1 if len(todo) < 4 * procs else 4)
            _STATE.clear()
            for k, r in zip(todo, outs):
                p.out[k] = r
        else:
            for k in todo:
                p.out[k] = p.compress(k)
        sweep.append((lev, keys))
    return sweep


def top(p: "O._Pass", sweep, procs: int):
    """_finish_top (skel.py:364-425) with H and the level sweeps on ``procs`` processes."""
    g, t = p.g, p.tree
    q = 3 * g.n_holes
    if not q or procs <= 1:
        return p.top(sweep)
    root = t.boxes[O.ROOT]
    rd = p.leaf_dofs(root) if root.leaf else np.concatenate([p.out[c].skel for c in root.kids])
    p.active[O.ROOT] = rd
    E_root = p.block_E(root)
    nd = 2 * len(g.positions)
    nonroot = np.ones(nd, dtype=bool)
    nonroot[rd] = False
    UH, m1 = _shared((nd, q))
    PsiV, m2 = _shared((nd, q))
    UH_div, m3 = _shared((nd, q))
    PsiV[...] = O.aug_functionals(g)
    UH_div[...] = 0.0
    points = np.atleast_2d(np.asarray(g.positions, float))
    centers = np.atleast_2d(np.asarray(g.hole_centers, float))
    _STATE.update(points=points, centers=centers, UH=UH, PsiV=PsiV, UH_div=UH_div)
    _STATE["pass"] = p
    schur = np.zeros((q, q))
    with _ctx().Pool(procs) as pool:
        chunks = [list(range(i, len(centers), procs)) for i in range(procs)]
        pool.map(_aug_cols, [c for c in chunks if c])
        for _, keys in sweep:
            order = _order(p, list(keys))
            parts = dict(zip(order, pool.map(_sweep, order, chunksize=1 if len(order) < 4 * procs else 4)))
            for k in keys:                       # box order of the serial loop
                nz, rows = parts[k]
                schur[nz] += rows
    _STATE.clear()
    ns = len(rd)
    C = np.zeros((ns + q, ns + q))
    C[:ns, :ns] = E_root
    C[:ns, ns:] = UH[rd]
    C[ns:, :ns] = PsiV[rd].T
    C[ns:, ns:] = -np.eye(q) - schur
    topf = O.LU(C)
    kpl = {lev: max((len(p.out[k].S) for k in keys), default=0) for lev, keys in sweep}
    f = O.OracleFactorization(g, t, p.tol, dict(p.out), sweep, rd, E_root, topf,
                              UH, PsiV, UH_div, nonroot,
                              {"k_per_level": kpl, "root_size": len(rd)})
    f._shared_maps = (m1, m2, m3)
    return f


def factor(g, tree, tol, proxy_count=64, proxy_factor=1.5, procs=None):
    """skel.py:428-453 on ``procs`` processes (default: all host cores)."""
    procs = procs or os.cpu_count() or 1
    t0 = time.perf_counter()
    with threadpool_limits(limits=1):          # skel.py:441
        p = O._Pass(g, tree, tol, proxy_count, proxy_factor)
        sweep = run(p, procs)
        f = top(p, sweep, procs)
    f.stats["factor_time"] = time.perf_counter() - t0
    return f


def factor_full(g, leaf_cap, tol, proxy_count, proxy_factor, procs=None):
    t = O.QTree(g.positions, leaf_cap)
    f = factor(g, t, tol, proxy_count, proxy_factor, procs)
    f.proxy_count, f.proxy_factor = proxy_count, proxy_factor
    return f
