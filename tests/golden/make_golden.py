"""Generate golden fixtures by running the UNMODIFIED reference ``skelsolve``.

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py

The reference is imported through the harness shim of SURVEY.md §8(c): a stub
``shapely.geometry.LinearRing`` (shapely is not installed; only
``geometry.py:236-238`` uses it) and a monkeypatch of ``_Compressor.far_dofs``
returning element [0] of its tuple (``skel.py:280`` vs ``skel.py:297``).  The
reference sources are not modified or copied.  Geometry comes from this repo's
analytic builders and is handed to the reference as ``Curve``/``Boundary``
objects built from the same arrays.
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from paper_2001_11619_b200 import configs  # noqa: E402
from paper_2001_11619_b200.geometry import MoveHole, apply_perturbation  # noqa: E402


def load_reference():
    shim = tempfile.mkdtemp(prefix="refshim_")
    os.makedirs(os.path.join(shim, "shapely"))
    open(os.path.join(shim, "shapely", "__init__.py"), "w").close()
    with open(os.path.join(shim, "shapely", "geometry.py"), "w") as fh:
        fh.write("class LinearRing:\n"
                 "    def __init__(self, pts): self.pts = pts\n"
                 "    is_simple = property(lambda self: True)\n")
    sys.path[:0] = [shim, "/root/reference/pkg/src"]
    import skelsolve as s
    from skelsolve import skel as sk
    orig = sk._Compressor.far_dofs
    sk._Compressor.far_dofs = lambda self, bx: orig(self, bx)[0]
    return s


def to_ref_boundary(s, b):
    """Reference Boundary from this repo's arrays (Curve bypasses the spline fit)."""
    curves = []
    for i, c in enumerate(b.curves):
        knots = c.nodes[:: max(1, c.n_nodes // 16)]
        spec = s.CurveSpec(knots, c.n_nodes, "outer" if i == 0 else "hole")
        curves.append(s.geometry.Curve(spec, c.nodes.copy(), c.weights.copy(),
                                       c.normals.copy(), c.curvatures.copy()))
    rb = s.Boundary(curves)
    assert np.array_equal(rb.positions, b.positions)
    assert np.array_equal(rb.hole_centers, b.hole_centers)
    return rb


def record_factor(s, wl, stack_boxes=2, t_boxes=6, pde=None):
    """Run the reference factor with a recorder on compress_box / PivotedQR."""
    from skelsolve import skel as sk
    b = to_ref_boundary(s, wl.boundary)
    spec = s.SystemSpec(pde or s.STOKES)
    tree = s.build_tree(b.positions, leaf_cap=wl.leaf_cap)
    rec = {}
    orig_cb = sk._Compressor.compress_box
    orig_qr = sk.PivotedQR.__init__
    cur = {}

    def qr_init(self, A):
        cur["stack"] = np.array(A, copy=True)
        orig_qr(self, A)
        cur["qr"] = self

    def cb(self, key):
        bx = self.tree.boxes[key]
        bf = orig_cb(self, key)
        F = self.far_dofs(bx)
        rec[key] = dict(active=np.array(bx.active), far=np.array(F), stack=cur["stack"],
                        k=len(bf.S_loc), S=np.array(bf.S_loc), T=bf.T,
                        diag=cur["qr"].diag.copy())
        return bf

    sk.PivotedQR.__init__ = qr_init
    sk._Compressor.compress_box = cb
    try:
        fct = s.factor(spec, b, tree, wl.tol, proxy_count=wl.proxy_count,
                       proxy_factor=wl.proxy_factor)
    finally:
        sk.PivotedQR.__init__ = orig_qr
        sk._Compressor.compress_box = orig_cb
    return b, spec, tree, fct, rec


def pack(rec, fct, prefix, stack_keys, t_keys):
    out = {}
    keys = sorted(rec)
    out[prefix + "keys"] = np.array(keys, dtype=np.int64)
    out[prefix + "k"] = np.array([rec[k]["k"] for k in keys], dtype=np.int64)
    S_all = [rec[k]["S"] for k in keys]
    out[prefix + "S_off"] = np.concatenate([[0], np.cumsum([len(x) for x in S_all])]).astype(np.int64)
    out[prefix + "S"] = np.concatenate(S_all).astype(np.int64)
    A_all = [rec[k]["active"] for k in keys]
    out[prefix + "act_off"] = np.concatenate([[0], np.cumsum([len(x) for x in A_all])]).astype(np.int64)
    out[prefix + "act"] = np.concatenate(A_all).astype(np.int64)
    F_all = [rec[k]["far"] for k in keys]
    out[prefix + "far_off"] = np.concatenate([[0], np.cumsum([len(x) for x in F_all])]).astype(np.int64)
    out[prefix + "far"] = np.concatenate(F_all).astype(np.int64)
    # pivot gaps for tie classification: min relative gap of |R_jj| over the first k
    for i, k in enumerate(stack_keys):
        out[prefix + f"stack{i}_key"] = np.array(k)
        out[prefix + f"stack{i}"] = rec[k]["stack"]
    for i, k in enumerate(t_keys):
        out[prefix + f"T{i}_key"] = np.array(k)
        out[prefix + f"T{i}"] = rec[k]["T"]
        out[prefix + f"diag{i}"] = rec[k]["diag"]
    out[prefix + "root_dofs"] = np.array(fct.root_dofs, dtype=np.int64)
    kpl = fct.stats["k_per_level"]
    out[prefix + "k_per_level"] = np.array([[l, kpl[l]] for l in sorted(kpl)], dtype=np.int64)
    return out


def main():
    s = load_reference()
    out = {}
    np.random.seed(0)

    # ---- SPEC.md:176-197 known-answer examples through the reference API
    idr = s.interpolative_decomposition(np.array([[1.0, 2.0], [2.0, 4.0]]), 1e-10)
    out["kat_rank1_S"] = np.array(idr.skeleton)
    out["kat_rank1_T"] = idr.T
    rng = np.random.default_rng(3)
    U = rng.standard_normal((60, 8))
    V = rng.standard_normal((8, 40))
    A = U @ V
    idr = s.interpolative_decomposition(A, 1e-10)
    out["kat_cluster_A"] = A
    out["kat_cluster_S"] = np.array(idr.skeleton)
    out["kat_cluster_T"] = idr.T

    # ---- cfg1 (simply connected star, the reference's CPU-runnable case)
    wl = configs.cfg1()
    b, spec, tree, fct, rec = record_factor(s, wl)
    leaf_keys = [k for k in sorted(rec) if k[0] == tree.depth]
    mid = [k for k in sorted(rec) if k[0] == 3 and not tree.boxes[k].is_leaf]
    stack_keys = [leaf_keys[0], mid[0]]
    t_keys = [leaf_keys[0], mid[0], sorted(k for k in rec if k[0] == 1)[0]]
    out.update(pack(rec, fct, "cfg1_", stack_keys, t_keys))
    f = wl.extra["rhs"]
    x = fct.solve(f)
    out["cfg1_rhs"] = f
    out["cfg1_x"] = x
    rng = np.random.default_rng(11)
    v = rng.standard_normal(fct.dim)
    out["cfg1_apply_in"] = v
    out["cfg1_apply_out"] = fct.apply(v)
    X = rng.standard_normal((fct.dim, 3))
    out["cfg1_multi_in"] = X
    out["cfg1_multi_x"] = fct.solve(X)
    # interior evaluation (skel.py:537-564) and the domain test (geometry.py:179-192)
    tg = configs.interior_targets(wl.boundary, 64, exterior=2)
    out["cfg1_targets"] = tg
    out["cfg1_in_domain"] = b.point_in_domain(tg)
    out["cfg1_interior"] = s.evaluate_interior(spec, b, x, tg[:64])
    print("cfg1 boxes", len(rec), "k/level", fct.stats["k_per_level"], "root", fct.stats["root_size"])

    # ---- mini multiply-connected case + one hole-move update
    wl = configs.mini_holes()
    b, spec, tree, fct, rec = record_factor(s, wl)
    leaf_keys = [k for k in sorted(rec) if k[0] == tree.depth]
    stack_keys = [leaf_keys[0]]
    t_keys = [leaf_keys[0], sorted(k for k in rec if k[0] == 1)[0]]
    out.update(pack(rec, fct, "mini_", stack_keys, t_keys))
    rhs = wl.extra["rhs"]
    out["mini_rhs"] = rhs
    out["mini_x"] = fct.solve(rhs)
    v = np.random.default_rng(12).standard_normal(fct.dim)
    out["mini_apply_in"] = v
    out["mini_apply_out"] = fct.apply(v)
    out["mini_corner_n"] = np.array(fct.top.n)
    tg = configs.interior_targets(wl.boundary, 64, exterior=3)
    out["mini_targets"] = tg
    out["mini_in_domain"] = b.point_in_domain(tg)
    out["mini_interior"] = s.evaluate_interior(spec, b, out["mini_x"], tg[:64])
    # hole move through the reference's own apply_perturbation/update
    nb_mine, rep_mine = apply_perturbation(wl.boundary, [MoveHole(2, translation=(0.1, -0.05))])
    b_new, rep = s.apply_perturbation(b, [s.MoveHole(2, translation=(0.1, -0.05))])
    assert np.array_equal(b_new.positions, nb_mine.positions)
    from skelsolve import skel as sk
    dirty_seen = {}
    orig_rl = sk._Compressor.run_level

    def rl(self, keys, workers, reuse=None, dirty=None, dof_map=None):
        if dirty is not None:
            dirty_seen["d"] = set(dirty)
        return orig_rl(self, keys, workers, reuse, dirty, dof_map)

    sk._Compressor.run_level = rl
    try:
        fu = s.update(fct, b_new, rep)
    finally:
        sk._Compressor.run_level = orig_rl
    out["mini_upd_dirty"] = np.array(sorted(dirty_seen["d"]), dtype=np.int64)
    out["mini_upd_x"] = fu.solve(rhs)
    print("mini boxes", len(rec), "k/level", fct.stats["k_per_level"], "n_dirty", fu.stats["n_dirty"])

    # ---- Laplace-Neumann branch (kernels.py:119-125,161-168,322-325,347-352,368-370)
    # on the cfg1 star: RHS = normal derivative of the harmonic log|x - c|, c outside
    wl = configs.cfg1()
    b, spec, tree, fct, rec = record_factor(s, wl, pde=s.LAPLACE)
    leaf_keys = [k for k in sorted(rec) if k[0] == tree.depth]
    out.update(pack(rec, fct, "lap_", [leaf_keys[0]], [leaf_keys[0]]))
    c0 = np.array([1.7, 0.4])
    d = wl.boundary.positions - c0[None, :]
    f = (d * wl.boundary.normals).sum(axis=1) / (d * d).sum(axis=1)
    out["lap_rhs"] = f
    out["lap_x"] = fct.solve(f)
    v = np.random.default_rng(13).standard_normal(fct.dim)
    out["lap_apply_in"] = v
    out["lap_apply_out"] = fct.apply(v)
    tg = configs.interior_targets(wl.boundary, 32, seed=4)
    out["lap_targets"] = tg
    out["lap_interior"] = s.evaluate_interior(spec, b, out["lap_x"], tg)
    print("laplace boxes", len(rec), "k/level", fct.stats["k_per_level"], "root", fct.stats["root_size"])
    # Laplace on the 3-hole geometry + a hole move (update path, no augmentation)
    wl = configs.mini_holes()
    b, spec, tree, fct, rec = record_factor(s, wl, pde=s.LAPLACE)
    out.update(pack(rec, fct, "lapm_", [], []))
    rhs = np.random.default_rng(14).standard_normal(fct.dim)
    out["lapm_rhs"] = rhs
    out["lapm_x"] = fct.solve(rhs)
    b_new, rep = s.apply_perturbation(b, [s.MoveHole(1, translation=(-0.08, 0.06))])
    fu = s.update(fct, b_new, rep)
    out["lapm_upd_x"] = fu.solve(rhs)
    out["lapm_upd_ndirty"] = np.array(fu.stats["n_dirty"])

    # ---- unphased cfg2: equispaced circles centred on box axes -> exact pivot
    # ties; per-box active sets, skeletons and |R_jj| for the tie-classified replay
    wl = configs.cfg2(phases=False)
    b, spec, tree, fct, rec = record_factor(s, wl)
    keys = sorted(rec)
    out["cfg2u_keys"] = np.array(keys, dtype=np.int64)
    out["cfg2u_k"] = np.array([rec[k]["k"] for k in keys], dtype=np.int64)
    for nm, fld in (("S", "S"), ("act", "active"), ("diag", "diag")):
        arrs = [np.asarray(rec[k][fld]) for k in keys]
        out[f"cfg2u_{nm}_off"] = np.concatenate([[0], np.cumsum([len(x) for x in arrs])]).astype(np.int64)
        out[f"cfg2u_{nm}"] = np.concatenate(arrs)
    out["cfg2u_root_dofs"] = np.array(fct.root_dofs, dtype=np.int64)
    out["cfg2u_x"] = fct.solve(wl.extra["rhs"])
    print("cfg2 unphased boxes", len(rec), "k/level", fct.stats["k_per_level"])

    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **{k: np.asarray(v) for k, v in out.items()})
    print("wrote", path, os.path.getsize(path) // 1024, "KiB")


if __name__ == "__main__":
    main()
