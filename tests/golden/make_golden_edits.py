"""Golden fixtures for non-DOF-preserving edits (DeleteHole / AddHole), recorded by
running the UNMODIFIED reference ``skelsolve`` through the same harness shim as
``make_golden.py`` (build container only, needs /root/reference):

    python tests/golden/make_golden_edits.py

On the 3-hole mini case: the reference's ``apply_perturbation`` + ``update`` for
(a) DeleteHole(2) and (b) AddHole (a spline-fitted circle; its discretised node
arrays are stored so that the same hole can be added on the GPU side), with the
dirty set the reference marks, its node map, and the updated solutions.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from make_golden import load_reference, to_ref_boundary  # noqa: E402
from paper_2001_11619_b200 import configs  # noqa: E402


def run_update(s, fct, b_new, rep):
    from skelsolve import skel as sk
    seen = {}
    orig = sk._Compressor.run_level

    def rl(self, keys, workers, reuse=None, dirty=None, dof_map=None):
        if dirty is not None:
            seen["d"] = set(dirty)
        return orig(self, keys, workers, reuse, dirty, dof_map)

    sk._Compressor.run_level = rl
    try:
        fu = s.update(fct, b_new, rep)
    finally:
        sk._Compressor.run_level = orig
    return fu, np.array(sorted(seen["d"]), dtype=np.int64)


def main():
    s = load_reference()
    out = {}
    wl = configs.mini_holes()
    b = to_ref_boundary(s, wl.boundary)
    spec = s.SystemSpec(s.STOKES)
    tree = s.build_tree(b.positions, leaf_cap=wl.leaf_cap)
    fct = s.factor(spec, b, tree, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
    rng = np.random.default_rng(31)

    # (a) delete hole 2
    b_del, rep = s.apply_perturbation(b, [s.DeleteHole(2)])
    fu, dirty = run_update(s, fct, b_del, rep)
    rhs = np.concatenate([rng.standard_normal(2 * b_del.n_nodes), np.zeros(3 * (len(b_del.curves) - 1))])
    out["del_old_to_new"] = rep.old_to_new
    out["del_mod_old"], out["del_mod_new"] = rep.modified_nodes_old, rep.modified_nodes_new
    out["del_dirty"] = dirty
    out["del_rhs"], out["del_x"] = rhs, fu.solve(rhs)
    out["del_n_dirty"] = np.array(fu.stats["n_dirty"])
    ff = s.factor(spec, b_del, s.build_tree(b_del.positions, leaf_cap=wl.leaf_cap,
                                           root_box=(tree.root_center, tree.root_half_width)),
                  wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
    out["del_x_refactor"] = ff.solve(rhs)

    # (b) add a hole (spline-fitted circle of radius 0.35 centred where it overlaps nothing)
    th = 2 * np.pi * np.arange(24) / 24
    knots = np.stack([0.35 * np.cos(-th), 0.35 * np.sin(-th)], axis=1) + np.array([-1.4, -0.9])
    cspec = s.CurveSpec(knots, 192, "hole")
    b_add, rep = s.apply_perturbation(b, [s.AddHole(cspec)])
    fu, dirty = run_update(s, fct, b_add, rep)
    c = b_add.curves[-1]
    out["add_nodes"], out["add_weights"] = c.nodes, c.weights
    out["add_normals"], out["add_curvatures"] = c.normals, c.curvatures
    rhs = np.concatenate([rng.standard_normal(2 * b_add.n_nodes), np.zeros(3 * (len(b_add.curves) - 1))])
    out["add_old_to_new"] = rep.old_to_new
    out["add_mod_old"], out["add_mod_new"] = rep.modified_nodes_old, rep.modified_nodes_new
    out["add_dirty"] = dirty
    out["add_rhs"], out["add_x"] = rhs, fu.solve(rhs)
    out["add_positions"] = b_add.positions
    out["add_hole_centers"] = b_add.hole_centers
    # (c) the sequential validation mode propagate_zeros=True (skel.py:267-270, 354-361)
    for nm, w in (("pzm", configs.mini_holes()), ("pz1", configs.cfg1())):
        rb = to_ref_boundary(s, w.boundary)
        tr = s.build_tree(rb.positions, leaf_cap=w.leaf_cap)
        fz = s.factor(spec, rb, tr, w.tol, proxy_count=w.proxy_count, proxy_factor=w.proxy_factor,
                      propagate_zeros=True)
        keys = sorted(fz.factors)
        out[nm + "_keys"] = np.array(keys, dtype=np.int64)
        sk_all = [np.asarray(fz.factors[k].skel_dofs) for k in keys]
        out[nm + "_skel_off"] = np.concatenate([[0], np.cumsum([len(x) for x in sk_all])]).astype(np.int64)
        out[nm + "_skel"] = np.concatenate(sk_all).astype(np.int64)
        out[nm + "_x"] = fz.solve(w.extra["rhs"])
        f0 = s.factor(spec, rb, tr, w.tol, proxy_count=w.proxy_count, proxy_factor=w.proxy_factor)
        ndiff = sum(len(fz.factors[k].S_loc) != len(f0.factors[k].S_loc) for k in keys)
        print(nm, "propagate_zeros: boxes with a different rank than the default mode:", ndiff, "of", len(keys))
    print("delete: dirty", len(out["del_dirty"]), "add: dirty", len(out["add_dirty"]),
          "update vs refactor (reference, delete)",
          np.linalg.norm(out["del_x"] - out["del_x_refactor"]) / np.linalg.norm(out["del_x"]))
    path = os.path.join(HERE, "reference_golden_edits.npz")
    np.savez_compressed(path, **{k: np.asarray(v) for k, v in out.items()})
    print("wrote", path, os.path.getsize(path) // 1024, "KiB")


if __name__ == "__main__":
    main()
