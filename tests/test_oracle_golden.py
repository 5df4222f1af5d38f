"""Pin the CPU oracle against fixtures recorded from the reference itself."""

import numpy as np
import pytest

from oracle import skel_oracle as O
from paper_2001_11619_b200 import configs


def _boxes(g, prefix):
    keys = [tuple(k) for k in g[prefix + "keys"]]
    so, S = g[prefix + "S_off"], g[prefix + "S"]
    ao, act = g[prefix + "act_off"], g[prefix + "act"]
    fo, far = g[prefix + "far_off"], g[prefix + "far"]
    out = {}
    for i, k in enumerate(keys):
        out[k] = dict(S=S[so[i]:so[i + 1]], act=act[ao[i]:ao[i + 1]], far=far[fo[i]:fo[i + 1]],
                      k=int(g[prefix + "k"][i]))
    return out


def test_kat_id(golden):
    qr = O.QRID(np.array([[1.0, 2.0], [2.0, 4.0]]))
    S, R, T = qr.split(qr.rank(1e-10))
    assert list(S) == list(golden["kat_rank1_S"]) == [1]
    assert np.array_equal(T, golden["kat_rank1_T"])
    qr = O.QRID(golden["kat_cluster_A"])
    S, R, T = qr.split(qr.rank(1e-10))
    assert len(S) == 8
    assert np.array_equal(S, golden["kat_cluster_S"])
    assert np.array_equal(T, golden["kat_cluster_T"])


@pytest.mark.parametrize("name,builder,pde", [("cfg1_", configs.cfg1, O.STOKES),
                                              ("mini_", configs.mini_holes, O.STOKES),
                                              ("lap_", configs.cfg1, O.LAPLACE),
                                              ("lapm_", configs.mini_holes, O.LAPLACE)])
def test_oracle_matches_reference(golden, name, builder, pde):
    wl = builder()
    rec = {}
    f = O.factor_full(wl.boundary, wl.leaf_cap, wl.tol, wl.proxy_count, wl.proxy_factor, record=rec,
                      pde=pde)
    ref = _boxes(golden, name)
    assert set(ref) == set(f.boxes)
    for k, r in ref.items():
        bo = f.boxes[k]
        assert np.array_equal(bo.dofs, r["act"]), k
        assert np.array_equal(rec[k]["far"], r["far"]), k
        assert len(bo.S) == r["k"], k
        assert np.array_equal(bo.S, r["S"]), k
    i = 0
    while name + f"stack{i}_key" in golden.files:
        k = tuple(golden[name + f"stack{i}_key"])
        assert np.array_equal(rec[k]["stack"], golden[name + f"stack{i}"]), k
        i += 1
    i = 0
    while name + f"T{i}_key" in golden.files:
        k = tuple(golden[name + f"T{i}_key"])
        np.testing.assert_allclose(rec[k]["T"], golden[name + f"T{i}"], rtol=0, atol=1e-12)
        i += 1
    assert np.array_equal(f.root_dofs, golden[name + "root_dofs"])
    kpl = {int(l): int(v) for l, v in golden[name + "k_per_level"]}
    assert f.stats["k_per_level"] == kpl
    x = f.solve(golden[name + "rhs"])
    xr = golden[name + "x"]
    assert np.linalg.norm(x - xr) / np.linalg.norm(xr) < 1e-13
    if name + "apply_in" in golden.files:
        y = f.apply(golden[name + "apply_in"])
        yr = golden[name + "apply_out"]
        assert np.linalg.norm(y - yr) / np.linalg.norm(yr) < 1e-13


def test_oracle_laplace_update_and_interior(golden):
    """Laplace-Neumann: hole-move update on the 3-hole geometry and interior
    evaluation u = -S mu against the reference (kernels.py:171-198)."""
    from paper_2001_11619_b200.geometry import MoveHole, apply_perturbation
    wl = configs.mini_holes()
    f = O.factor_full(wl.boundary, wl.leaf_cap, wl.tol, wl.proxy_count, wl.proxy_factor, pde=O.LAPLACE)
    nb, rep = apply_perturbation(wl.boundary, [MoveHole(1, translation=(-0.08, 0.06))])
    fu = O.update(f, nb, rep)
    assert fu.stats["n_dirty"] == int(golden["lapm_upd_ndirty"])
    x = fu.solve(golden["lapm_rhs"])
    assert np.linalg.norm(x - golden["lapm_upd_x"]) / np.linalg.norm(golden["lapm_upd_x"]) < 1e-13
    wl = configs.cfg1()
    u = O.evaluate_interior(wl.boundary, golden["lap_x"], golden["lap_targets"], pde=O.LAPLACE)
    ref = golden["lap_interior"]
    assert np.max(np.abs(u - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_oracle_update_dirty_set(golden):
    from paper_2001_11619_b200.geometry import MoveHole, apply_perturbation
    wl = configs.mini_holes()
    f = O.factor_full(wl.boundary, wl.leaf_cap, wl.tol, wl.proxy_count, wl.proxy_factor)
    nb, rep = apply_perturbation(wl.boundary, [MoveHole(2, translation=(0.1, -0.05))])
    fu = O.update(f, nb, rep)
    ref_dirty = {tuple(k) for k in golden["mini_upd_dirty"]}
    assert fu.stats["dirty"] == ref_dirty
    x = fu.solve(golden["mini_rhs"])
    xr = golden["mini_upd_x"]
    assert np.linalg.norm(x - xr) / np.linalg.norm(xr) < 1e-13
    # update == refactor on the new geometry (reference claim skel.py:459-465)
    fr = O.factor_full(nb, wl.leaf_cap, wl.tol, wl.proxy_count, wl.proxy_factor)
    assert np.array_equal(fr.solve(golden["mini_rhs"]), x)


@pytest.mark.parametrize("name,builder", [("cfg1_", configs.cfg1), ("mini_", configs.mini_holes)])
def test_oracle_interior_evaluation_vs_reference(golden, name, builder):
    """evaluate_interior / point_in_domain restatements vs the reference's outputs
    (skel.py:537-564, geometry.py:179-199) on seeded targets."""
    wl = builder()
    tg = golden[name + "targets"]
    assert np.array_equal(O.point_in_domain(wl.boundary, tg), golden[name + "in_domain"])
    u = O.evaluate_interior(wl.boundary, golden[name + "x"], tg[:64])
    ref = golden[name + "interior"]
    assert np.max(np.abs(u - ref)) <= 1e-12 * np.max(np.abs(ref))
    with pytest.raises(ValueError):
        O.evaluate_interior(wl.boundary, golden[name + "x"], tg)


def test_oracle_unphased_cfg2_vs_reference(golden):
    """Tie-rich fixture: on unphased cfg2 (exact pivot ties from equispaced
    circles) the oracle, with the reference's LAPACK calls, reproduces every
    per-box skeleton and the solution bitwise."""
    wl = configs.cfg2(phases=False)
    f = O.factor_full(wl.boundary, wl.leaf_cap, wl.tol, wl.proxy_count, wl.proxy_factor)
    keys = [tuple(k) for k in golden["cfg2u_keys"]]
    so, S = golden["cfg2u_S_off"], golden["cfg2u_S"]
    assert sorted(f.boxes) == sorted(keys)
    for i, k in enumerate(keys):
        assert np.array_equal(f.boxes[k].S, S[so[i]:so[i + 1]]), k
    assert np.array_equal(f.solve(wl.extra["rhs"]), golden["cfg2u_x"])


@pytest.mark.parametrize("nm,builder", [("pzm", configs.mini_holes), ("pz1", configs.cfg1)])
def test_oracle_propagate_zeros_matches_reference(nm, builder):
    """propagate_zeros=True (skel.py:267-270, 354-361): the oracle's sequential
    mode picks the reference's skeletons box for box and solves to its bits."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden_edits.npz"))
    wl = builder()
    f = O.factor_full(wl.boundary, wl.leaf_cap, wl.tol, wl.proxy_count, wl.proxy_factor,
                      propagate_zeros=True)
    keys = [tuple(int(v) for v in k) for k in g[nm + "_keys"]]
    off = g[nm + "_skel_off"]
    assert set(keys) == set(f.boxes)
    for i, k in enumerate(keys):
        assert np.array_equal(f.boxes[k].skel, g[nm + "_skel"][off[i]:off[i + 1]]), k
    assert np.array_equal(f.solve(wl.extra["rhs"]), g[nm + "_x"])
