"""Host-side logic (no GPU): quadtree, far-field lists, proxy rings, dirty sets."""

import numpy as np
import pytest

from oracle import skel_oracle as O
from paper_2001_11619_b200 import configs, skel
from paper_2001_11619_b200.geometry import MoveHole, apply_perturbation
from paper_2001_11619_b200.tree import build_tree, dirty_set, refit_tree


@pytest.mark.parametrize("builder", [configs.cfg1, configs.mini_holes])
def test_tree_matches_oracle(builder):
    wl = builder()
    t = build_tree(wl.boundary.positions, wl.leaf_cap)
    ot = O.QTree(wl.boundary.positions, wl.leaf_cap)
    assert t.levels == ot.levels
    for i in range(len(t.lev)):
        key = t.key(i)
        ob = ot.boxes[key]
        assert np.array_equal(t.center[i], ob.center)
        assert t.hw[i] == ob.hw
        assert np.array_equal(t.nodes_of(i), ob.nodes)
        assert [t.key(c) for c in t.children_of(i)] == ob.kids
        assert t.colleagues(key) == ot.neighbours(key)


def _boxes(g, prefix):
    keys = [tuple(k) for k in g[prefix + "keys"]]
    out = {}
    for i, k in enumerate(keys):
        sl = lambda a: g[prefix + a][g[prefix + a + "_off"][i]:g[prefix + a + "_off"][i + 1]]
        out[k] = dict(act=sl("act"), far=sl("far"), S=g[prefix + "S"][g[prefix + "S_off"][i]:g[prefix + "S_off"][i + 1]])
    return out


@pytest.mark.parametrize("name,builder", [("cfg1_", configs.cfg1), ("mini_", configs.mini_holes)])
def test_far_lists_and_proxies_match_reference(golden, name, builder):
    """Replay the reference's active sets and check F_int lists bitwise."""
    wl = builder()
    t = build_tree(wl.boundary.positions, wl.leaf_cap)
    ctx = skel._Ctx(skel.SystemSpec(), wl.boundary, t, wl.tol, wl.proxy_count, wl.proxy_factor)
    ref = _boxes(golden, name)
    act_of = {}
    for i in range(len(t.lev)):
        key = t.key(i)
        if key in ref:
            act_of[i] = ref[key]["act"]
        elif t.is_leaf[i]:
            act_of[i] = (2 * t.nodes_of(i)[:, None] + np.arange(2)).ravel()
    for lev in range(t.depth, 0, -1):
        idx = t.level_indices(lev)
        off, F = ctx.far_lists(idx, skel.ActStore.replay(t, act_of))
        for bi, i in enumerate(idx):
            assert np.array_equal(F[off[bi]:off[bi + 1]], ref[t.key(i)]["far"]), t.key(i)
        pts, pn, pw = ctx.proxies(idx)
        for bi, i in enumerate(idx):
            rp = O.proxy_radius(t.hw[i], wl.proxy_factor)
            p2, w2 = O.proxy_ring(t.center[i], rp, wl.proxy_count)
            assert np.array_equal(pts[bi], p2)
            assert np.array_equal(pn[bi], O.proxy_normals(p2))
            assert pw[bi] == w2[0]


def test_dirty_set_matches_reference(golden):
    wl = configs.mini_holes()
    t = build_tree(wl.boundary.positions, wl.leaf_cap)
    nb, rep = apply_perturbation(wl.boundary, [MoveHole(2, translation=(0.1, -0.05))])
    t2 = refit_tree(t, nb.positions)
    d = dirty_set(t, t2, nb, rep, wl.proxy_factor)
    assert d == {tuple(k) for k in golden["mini_upd_dirty"]}


def test_cfg4_dirty_sets_match_oracle():
    wl = configs.cfg2()
    t = build_tree(wl.boundary.positions, wl.leaf_cap)
    ot = O.QTree(wl.boundary.positions, wl.leaf_cap)
    for h, d, nb, rep in configs.hole_move_sequence(wl.boundary, 3):
        t2 = refit_tree(t, nb.positions)
        ot2 = O.QTree(nb.positions, wl.leaf_cap, (ot.root_center, ot.root_hw))
        mine = dirty_set(t, t2, nb, rep, wl.proxy_factor)
        ref = O.dirty_set(ot, ot2, nb, rep, wl.proxy_factor)
        assert mine == ref
        t, ot = t2, ot2


def test_native_far_lists_and_proxies_match_numpy():
    """Native host runtime (csrc/host.cpp) == the NumPy restatement, bitwise,
    on every level of cfg2 with synthetic (seeded random) skeletons."""
    wl = configs.cfg2()
    b = wl.boundary
    t = build_tree(b.positions, wl.leaf_cap)
    rng = np.random.default_rng(7)
    store = skel.ActStore(t)
    for lev in range(t.depth, 0, -1):
        idx = t.level_indices(lev)
        store.set_internal(t, idx)
        act_off, act = store.acts(idx)
        k = np.array([rng.integers(0, n + 1) for n in np.diff(act_off)], np.int64)
        perm = np.concatenate([rng.permutation(n) for n in np.diff(act_off)]).astype(np.int32)
        store.set_skel(idx, act_off, act, perm, k)
    ctx = skel._Ctx(skel.SystemSpec(), b, t, wl.tol, wl.proxy_count, wl.proxy_factor)
    for lev in range(t.depth, 0, -1):
        idx = t.level_indices(lev)
        off, F = ctx.far_lists(idx, store)
        off2, F2 = ctx.far_lists_np(idx, store)
        assert np.array_equal(off, off2) and np.array_equal(F, F2)
        for a, a2 in zip(ctx.proxies(idx), ctx.proxies_np(idx)):
            assert np.array_equal(a, a2)


@pytest.mark.parametrize("name", ["cfg1", "mini", "cfg2"])
def test_native_tree_matches_numpy(name):
    """Native quadtree build (csrc/host.cpp) == the NumPy restatement."""
    from paper_2001_11619_b200.tree import build_tree_np
    wl = configs.by_name(name)
    a = build_tree(wl.boundary.positions, wl.leaf_cap)
    b = build_tree_np(wl.boundary.positions, wl.leaf_cap)
    for f in ("level_start", "lev", "ix", "iy", "parent", "children", "nchild", "node_start",
              "node_cnt", "neighbors", "node_leaf", "is_leaf", "center", "hw"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert all(np.array_equal(x, y) for x, y in zip(a.level_nodes, b.level_nodes))


def test_native_dirty_sets_match_numpy():
    from paper_2001_11619_b200.tree import dirty_set_np
    wl = configs.cfg2()
    b = wl.boundary
    t = build_tree(b.positions, wl.leaf_cap)
    for h, d, nb, rep in configs.hole_move_sequence(b, 6):
        tn = refit_tree(t, nb.positions)
        assert dirty_set(t, tn, nb, rep, wl.proxy_factor) == dirty_set_np(t, tn, nb, rep, wl.proxy_factor)
        t = tn


def test_native_leaf_actives_match_numpy():
    """ActStore leaf actives (skel.py:243-249): the native host runtime on a
    natively built tree equals the NumPy path on the NumPy-built tree."""
    from paper_2001_11619_b200.skel import ActStore
    from paper_2001_11619_b200.tree import build_tree_np
    for wl in (configs.cfg1(), configs.mini_holes()):
        b = wl.boundary
        tn, tp = build_tree(b.positions, wl.leaf_cap), build_tree_np(b.positions, wl.leaf_cap)
        for dpn in (1, 2):
            a, r = ActStore(tn, dpn=dpn), ActStore(tp, dpn=dpn)
            assert a.fill == r.fill
            assert np.array_equal(a.big[:a.fill], r.big[:r.fill])
            assert np.array_equal(a.a_start, r.a_start) and np.array_equal(a.a_len, r.a_len)


def _edit_cases():
    """(name, new boundary, report) for the DeleteHole / AddHole fixtures recorded
    from the reference (tests/golden/make_golden_edits.py)."""
    import os
    from paper_2001_11619_b200.geometry import AddHole, Curve, DeleteHole, HOLE
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden_edits.npz"))
    b = configs.mini_holes().boundary
    nb_d, rep_d = apply_perturbation(b, [DeleteHole(2)])
    nodes = g["add_nodes"]
    rad = float(np.sqrt(((nodes - nodes.mean(axis=0)) ** 2).sum(axis=1)).max())
    hole = Curve(nodes, g["add_weights"], g["add_normals"], g["add_curvatures"], HOLE, rad)
    nb_a, rep_a = apply_perturbation(b, [AddHole(hole)])
    return g, b, (("del", nb_d, rep_d), ("add", nb_a, rep_a))


def test_add_delete_hole_reports_and_dirty_sets_match_reference():
    """Non-DOF-preserving edits: node map, modified-node lists and the dirty set
    (reference geometry.py:328-390, skel.py:476-491) equal the reference's."""
    g, b, cases = _edit_cases()
    wl = configs.mini_holes()
    t_old = build_tree(b.positions, wl.leaf_cap)
    assert np.array_equal(cases[1][1].positions, g["add_positions"])
    assert np.array_equal(cases[1][1].hole_centers, g["add_hole_centers"])
    for name, nb, rep in cases:
        assert np.array_equal(rep.old_to_new, g[f"{name}_old_to_new"])
        assert np.array_equal(rep.modified_nodes_old, g[f"{name}_mod_old"])
        assert np.array_equal(rep.modified_nodes_new, g[f"{name}_mod_new"])
        t_new = refit_tree(t_old, nb.positions)
        want = {tuple(int(v) for v in k) for k in g[f"{name}_dirty"]}
        assert dirty_set(t_old, t_new, nb, rep, wl.proxy_factor) == want
