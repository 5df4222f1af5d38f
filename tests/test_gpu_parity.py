"""End-to-end parity on a B200 against the reference fixtures and the CPU oracle:
identical skeletons per box, solve/apply within 10*eps (relative 2-norm)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import skel_oracle as O  # noqa: E402
from paper_2001_11619_b200 import SystemSpec, build_tree, configs, factor, update  # noqa: E402
from paper_2001_11619_b200 import skel  # noqa: E402
from paper_2001_11619_b200.geometry import MoveHole, apply_perturbation  # noqa: E402


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def _factor(wl):
    t = build_tree(wl.boundary.positions, wl.leaf_cap)
    return factor(SystemSpec(), wl.boundary, t, wl.tol, proxy_count=wl.proxy_count,
                  proxy_factor=wl.proxy_factor)


@pytest.mark.parametrize("name,builder", [("cfg1_", configs.cfg1), ("mini_", configs.mini_holes)])
def test_factor_solve_apply_vs_reference(golden, name, builder):
    wl = builder()
    f = _factor(wl)
    keys = [tuple(k) for k in golden[name + "keys"]]
    so, S = golden[name + "S_off"], golden[name + "S"]
    bad = []
    for i, k in enumerate(keys):
        if not np.array_equal(f.factors[k].S_loc, S[so[i]:so[i + 1]]):
            bad.append(k)
    assert not bad, bad
    assert np.array_equal(f.root_dofs, golden[name + "root_dofs"])
    kpl = {int(l): int(v) for l, v in golden[name + "k_per_level"]}
    assert f.stats["k_per_level"] == kpl
    x = f.solve(golden[name + "rhs"])
    assert _rel(x, golden[name + "x"]) <= 10 * wl.tol
    y = f.apply(golden[name + "apply_in"])
    assert _rel(y, golden[name + "apply_out"]) <= 10 * wl.tol


def test_multi_rhs_matches_columns(golden):
    wl = configs.cfg1()
    f = _factor(wl)
    X = golden["cfg1_multi_in"]
    got = f.solve(X)
    assert got.shape == X.shape
    assert _rel(got, golden["cfg1_multi_x"]) <= 10 * wl.tol
    for j in range(X.shape[1]):
        assert _rel(got[:, j], f.solve(X[:, j])) <= 1e-13


def test_cfg1_against_dense_and_exact_field():
    """Independent oracles: dense LU of the full system and the exact Stokeslet field."""
    wl = configs.cfg1()
    f = _factor(wl)
    x = f.solve(wl.extra["rhs"])
    A = O.dense_system(wl.boundary)
    xd = np.linalg.solve(A, wl.extra["rhs"])
    assert _rel(x, xd) < 1e-8
    r = A @ x - wl.extra["rhs"]
    assert np.linalg.norm(r) / np.linalg.norm(wl.extra["rhs"]) < 1e-8


def test_update_equals_refactor_and_reference(golden):
    wl = configs.mini_holes()
    f = _factor(wl)
    nb, rep = apply_perturbation(wl.boundary, [MoveHole(2, translation=(0.1, -0.05))])
    fu = update(f, nb, rep)
    assert fu.stats["dirty"] == {tuple(k) for k in golden["mini_upd_dirty"]}
    rhs = golden["mini_rhs"]
    xu = fu.solve(rhs)
    assert _rel(xu, golden["mini_upd_x"]) <= 10 * wl.tol
    t2 = build_tree(nb.positions, wl.leaf_cap, root_box=(f.tree.root_center, f.tree.root_half_width))
    fr = factor(SystemSpec(), nb, t2, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
    assert np.array_equal(fr.solve(rhs), xu)       # bitwise: update == refactor


def test_cfg2_against_oracle():
    wl = configs.cfg2()
    f = _factor(wl)
    ref = O.factor_full(wl.boundary, wl.leaf_cap, wl.tol, wl.proxy_count, wl.proxy_factor)
    same = sum(np.array_equal(f.factors[k].skel_dofs, ref.boxes[k].skel) for k in ref.boxes)
    rhs = wl.extra["rhs"]
    x = f.solve(rhs)
    xr = ref.solve(rhs)
    err = _rel(x, xr)
    print(f"cfg2: {same}/{len(ref.boxes)} identical skeletons; solve rel diff {err:.3e}")
    assert same == len(ref.boxes)
    assert err <= 10 * wl.tol


@pytest.mark.parametrize("builder", [configs.cfg1, configs.mini_holes])
def test_system_matvec_vs_oracle(builder):
    """GPU direct-summation operator vs the oracle's exact_matvec (kernels.py:393-414)."""
    from paper_2001_11619_b200 import system_matvec
    wl = builder()
    b = wl.boundary
    dim = 2 * b.n_nodes + 3 * b.n_holes
    X = np.random.default_rng(3).standard_normal((dim, 5))
    Y = system_matvec(SystemSpec(), b, X)
    for j in range(5):
        ref = O.exact_matvec(b, X[:, j])
        assert _rel(Y[:, j], ref) < 1e-12


@pytest.mark.slow
def test_cfg4_update_sequence_vs_oracle():
    """cfg4 regime (hole moves on cfg2) on the default path (native engine):
    the GPU dirty set equals the reference rules' (oracle) at every step;
    update == refactor bitwise while the reference rules guarantee it (first 10
    moves here), and to rounding afterwards -- the reference's own update
    differs from its refactor by ~6e-15 from move 15 on (a coarse-leaf split
    reorders a clean box's far-field rows; test_cfg4_hundred_moves)."""
    wl = configs.cfg2()
    b = wl.boundary
    f = _factor(wl)
    of = O.factor_full(b, wl.leaf_cap, wl.tol, wl.proxy_count, wl.proxy_factor)
    rhs = wl.extra["rhs"]
    cur, ocur = f, of
    for s, (h, d, nb, rep) in enumerate(configs.hole_move_sequence(b, 12)):
        cur = update(cur, nb, rep)
        ocur = O.update(ocur, nb, rep)
        assert cur.stats["dirty"] == ocur.stats["dirty"], s
        if (s + 1) % 6 == 0:
            t2 = build_tree(nb.positions, wl.leaf_cap, root_box=(f.tree.root_center, f.tree.root_half_width))
            fr = factor(SystemSpec(), nb, t2, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
            xu, xr = cur.solve(rhs), fr.solve(rhs)
            if s + 1 <= 10:
                assert np.array_equal(xu, xr)
            assert _rel(xu, xr) < 1e-13
            assert _rel(xu, ocur.solve(rhs)) <= 10 * wl.tol


def test_migration_path(monkeypatch):
    """Exercise the R -> S migration rule (skel.py:317-330) with a raised
    pivot-ratio floor.  The floor decision itself compares X_RR pivot ratios,
    which differ by a few percent between LU implementations near the floor, so
    the test checks the mechanism: migrated boxes get larger ranks (the next
    pivots of the same QRCP), every box with equal rank on both sides has the
    same skeleton as the oracle, and the solution stays within 10 eps."""
    from paper_2001_11619_b200 import skel as S
    wl = configs.mini_holes()
    f0 = _factor(wl)
    floor = 0.0172
    monkeypatch.setattr(S, "PIVOT_RATIO_FLOOR", floor)
    monkeypatch.setattr(O, "PIVOT_FLOOR", floor)
    ref = O.factor_full(wl.boundary, wl.leaf_cap, wl.tol, wl.proxy_count, wl.proxy_factor)
    f = _factor(wl)
    grew = [k for k in ref.boxes if len(f.factors[k].S_loc) > len(f0.factors[k].S_loc)]
    assert grew, "no migration on the GPU"
    for k in grew:
        k0 = len(f0.factors[k].S_loc)
        assert np.array_equal(f.factors[k].S_loc[:k0], f0.factors[k].S_loc)   # same pivot sequence
    same_k = [k for k in ref.boxes if len(f.factors[k].S_loc) == len(ref.boxes[k].S)
              and np.array_equal(f.factors[k].b_dofs, ref.boxes[k].dofs)]
    assert len(same_k) >= len(ref.boxes) - 4
    for k in same_k:
        assert np.array_equal(f.factors[k].S_loc, ref.boxes[k].S), k
    rhs = wl.extra["rhs"]
    assert _rel(f.solve(rhs), ref.solve(rhs)) <= 10 * wl.tol


def test_engine_matches_python_level_loop(monkeypatch):
    """The native level engine (csrc/engine.cu) and the single-threaded Python
    level loop produce bitwise identical factorizations and updates (same host
    functions and kernels; regression test for the LU pivot read/swap race that
    only showed under the engine's concurrency)."""
    wl = configs.mini_holes()
    b = wl.boundary
    rhs = np.random.default_rng(11).standard_normal(2 * b.n_nodes + 3 * b.n_holes)
    nb, rep = apply_perturbation(b, [MoveHole(1, translation=(0.05, 0.02))])
    out = {}
    for on in (False, True):
        monkeypatch.setattr(skel, "_ENGINE_ON", on)
        f = _factor(wl)
        fu = update(f, nb, rep)
        out[on] = (f.solve(rhs), fu.solve(rhs),
                   {k: f.factors[k].skel_dofs for k in f.factors.keys()})
    assert np.array_equal(out[False][0], out[True][0])
    assert np.array_equal(out[False][1], out[True][1])
    assert all(np.array_equal(out[False][2][k], out[True][2][k]) for k in out[False][2])


def test_native_driver_matches_python_consumer(monkeypatch):
    """The native level driver (csrc/engine.cu skb_drv_run: merge, layout, Schur
    stage, sweeps, level lists in C++) and the Python consumer loop over the
    same engine give bitwise identical factorizations and update chains on
    cfg2, and the same per-level arrays (skeleton / redundant lists, hole
    columns, ranks)."""
    wl = configs.cfg2()
    b = wl.boundary
    rhs = wl.extra["rhs"]
    seq = configs.hole_move_sequence(b, 3)
    out = {}
    for native in (False, True):
        monkeypatch.setattr(skel, "_NATIVE_ON", native)
        f = _factor(wl)
        xs = [f.solve(rhs)]
        lv = [(L.lev, L.k.copy(), L.sd.copy(), L.rd.copy(), L.cols.copy(), L.cols_off.copy()) for L in f.levels]
        cur = f
        for (h, d, nb, rep) in seq:
            cur = update(cur, nb, rep)
            xs.append(cur.solve(rhs))
        lv += [(L.lev, L.k.copy(), L.sd.copy(), L.rd.copy(), L.cols.copy(), L.cols_off.copy()) for L in cur.levels]
        out[native] = (xs, lv, cur.stats["dirty"])
    for a, c in zip(out[False][0], out[True][0]):
        assert np.array_equal(a, c)
    assert out[False][2] == out[True][2]
    for la, lc in zip(out[False][1], out[True][1]):
        assert la[0] == lc[0]
        for x, y in zip(la[1:], lc[1:]):
            assert np.array_equal(x, y)


def test_engine_repeatable_cfg2():
    """Repeated engine factorizations of cfg2 are bitwise identical."""
    wl = configs.cfg2()
    xs = []
    for _ in range(3):
        f = _factor(wl)
        xs.append(f.solve(wl.extra["rhs"]))
        del f
    assert np.array_equal(xs[0], xs[1]) and np.array_equal(xs[0], xs[2])


def test_update_chains_repeatable(monkeypatch):
    """Identical hole-move update chains give bitwise equal solves at every
    step, on the native engine (unbounded run-ahead, the default, and one
    level of run-ahead) and on the Python level loop.  Regression test for the
    cluster-QRCP races (k_qrcp2 MODE 1: pivot candidates now double-buffered
    by step parity, the deferred last R(i, p) written before the write-back)
    that made ~5 % of engine update steps differ run to run."""
    wl = configs.cfg2()
    b = wl.boundary
    rhs = wl.extra["rhs"]
    seq = configs.hole_move_sequence(b, 4)
    base = _factor(wl)

    def chains(n):
        runs = []
        for _ in range(n):
            cur = base
            xs = []
            for (h, d, nb, rep) in seq:
                cur = update(cur, nb, rep)
                xs.append(cur.solve(rhs))
            runs.append(xs)
            del cur
        return runs

    ref = None
    for engine, lead in ((True, None), (True, "1"), (False, None)):
        monkeypatch.setattr(skel, "_ENGINE_ON", engine)
        if lead is None:
            monkeypatch.delenv("SKB_ENGINE_LEAD", raising=False)
        else:
            monkeypatch.setenv("SKB_ENGINE_LEAD", lead)
        runs = chains(4 if engine and lead is None else 2)
        ref = runs[0] if ref is None else ref
        for xs in runs:
            for s, (a, c) in enumerate(zip(ref, xs)):
                assert np.array_equal(a, c), (engine, lead, s)


def test_noop_and_coarse_only_updates():
    """Updates whose deepest dirty level is shallow (none at all, or only
    coarse boxes) complete on the engine (no run-ahead stall: levels without
    boxes to compress count as acknowledged) and equal the refactor."""
    from paper_2001_11619_b200.geometry import PerturbationReport
    from paper_2001_11619_b200.tree import dirty_mask
    wl = configs.cfg1()
    b = wl.boundary
    f = _factor(wl)
    rhs = wl.extra["rhs"]
    x0 = f.solve(rhs)
    nb, rep = apply_perturbation(b, [])                       # no-op edit
    fu = update(f, nb, rep)
    assert fu.stats["n_dirty"] == 0
    assert np.array_equal(fu.solve(rhs), x0)
    # a "modified" node (unchanged position) in a coarse leaf: only shallow boxes dirty
    t = f.tree
    found = None
    for leaf in np.flatnonzero(t.is_leaf):
        if t.lev[leaf] > t.depth - 2 or t.node_cnt[leaf] == 0:
            continue
        node = int(t.level_nodes[t.lev[leaf]][t.node_start[leaf]])
        r = PerturbationReport(np.array([node]), np.array([node]), np.arange(b.n_nodes), b.positions)
        m = dirty_mask(t, t, b, r, f.proxy_factor)
        if m.any() and t.lev[np.flatnonzero(m)].max() <= t.depth - 2:
            found = r
            break
    assert found is not None
    fu = update(f, b, found)
    assert 0 < fu.stats["n_dirty"]
    assert np.array_equal(fu.solve(rhs), x0)


@pytest.mark.parametrize("name,builder", [("cfg1_", configs.cfg1), ("mini_", configs.mini_holes)])
def test_evaluate_interior_vs_reference(golden, name, builder):
    """Interior evaluation (reference evaluate_interior skel.py:537-564) on the
    GPU from the reference's own solution: within 1e-12 of the reference's field;
    point_in_domain (geometry.py:179-192) identical; exterior targets rejected."""
    from paper_2001_11619_b200 import evaluate_interior, point_in_domain
    wl = builder()
    b = wl.boundary
    tg = golden[name + "targets"]
    assert np.array_equal(point_in_domain(b, tg), golden[name + "in_domain"])
    assert np.array_equal(b.point_in_domain(tg), golden[name + "in_domain"])
    u = evaluate_interior(SystemSpec(), b, golden[name + "x"], tg[:64])
    ref = golden[name + "interior"]
    assert u.shape == ref.shape
    assert np.max(np.abs(u - ref)) <= 1e-12 * np.max(np.abs(ref))
    with pytest.raises(ValueError):
        evaluate_interior(SystemSpec(), b, golden[name + "x"], tg)
    # multi-column solutions: column-wise equal to the single-column result
    X = np.stack([golden[name + "x"], 2.0 * golden[name + "x"]], axis=1)
    U = evaluate_interior(SystemSpec(), b, X, tg[:64])
    assert np.array_equal(U[:, :, 0], u)


def test_interior_field_exact_cfg1():
    """Independent oracle: cfg1's RHS is the boundary trace of 4 exterior
    Stokeslets, so the field evaluated from the GPU solve at interior points
    equals the exact Stokeslet field (2.6e-10 on the CPU)."""
    from paper_2001_11619_b200 import evaluate_interior
    wl = configs.cfg1()
    b = wl.boundary
    f = _factor(wl)
    x = f.solve(wl.extra["rhs"])
    tg = configs.interior_targets(b, 200, seed=3)
    u = evaluate_interior(SystemSpec(), b, x, tg)
    H = configs.stokeslet_columns(tg, wl.extra["sources"])
    al = wl.extra["alpha"]
    exact = sum(H[:, 3 * i] * al[i, 0] + H[:, 3 * i + 1] * al[i, 1] for i in range(4)).reshape(-1, 2)
    assert _rel(u.ravel(), exact.ravel()) < 1e-8


def test_unphased_cfg2_end_to_end(golden):
    """Tie-rich geometry end to end: skeleton agreement with the reference is
    reported; the GPU solve's backward error (exact operator) stays within 2x
    the reference solution's (tie flips move the forward solution by ~50 eps,
    SURVEY.md §0)."""
    from paper_2001_11619_b200 import system_matvec
    wl = configs.cfg2(phases=False)
    b = wl.boundary
    f = _factor(wl)
    keys = [tuple(k) for k in golden["cfg2u_keys"]]
    so, S = golden["cfg2u_S_off"], golden["cfg2u_S"]
    same = sum(np.array_equal(f.factors[k].S_loc, S[so[i]:so[i + 1]]) for i, k in enumerate(keys)
               if k in f.factors)
    rhs = wl.extra["rhs"]
    x = f.solve(rhs)
    xr = golden["cfg2u_x"]
    R = system_matvec(SystemSpec(), b, np.stack([x, xr], axis=1)) - rhs[:, None]
    rg, rc = np.linalg.norm(R, axis=0) / np.linalg.norm(rhs)
    print(f"unphased cfg2: {same}/{len(keys)} identical skeletons end to end; solve rel diff "
          f"{_rel(x, xr):.2e}; residual GPU {rg:.2e} reference {rc:.2e}")
    assert rg <= 2 * rc


@pytest.mark.parametrize("name,builder", [("lap_", configs.cfg1), ("lapm_", configs.mini_holes)])
def test_laplace_factor_solve_vs_reference(golden, name, builder):
    """Laplace-Neumann variant (kernels.py:119-125,
    161-168, 322-325, 347-352, 368-370): identical skeletons per box and root
    DOFs, solve / apply within 10 eps of the reference, residual against the
    exact operator, and the interior field u = -S mu."""
    from paper_2001_11619_b200 import LAPLACE, evaluate_interior, system_matvec
    wl = builder()
    b = wl.boundary
    spec = SystemSpec(LAPLACE)
    t = build_tree(b.positions, wl.leaf_cap)
    f = factor(spec, b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
    assert f.dim == b.n_nodes
    keys = [tuple(k) for k in golden[name + "keys"]]
    so, S = golden[name + "S_off"], golden[name + "S"]
    bad = [k for i, k in enumerate(keys) if not np.array_equal(f.factors[k].S_loc, S[so[i]:so[i + 1]])]
    assert not bad, bad
    assert np.array_equal(f.root_dofs, golden[name + "root_dofs"])
    kpl = {int(l): int(v) for l, v in golden[name + "k_per_level"]}
    assert f.stats["k_per_level"] == kpl
    rhs = golden[name + "rhs"]
    x = f.solve(rhs)
    assert _rel(x, golden[name + "x"]) <= 10 * wl.tol
    r = system_matvec(spec, b, x) - rhs
    assert np.linalg.norm(r) / np.linalg.norm(rhs) < 1e-8
    if name + "apply_in" in golden.files:
        y = f.apply(golden[name + "apply_in"])
        assert _rel(y, golden[name + "apply_out"]) <= 10 * wl.tol
    if name + "interior" in golden.files:
        u = evaluate_interior(spec, b, golden[name + "x"], golden[name + "targets"])
        ref = golden[name + "interior"]
        assert u.shape == ref.shape
        assert np.max(np.abs(u - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_laplace_update_equals_refactor(golden):
    """Laplace hole-move update on the 3-hole geometry: equals the reference's
    update within 10 eps and the GPU refactor bitwise."""
    from paper_2001_11619_b200 import LAPLACE
    wl = configs.mini_holes()
    b = wl.boundary
    spec = SystemSpec(LAPLACE)
    f = factor(spec, b, build_tree(b.positions, wl.leaf_cap), wl.tol, proxy_count=wl.proxy_count,
               proxy_factor=wl.proxy_factor)
    nb, rep = apply_perturbation(b, [MoveHole(1, translation=(-0.08, 0.06))])
    fu = update(f, nb, rep)
    assert fu.stats["n_dirty"] == int(golden["lapm_upd_ndirty"])
    rhs = golden["lapm_rhs"]
    xu = fu.solve(rhs)
    assert _rel(xu, golden["lapm_upd_x"]) <= 10 * wl.tol
    t2 = build_tree(nb.positions, wl.leaf_cap, root_box=(f.tree.root_center, f.tree.root_half_width))
    fr = factor(spec, nb, t2, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
    assert np.array_equal(fr.solve(rhs), xu)


def test_box_factors_lu_view():
    """BoxFactors.lu (reference skel.py:69): host copy of the X_RR LU factors
    and pivots; lu.solve(X_RR) reproduces the identity."""
    wl = configs.cfg1()
    f = _factor(wl)
    k = [k for k in f.factors if len(f.factors[k].R_loc) > 20][0]
    bf = f.factors[k]
    lu = bf.lu
    X = bf.X_rr
    assert lu.n == X.shape[0] and lu.piv.shape == (X.shape[0],)
    assert np.abs(lu.solve(X) - np.eye(lu.n)).max() < 1e-10
    assert 0 < lu.pivot_ratio <= 1


def test_add_and_delete_hole_updates(monkeypatch):
    """Non-DOF-preserving edits (reference skel.py:493-498, BoxFactors.remapped):
    update() after DeleteHole / AddHole marks the reference's dirty set, solves
    within 10 eps of the reference's updated factorization (fixtures recorded from
    the unmodified reference, tests/golden/make_golden_edits.py) and equals a GPU
    refactorization of the new geometry bitwise -- on the native driver and on the
    Python level loop; a hole move chained after the edit stays incremental."""
    import os
    from paper_2001_11619_b200.geometry import AddHole, Curve, DeleteHole, HOLE
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden_edits.npz"))
    wl = configs.mini_holes()
    b = wl.boundary
    nodes = g["add_nodes"]
    rad = float(np.sqrt(((nodes - nodes.mean(axis=0)) ** 2).sum(axis=1)).max())
    hole = Curve(nodes, g["add_weights"], g["add_normals"], g["add_curvatures"], HOLE, rad)
    cases = (("del", [DeleteHole(2)]), ("add", [AddHole(hole)]))
    for engine in (True, False):
        monkeypatch.setattr(skel, "_ENGINE_ON", engine)
        f = _factor(wl)
        for name, edits in cases:
            nb, rep = apply_perturbation(b, edits)
            fu = update(f, nb, rep)
            want = {tuple(int(v) for v in k) for k in g[f"{name}_dirty"]}
            assert fu.stats["dirty"] == want, (engine, name)
            rhs = g[f"{name}_rhs"]
            assert fu.dim == len(rhs)
            x = fu.solve(rhs)
            assert _rel(x, g[f"{name}_x"]) <= 10 * wl.tol, (engine, name, _rel(x, g[f"{name}_x"]))
            t2 = build_tree(nb.positions, wl.leaf_cap, root_box=(f.tree.root_center, f.tree.root_half_width))
            fr = factor(SystemSpec(), nb, t2, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
            assert set(fu.factors.keys()) == set(fr.factors.keys())
            for k in fr.factors.keys():
                assert np.array_equal(fu.factors[k].skel_dofs, fr.factors[k].skel_dofs), (engine, name, k)
            assert np.array_equal(x, fr.solve(rhs)), (engine, name)
            # a hole move on top of the edited factorization (incremental sweep again)
            nb2, rep2 = apply_perturbation(nb, [MoveHole(1, translation=(0.04, -0.03))])
            fu2 = update(fu, nb2, rep2)
            t3 = build_tree(nb2.positions, wl.leaf_cap, root_box=(f.tree.root_center, f.tree.root_half_width))
            fr2 = factor(SystemSpec(), nb2, t3, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
            assert np.array_equal(fu2.solve(rhs), fr2.solve(rhs)), (engine, name, "move after edit")


@pytest.mark.parametrize("nm,builder", [("pzm", configs.mini_holes), ("pz1", configs.cfg1)])
def test_propagate_zeros_mode_vs_reference(nm, builder):
    """factor(propagate_zeros=True), the reference's sequential validation mode
    (skel.py:267-270, 354-361): skeletons identical to the reference's box for box
    (fixtures recorded from the unmodified reference) and the solve within 10 eps;
    it differs from the default mode on some boxes, so the mode is exercised."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden_edits.npz"))
    wl = builder()
    b = wl.boundary
    t = build_tree(b.positions, wl.leaf_cap)
    f = factor(SystemSpec(), b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor,
               propagate_zeros=True)
    keys = [tuple(int(v) for v in k) for k in g[nm + "_keys"]]
    off = g[nm + "_skel_off"]
    assert set(keys) == set(f.factors.keys())
    for i, k in enumerate(keys):
        assert np.array_equal(f.factors[k].skel_dofs, g[nm + "_skel"][off[i]:off[i + 1]]), k
    assert _rel(f.solve(wl.extra["rhs"]), g[nm + "_x"]) <= 10 * wl.tol
    f0 = _factor(wl)
    assert any(len(f.factors[k].skel_dofs) != len(f0.factors[k].skel_dofs) for k in keys)


def test_mixed_edit_chain_equals_refactor():
    """A chain of mixed edits on the 3-hole case (moves, a deletion, additions, a
    deletion of an added hole): every updated factorization has the skeletons and
    the solve of a GPU refactorization of the same geometry, bitwise, and the
    augmentation block follows the hole count."""
    from paper_2001_11619_b200.geometry import AddHole, DeleteHole, GeometryError, circle_curve, ellipse_curve
    wl = configs.mini_holes()
    b = wl.boundary
    f = _factor(wl)
    root = (f.tree.root_center, f.tree.root_half_width)
    rng = np.random.default_rng(17)
    script = [
        [MoveHole(1, translation=(0.05, 0.02))],
        [DeleteHole(2)],
        [AddHole(circle_curve(160, center=(-1.3, -1.0), radius=0.3, clockwise=True))],
        [MoveHole(3, translation=(0.03, 0.04)), MoveHole(1, translation=(-0.02, 0.01))],
        [AddHole(circle_curve(128, center=(1.2, 1.3), radius=0.25, clockwise=True)), DeleteHole(1)],
        [MoveHole(2, translation=(0.0, -0.05))],
        [DeleteHole(3)],
    ]
    cur, cb = f, b
    for step, edits in enumerate(script):
        nb, rep = apply_perturbation(cb, edits)
        cur = update(cur, nb, rep)
        assert cur.n_aug == 3 * nb.n_holes and cur.dim == 2 * nb.n_nodes + 3 * nb.n_holes
        t2 = build_tree(nb.positions, wl.leaf_cap, root_box=root)
        fr = factor(SystemSpec(), nb, t2, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
        rhs = np.concatenate([rng.standard_normal(2 * nb.n_nodes), np.zeros(3 * nb.n_holes)])
        assert set(cur.factors.keys()) == set(fr.factors.keys()), step
        for k in fr.factors.keys():
            assert np.array_equal(cur.factors[k].skel_dofs, fr.factors[k].skel_dofs), (step, k)
        assert np.array_equal(cur.solve(rhs), fr.solve(rhs)), step
        y = np.random.default_rng(step).standard_normal(cur.dim)
        assert np.array_equal(cur.apply(y), fr.apply(y)), step
        cb = nb
        del fr


def test_laplace_add_delete_hole_updates():
    """The Laplace-Neumann branch (one DOF per node, no augmentation) through the
    non-DOF-preserving edits: update == GPU refactor bitwise and within 10 eps of
    the CPU oracle's factorization of the edited geometry."""
    from paper_2001_11619_b200 import LAPLACE
    from paper_2001_11619_b200.geometry import AddHole, DeleteHole, circle_curve
    wl = configs.mini_holes()
    b = wl.boundary
    spec = SystemSpec(LAPLACE)
    t = build_tree(b.positions, wl.leaf_cap)
    f = factor(spec, b, t, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
    root = (t.root_center, t.root_half_width)
    # DeleteHole(1): the reference's own update differs from its refactor in the last
    # ulp there (checked with the unmodified reference: skeletons equal, 7e-16), so
    # that edit is held to 1e-13; the other two are bitwise
    hole = circle_curve(160, center=(-1.3, -1.0), radius=0.3, clockwise=True)
    for edits, exact in (([DeleteHole(2)], True), ([AddHole(hole)], True), ([DeleteHole(1)], False)):
        nb, rep = apply_perturbation(b, edits)
        fu = update(f, nb, rep)
        t2 = build_tree(nb.positions, wl.leaf_cap, root_box=root)
        fr = factor(spec, nb, t2, wl.tol, proxy_count=wl.proxy_count, proxy_factor=wl.proxy_factor)
        rhs = np.random.default_rng(3).standard_normal(fu.dim)
        x = fu.solve(rhs)
        assert fu.dim == nb.n_nodes
        for k in fr.factors.keys():
            assert np.array_equal(fu.factors[k].skel_dofs, fr.factors[k].skel_dofs), k
        xr = fr.solve(rhs)
        assert np.array_equal(x, xr) if exact else _rel(x, xr) < 1e-13
        ref = O.factor(nb, O.QTree(nb.positions, wl.leaf_cap, root_box=root), wl.tol, wl.proxy_count,
                       wl.proxy_factor, pde=O.LAPLACE)
        assert _rel(x, ref.solve(rhs)) <= 10 * wl.tol
