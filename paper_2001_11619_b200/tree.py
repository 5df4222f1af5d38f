"""Adaptive quadtree over boundary nodes, flat struct-of-arrays, built level by level.

Same semantics as the reference ``tree.py`` (``/root/reference/pkg/src/skelsolve``):
geometric keys ``(level, ix, iy)`` with root ``(0, 0, 0)`` (``tree.py:1-11``),
child order SW, SE, NW, NE with empty children pruned (``tree.py:19``),
split while a box holds more than ``leaf_cap`` nodes, ``east = x >= cx``,
``north = y >= cy`` (``tree.py:127-144``), default root = bounding square
inflated by 10% (``tree.py:102-107``), fixed root for refits
(``tree.py:239-248``).  Box centres are formed with the reference's exact
floating-point expressions so proxy discs and far-field filters agree bitwise.

Boxes are indexed globally level by level, keys sorted within a level
(``Tree.levels[l]`` = sorted keys, ``tree.py:148``).  Neighbour queries,
coarse-leaf disc queries, far-field DOF lists and the update's dirty marking
are vectorised NumPy (the reference walks Python dicts per box).
"""

from __future__ import annotations

import numpy as np

CHILD_OFFSETS = ((0, 0), (1, 0), (0, 1), (1, 1))   # SW, SE, NW, NE
NBR_OFFSETS = [(dx, dy) for dx in (-1, 0, 1) for dy in (-1, 0, 1) if dx or dy]  # sorted order


class TreeError(ValueError):
    pass


def default_root_box(positions, inflate: float = 0.1):
    """Reference tree.py:102-107."""
    lo = positions.min(axis=0)
    hi = positions.max(axis=0)
    center = 0.5 * (lo + hi)
    hw = 0.5 * float((hi - lo).max()) * (1.0 + inflate)
    return center, hw


def proxy_radius(half_width, factor: float = 1.5):
    """Reference tree.py:158-160 (factor x circumradius)."""
    return factor * half_width * np.sqrt(2.0)


class Tree:
    """Flat quadtree.  Per-box arrays are indexed by global box index."""

    def __init__(self, root_center, root_hw, leaf_cap, max_depth):
        self.root_center = np.asarray(root_center, float)
        self.root_half_width = float(root_hw)
        self.leaf_cap = leaf_cap
        self.max_depth = max_depth

    # -- reference-like accessors -------------------------------------------
    @property
    def depth(self) -> int:
        return len(self.level_start) - 2

    @property
    def levels(self):
        return [[self.key(i) for i in range(self.level_start[l], self.level_start[l + 1])]
                for l in range(self.depth + 1)]

    def key(self, i) -> tuple:
        return (int(self.lev[i]), int(self.ix[i]), int(self.iy[i]))

    @property
    def _index(self) -> dict:
        idx = self.__dict__.get("_index_d")
        if idx is None:
            idx = {self.key(i): i for i in range(len(self.lev))}
            self.__dict__["_index_d"] = idx
        return idx

    def index(self, key) -> int:
        return self._index[tuple(int(v) for v in key)]

    def has(self, key) -> bool:
        return tuple(int(v) for v in key) in self._index

    def level_indices(self, l):
        return np.arange(self.level_start[l], self.level_start[l + 1])

    def nodes_of(self, i) -> np.ndarray:
        l = self.lev[i]
        s = self.node_start[i]
        return self.level_nodes[l][s:s + self.node_cnt[i]]

    def children_of(self, i):
        return [int(c) for c in self.children[i] if c >= 0]

    def colleagues(self, key) -> list:
        i = self.index(key)
        return [self.key(j) for j in self.neighbors[i] if j >= 0]

    # -- vectorised queries ---------------------------------------------------
    def _finish(self):
        n = len(self.lev)
        self.is_leaf = self.nchild == 0
        # same-level neighbours in sorted key order (tree.py:70-81)
        self.neighbors = np.full((n, 8), -1, dtype=np.int64)
        for l in range(self.depth + 1):
            idx = self.level_indices(l)
            if len(idx) == 0:
                continue
            side = np.int64(1) << np.int64(l)
            codes = self.ix[idx] * side + self.iy[idx]
            for s, (dx, dy) in enumerate(NBR_OFFSETS):
                nx, ny = self.ix[idx] + dx, self.iy[idx] + dy
                ok = (nx >= 0) & (ny >= 0) & (nx < side) & (ny < side)
                c = nx * side + ny
                pos = np.searchsorted(codes, c)
                pos_c = np.minimum(pos, len(codes) - 1)
                hit = ok & (codes[pos_c] == c)
                self.neighbors[idx[hit], s] = idx[pos_c[hit]]
        self.node_leaf = np.empty(self.n_nodes, dtype=np.int64)
        for l in range(self.depth + 1):
            idx = self.level_indices(l)
            leaves = idx[self.is_leaf[idx]]
            for i in leaves:
                self.node_leaf[self.nodes_of(i)] = i

    def coarse_leaves(self, box_idx, radius):
        """Leaves above the boxes' level meeting the disc (centre, radius), as
        (box position, leaf index) pairs sorted by key per box -- reference
        Tree.shallow_leaves_near, tree.py:83-99.  Candidates come from the
        level grid (every box of a coarser level covering a cell the disc's
        bounding square touches), then the reference's box-disc test."""
        box_idx = np.asarray(box_idx, np.int64)
        B = len(box_idx)
        if B == 0:
            return np.zeros(0, np.int64), np.zeros(0, np.int64)
        L = int(self.lev[box_idx[0]])
        c = self.center[box_idx]
        r = np.asarray(radius, float)
        origin = self.root_center - self.root_half_width
        side = np.int64(1) << np.int64(L)
        cell = 2.0 * self.root_half_width / float(side)
        lo = np.floor((c - r[:, None] - origin[None, :]) / cell).astype(np.int64)
        hi = np.floor((c + r[:, None] - origin[None, :]) / cell).astype(np.int64)
        lo = np.clip(lo, 0, side - 1)
        hi = np.clip(hi, 0, side - 1)
        pb_all, pc_all = [], []
        for lp in range(L):
            idx_l = self.level_indices(lp)
            if len(idx_l) == 0:
                continue
            sh = np.int64(L - lp)
            s_l = np.int64(1) << np.int64(lp)
            clo, chi = lo >> sh, hi >> sh            # cell ranges covered at level lp
            codes_l = self.ix[idx_l] * s_l + self.iy[idx_l]
            wx = int((chi[:, 0] - clo[:, 0]).max()) + 1
            wy = int((chi[:, 1] - clo[:, 1]).max()) + 1
            for ox in range(wx):
                for oy in range(wy):
                    cx = clo[:, 0] + ox
                    cy = clo[:, 1] + oy
                    dup = (cx > chi[:, 0]) | (cy > chi[:, 1])
                    code = cx * s_l + cy
                    pos = np.searchsorted(codes_l, code)
                    pos_c = np.minimum(pos, len(codes_l) - 1)
                    hit = (~dup) & (codes_l[pos_c] == code)
                    j = idx_l[pos_c[hit]]
                    leaf = self.is_leaf[j]
                    pb_all.append(np.flatnonzero(hit)[leaf])
                    pc_all.append(j[leaf])
        if not pb_all:
            return np.zeros(0, np.int64), np.zeros(0, np.int64)
        pb = np.concatenate(pb_all)
        pc = np.concatenate(pc_all)
        if len(pb) == 0:
            return pb, pc
        d = np.maximum(np.abs(c[pb] - self.center[pc]) - self.hw[pc][:, None], 0.0)
        keep = ~(d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1] > r[pb] * r[pb])
        pb, pc = pb[keep], pc[keep]
        # sort by (box, key); global index order == key order (levels ascending, keys sorted)
        order = np.lexsort((pc, pb))
        return pb[order], pc[order]

    def coarse_leaves_mask(self, box_idx, radius):
        """Dense variant (box x all coarser leaves), kept for tests."""
        l = int(self.lev[box_idx[0]])
        cand = np.flatnonzero(self.is_leaf & (self.lev < l))
        if len(cand) == 0 or len(box_idx) == 0:
            return np.zeros((len(box_idx), 0), bool), cand
        c = self.center[box_idx]
        d = np.maximum(np.abs(c[:, None, :] - self.center[cand][None, :, :])
                       - self.hw[cand][None, :, None], 0.0)
        dd = d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]
        r = np.asarray(radius, float)
        mask = ~(dd > (r * r)[:, None])
        return mask, cand

    def hole_pairs(self, curve_offsets):
        """(box, curve) membership for every box, propagated leaves -> root."""
        nbox = len(self.lev)
        leaves = np.flatnonzero(self.is_leaf)
        boxes, curves = [], []
        for l in range(self.depth + 1):
            li = leaves[self.lev[leaves] == l]
            if len(li) == 0:
                continue
            st = self.node_start[li]
            cnt = self.node_cnt[li]
            off = np.zeros(len(li) + 1, np.int64)
            np.cumsum(cnt, out=off[1:])
            idx = np.repeat(st - off[:-1], cnt) + np.arange(off[-1])
            nodes = self.level_nodes[l][idx]
            cur = np.searchsorted(curve_offsets, nodes, side="right") - 1
            boxes.append(np.repeat(li, cnt))
            curves.append(cur)
        b = np.concatenate(boxes)
        cv = np.concatenate(curves)
        nc = int(len(curve_offsets))
        key = np.unique(b * nc + cv)
        b, cv = key // nc, key % nc
        allb, allc = [b], [cv]
        cur_b, cur_c = b, cv
        while True:
            par = self.parent[cur_b]
            ok = par >= 0
            if not ok.any():
                break
            key = np.unique(par[ok] * nc + cur_c[ok])
            cur_b, cur_c = key // nc, key % nc
            allb.append(cur_b)
            allc.append(cur_c)
        key = np.unique(np.concatenate(allb) * nc + np.concatenate(allc))
        return key // nc, key % nc


def build_tree(positions, leaf_cap: int = 64, root_box=None, max_depth: int = 40) -> Tree:
    """Reference build_tree (tree.py:110-155) in the native host runtime
    (csrc/host.cpp skb_tree_build); same tree as ``build_tree_np``."""
    from . import _lib
    pos = np.ascontiguousarray(positions, np.float64)
    N = len(pos)
    if root_box is None:
        center, hw = default_root_box(pos)
    else:
        center, hw = np.asarray(root_box[0], float), float(root_box[1])
        if np.any(np.abs(pos - center[None, :]) > hw * (1 + 1e-12)):
            raise TreeError("node outside the fixed root box")
    max_depth_eff = min(max_depth, 30)   # keys are int64 codes; deeper trees never occur here
    lib = _lib.load()
    root = np.array([center[0], center[1], hw], np.float64)
    h = np.zeros(1, np.int64)
    lib.skb_tree_build(pos.ctypes.data, N, leaf_cap, max_depth_eff, root.ctypes.data, h.ctypes.data)
    try:
        sz = np.zeros(3, np.int64)
        lib.skb_tree_sizes(int(h[0]), sz.ctypes.data)
        nbox, depth, nln = (int(v) for v in sz)
        t = Tree(center, hw, leaf_cap, max_depth)
        t.n_nodes = N
        a = {k: np.empty(n, np.int64) for k, n in (
            ("level_start", depth + 2), ("lev", nbox), ("ix", nbox), ("iy", nbox), ("parent", nbox),
            ("children", 4 * nbox), ("nchild", nbox), ("node_start", nbox), ("node_cnt", nbox),
            ("level_nodes", nln), ("level_nodes_off", depth + 2), ("nbr", 8 * nbox),
            ("node_leaf", N))}
        cen = np.empty((nbox, 2))
        hws = np.empty(nbox)
        lib.skb_tree_export(int(h[0]), *(a[k].ctypes.data for k in (
            "level_start", "lev", "ix", "iy", "parent")), cen.ctypes.data, hws.ctypes.data,
            *(a[k].ctypes.data for k in ("children", "nchild", "node_start", "node_cnt",
                                        "level_nodes", "level_nodes_off", "nbr", "node_leaf")))
    finally:
        lib.skb_tree_free(int(h[0]))
    t.level_start, t.lev, t.ix, t.iy, t.parent = (a["level_start"], a["lev"], a["ix"], a["iy"],
                                                  a["parent"])
    t.center, t.hw = cen, hws
    t.children = a["children"].reshape(nbox, 4)
    t.nchild = a["nchild"]
    t.node_start, t.node_cnt = a["node_start"], a["node_cnt"]
    lo = a["level_nodes_off"]
    t.level_nodes = [a["level_nodes"][lo[l]:lo[l + 1]] for l in range(depth + 1)]
    t._level_nodes_flat, t._level_nodes_off = a["level_nodes"], lo
    t.is_leaf = t.nchild == 0
    t.neighbors = a["nbr"].reshape(nbox, 8)
    t.node_leaf = a["node_leaf"]
    return t


def build_tree_np(positions, leaf_cap: int = 64, root_box=None, max_depth: int = 40) -> Tree:
    """Reference build_tree (tree.py:110-155), vectorised per level (NumPy
    restatement of the native build, kept as its test oracle)."""
    pos = np.asarray(positions, float)
    N = len(pos)
    if root_box is None:
        center, hw = default_root_box(pos)
    else:
        center, hw = np.asarray(root_box[0], float), float(root_box[1])
        if np.any(np.abs(pos - center[None, :]) > hw * (1 + 1e-12)):
            raise TreeError("node outside the fixed root box")
    if max_depth > 30:
        max_depth_eff = 30   # keys are int64 codes; deeper trees never occur here
    else:
        max_depth_eff = max_depth
    t = Tree(center, hw, leaf_cap, max_depth)
    t.n_nodes = N
    L_ix, L_iy, L_cen, L_hw, L_par, L_nstart, L_ncnt, L_nodes = [], [], [], [], [], [], [], []
    L_children = []
    ix = np.zeros(1, np.int64)
    iy = np.zeros(1, np.int64)
    cen = center[None, :].copy()
    half = np.array([hw])
    par_local = np.array([-1], np.int64)
    nodes = np.arange(N, dtype=np.int64)
    cnt = np.array([N], np.int64)
    l = 0
    while True:
        nb = len(ix)
        start = np.concatenate([[0], np.cumsum(cnt)[:-1]]).astype(np.int64)
        L_ix.append(ix); L_iy.append(iy); L_cen.append(cen); L_hw.append(half)
        L_par.append(par_local); L_nstart.append(start); L_ncnt.append(cnt); L_nodes.append(nodes)
        split = (cnt > leaf_cap) & (l < max_depth_eff)
        ch = np.full((nb, 4), -1, np.int64)
        L_children.append(ch)
        if not split.any():
            break
        box_of = np.repeat(np.arange(nb), cnt)
        sel = split[box_of]
        sn = nodes[sel]
        sb = box_of[sel]
        east = pos[sn, 0] >= cen[sb, 0]
        north = pos[sn, 1] >= cen[sb, 1]
        dx = east.astype(np.int64)
        dy = north.astype(np.int64)
        cix = 2 * ix[sb] + dx
        ciy = 2 * iy[sb] + dy
        side = np.int64(1) << np.int64(l + 1)
        code = cix * side + ciy
        ucode, first, inv = np.unique(code, return_index=True, return_inverse=True)
        order = np.argsort(inv, kind="stable")
        nodes = sn[order]
        cnt = np.bincount(inv, minlength=len(ucode)).astype(np.int64)
        pb = sb[first]
        q = (dx + 2 * dy)[first]
        ix = cix[first]
        iy = ciy[first]
        d = np.stack([dx[first], dy[first]], axis=1).astype(float)
        cen = cen[pb] + (d - 0.5) * half[pb][:, None]
        half = half[pb] / 2
        par_local = pb
        ch[pb, q] = np.arange(len(ucode))
        l += 1
    depth = l
    sizes = [len(a) for a in L_ix]
    t.level_start = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    t.lev = np.concatenate([np.full(s, li, np.int64) for li, s in enumerate(sizes)])
    t.ix = np.concatenate(L_ix)
    t.iy = np.concatenate(L_iy)
    t.center = np.concatenate(L_cen)
    t.hw = np.concatenate(L_hw)
    t.parent = np.concatenate([np.where(p >= 0, p + t.level_start[max(li - 1, 0)], -1)
                               for li, p in enumerate(L_par)])
    children = []
    for li, ch in enumerate(L_children):
        base = t.level_start[li + 1] if li + 1 <= depth else 0
        # compact in child order (SW, SE, NW, NE), drop empties
        out = np.full_like(ch, -1)
        for r in range(len(ch)):
            k = ch[r][ch[r] >= 0]
            out[r, :len(k)] = k + base
        children.append(out)
    t.children = np.concatenate(children)
    t.nchild = (t.children >= 0).sum(axis=1)
    t.node_start = np.concatenate(L_nstart)
    t.node_cnt = np.concatenate(L_ncnt)
    t.level_nodes = L_nodes
    t._finish()
    return t


def refit_tree(t: Tree, positions_new) -> Tree:
    """Reference tree.py:239-248: rebuild with the same root box."""
    return build_tree(positions_new, t.leaf_cap, root_box=(t.root_center, t.root_half_width),
                      max_depth=t.max_depth)


# ---------------------------------------------------------------------------
# update bookkeeping (reference skel.py:476-491, 517-534; tree.py:215-270)
# ---------------------------------------------------------------------------
def ownership_changed(t_new: Tree, t_old: Tree, old_to_new) -> set:
    """Keys of new-tree boxes whose owned node set differs from their twin
    (reference tree.py:251-270), compared level by level on node segments."""
    old_to_new = np.asarray(old_to_new, np.int64)
    changed = set()
    for l in range(max(t_new.depth, t_old.depth) + 1):
        in_new = t_new.level_indices(l) if l <= t_new.depth else np.zeros(0, np.int64)
        in_old = t_old.level_indices(l) if l <= t_old.depth else np.zeros(0, np.int64)
        side = np.int64(1) << np.int64(l)
        cn = t_new.ix[in_new] * side + t_new.iy[in_new]
        co = t_old.ix[in_old] * side + t_old.iy[in_old]
        pos = np.searchsorted(co, cn)
        pos_c = np.minimum(pos, max(len(co) - 1, 0))
        twin = (len(co) > 0) & (co[pos_c] == cn) if len(co) else np.zeros(len(cn), bool)
        for i in in_new[~twin]:
            changed.add(t_new.key(i))
        bn, bo = in_new[twin], in_old[pos_c[twin]]
        if len(bn):
            cnt_n, cnt_o = t_new.node_cnt[bn], t_old.node_cnt[bo]
            same_cnt = cnt_n == cnt_o
            bn2, bo2 = bn[same_cnt], bo[same_cnt]
            for i in bn[~same_cnt]:
                changed.add(t_new.key(i))
            if len(bn2):
                cnt = t_new.node_cnt[bn2]
                off = np.zeros(len(bn2) + 1, np.int64)
                np.cumsum(cnt, out=off[1:])
                rel = np.arange(off[-1]) - np.repeat(off[:-1], cnt)
                nn = t_new.level_nodes[l][np.repeat(t_new.node_start[bn2], cnt) + rel]
                oo = old_to_new[t_old.level_nodes[l][np.repeat(t_old.node_start[bo2], cnt) + rel]]
                diff = (nn != oo).astype(np.int64)
                bad = np.add.reduceat(diff, off[:-1]) > 0 if off[-1] else np.zeros(len(bn2), bool)
                bad &= cnt > 0
                for i in bn2[bad]:
                    changed.add(t_new.key(i))
        # boxes that vanished: their nearest surviving ancestor changed
        if len(in_old):
            pos2 = np.searchsorted(cn, co) if len(cn) else np.zeros(len(co), np.int64)
            pos2c = np.minimum(pos2, max(len(cn) - 1, 0))
            gone = ~((len(cn) > 0) & (cn[pos2c] == co)) if len(cn) else np.ones(len(co), bool)
            for j in in_old[gone]:
                p = int(j)
                while p >= 0 and not t_new.has(t_old.key(p)):
                    p = int(t_old.parent[p])
                if p >= 0:
                    changed.add(t_old.key(p))
    return changed


def mark_disc_hits(t: Tree, pts, proxy_factor, out: set):
    """Boxes whose proxy disc contains a point (tree.py:215-236): candidates from
    the (2 reach + 1)^2 cell neighbourhood of each point, then the distance test."""
    pts = np.asarray(pts, float)
    for lev in range(t.depth + 1):
        idx = t.level_indices(lev)
        if len(idx) == 0:
            continue
        hw = t.root_half_width / 2 ** lev
        rad = proxy_radius(hw, proxy_factor)
        step = 2 * hw
        origin = t.root_center - t.root_half_width
        cells = np.floor((pts - origin[None, :]) / step).astype(np.int64)
        reach = int(np.ceil(rad / step)) + 1
        side = np.int64(1) << np.int64(lev)
        codes = t.ix[idx] * side + t.iy[idx]
        ucell = np.unique(cells[:, 0] * (side + 2 * reach + 2) + cells[:, 1])
        cx = ucell // (side + 2 * reach + 2)
        cy = ucell - cx * (side + 2 * reach + 2)
        cand = []
        for dx in range(-reach, reach + 1):
            for dy in range(-reach, reach + 1):
                nx, ny = cx + dx, cy + dy
                ok = (nx >= 0) & (ny >= 0) & (nx < side) & (ny < side)
                c = nx * side + ny
                pos = np.searchsorted(codes, c)
                pc = np.minimum(pos, len(codes) - 1)
                hit = ok & (codes[pc] == c)
                cand.append(idx[pc[hit]])
        cand = np.unique(np.concatenate(cand)) if cand else np.zeros(0, np.int64)
        for k in cand:
            d2 = ((pts - t.center[k][None, :]) ** 2).sum(axis=1)
            if (d2 <= rad * rad).any():
                out.add(t.key(k))


def dirty_closure(t: Tree, content: set) -> set:
    """Parents + colleagues closure, reference skel.py:517-534."""
    marked = {l: set() for l in range(t.depth + 1)}
    for key in content:
        marked[key[0]].add(key)
    for lev in range(t.depth, -1, -1):
        grew = set(marked[lev])
        if lev + 1 <= t.depth:
            for key in marked[lev + 1]:
                p = int(t.parent[t.index(key)])
                if p >= 0:
                    grew.add(t.key(p))
        for key in list(grew):
            grew.update(t.colleagues(key))
        marked[lev] = grew
    out = set()
    for s in marked.values():
        out |= s
    return out


def _flat_arrays(t: Tree):
    if not hasattr(t, "_level_nodes_flat"):
        t._level_nodes_off = np.zeros(t.depth + 2, np.int64)
        np.cumsum([len(x) for x in t.level_nodes], out=t._level_nodes_off[1:])
        t._level_nodes_flat = np.concatenate(t.level_nodes).astype(np.int64)
    arrs = [np.ascontiguousarray(x, np.int64) for x in (
        t.level_start, t.lev, t.ix, t.iy, t.parent, t.node_start, t.node_cnt,
        t._level_nodes_flat, t._level_nodes_off, t.neighbors, t.node_leaf)]
    return arrs, (np.ctypeslib.as_ctypes_type(np.uint64) * len(arrs))(*[x.ctypes.data for x in arrs])


def dirty_mask(t_old: Tree, t_new: Tree, b_new, report, proxy_factor) -> np.ndarray:
    """Dirty boxes of an update (reference skel.py:476-491) as a mask over the
    new tree, from the native host runtime (csrc/host.cpp skb_dirty_set)."""
    from . import _lib
    pts = []
    if len(report.modified_nodes_old):
        pts.append(report.old_positions[report.modified_nodes_old])
    if len(report.modified_nodes_new):
        pts.append(b_new.positions[report.modified_nodes_new])
    pts = np.ascontiguousarray(np.concatenate(pts) if pts else np.zeros((0, 2)), np.float64)
    an, pn = _flat_arrays(t_new)
    ao, po = _flat_arrays(t_old)
    root = np.array([t_new.root_center[0], t_new.root_center[1], t_new.root_half_width])
    o2n = np.ascontiguousarray(report.old_to_new, np.int64)
    mod = np.ascontiguousarray(report.modified_nodes_new, np.int64)
    cen = np.ascontiguousarray(t_new.center, np.float64)
    out = np.zeros(len(t_new.lev), np.uint8)
    _lib.load().skb_dirty_set(pn, cen.ctypes.data, t_new.depth, po, t_old.depth, root.ctypes.data,
                              o2n.ctypes.data, pts.ctypes.data, len(pts), mod.ctypes.data, len(mod),
                              float(proxy_factor), out.ctypes.data)
    del an, ao
    return out.astype(bool)


def dirty_set(t_old: Tree, t_new: Tree, b_new, report, proxy_factor) -> set:
    """Dirty boxes of an update (reference skel.py:476-491), as keys."""
    m = dirty_mask(t_old, t_new, b_new, report, proxy_factor)
    return {t_new.key(i) for i in np.flatnonzero(m)}


def dirty_set_np(t_old: Tree, t_new: Tree, b_new, report, proxy_factor) -> set:
    """NumPy restatement of ``dirty_set`` (reference skel.py:476-491)."""
    content = set(ownership_changed(t_new, t_old, report.old_to_new))
    pts = []
    if len(report.modified_nodes_old):
        pts.append(report.old_positions[report.modified_nodes_old])
    if len(report.modified_nodes_new):
        pts.append(b_new.positions[report.modified_nodes_new])
    pts = np.concatenate(pts) if pts else np.zeros((0, 2))
    if len(pts):
        mark_disc_hits(t_new, pts, proxy_factor, content)
    for nid in report.modified_nodes_new:
        i = int(t_new.node_leaf[nid])
        while i >= 0 and t_new.key(i) not in content:
            content.add(t_new.key(i))
            i = int(t_new.parent[i])
    return dirty_closure(t_new, content)
