"""CPU oracle for the skeletonization hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and only
as the checker / the timed CPU reference arm.  The product package
``paper_2001_11619_b200`` never imports it and has no CPU fallback.

This is a numpy/scipy restatement of the reference package ``skelsolve``
(``/root/reference/pkg/src/skelsolve``), fp64 throughout.  Every function cites
the reference file:line it restates.  The dense arithmetic is delegated, as in
the reference, to SciPy's LAPACK (third-party: scipy 1.18.1 bundling
scipy-openblas32 0.3.31.dev; ``dgeqrf``/``dgeqp3``/``dtrtrs``/``dgetrf``/
``dgetrs``) -- the published LAPACK algorithms, called with the same arguments
as the reference call sites (``dense.py:59,60,77,122,135``).

Pinning: ``tests/golden/make_golden.py`` imported the unmodified reference in
the build container (through a two-line harness shim: a ``shapely`` stub and
the ``far_dofs`` tuple fix) and recorded per-box skeletons,
ID stacks, T blocks and solve/apply outputs; ``tests/test_oracle_golden.py``
checks this oracle against those fixtures bit for bit.

Kernel-entry formulas keep NumPy's operation order so stacks match the
reference bitwise.
"""

from __future__ import annotations

import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.linalg as sla
from threadpoolctl import threadpool_limits

JUMP = -0.5                 # kernels.py:38
PIVOT_FLOOR = 1e-12         # skel.py:46
ROOT = (0, 0, 0)
CHILD_ORDER = ((0, 0), (1, 0), (0, 1), (1, 1))   # tree.py:19 (SW, SE, NW, NE)


# ---------------------------------------------------------------------------
# Stokes kernel blocks (kernels.py)
# ---------------------------------------------------------------------------
def _split(dofs):
    d = np.asarray(dofs, dtype=np.int64)
    return d // 2, d % 2


def self_block(g, rows, cols):
    """Dense system-matrix block, Stokes branch of kernels.py:89-130."""
    na, ca = _split(rows)
    nb, cb = _split(cols)
    pa, pb = g.positions[na], g.positions[nb]
    dx = pa[:, None, 0] - pb[None, :, 0]
    dy = pa[:, None, 1] - pb[None, :, 1]
    d2 = dx * dx + dy * dy
    coincide = na[:, None] == nb[None, :]
    d2s = np.where(coincide, 1.0, d2)
    nrm_b = g.normals[nb]
    proj = dx * nrm_b[None, :, 0] + dy * nrm_b[None, :, 1]
    c = proj / (np.pi * d2s * d2s)
    ra = np.where((ca == 0)[:, None], dx, dy)
    rb = np.where((cb == 0)[None, :], dx, dy)
    val = c * ra * rb
    tang = np.stack([-g.normals[:, 1], g.normals[:, 0]], axis=1)
    ta, tb = tang[na, ca], tang[nb, cb]
    limit = -(g.curvatures[nb][None, :] / (2 * np.pi)) * ta[:, None] * tb[None, :]
    val = np.where(coincide, limit, val)
    val += g.normals[na, ca][:, None] * g.normals[nb, cb][None, :]
    out = val * g.weights[nb][None, :]
    out += np.where(np.asarray(rows, np.int64)[:, None] == np.asarray(cols, np.int64)[None, :],
                    JUMP, 0.0)
    return out


def pair_blocks(g, far, box):
    """(K[far, box], K[box, far]^T), Stokes branch of kernels.py:133-160."""
    nf, cf = _split(far)
    nb, cb = _split(box)
    pf, pb = g.positions[nf], g.positions[nb]
    dx = pf[:, None, 0] - pb[None, :, 0]
    dy = pf[:, None, 1] - pb[None, :, 1]
    d2 = dx * dx + dy * dy
    wf = g.weights[nf][:, None]
    wb = g.weights[nb][None, :]
    nbv, nfv = g.normals[nb], g.normals[nf]
    proj_b = dx * nbv[None, :, 0] + dy * nbv[None, :, 1]
    proj_f = dx * nfv[:, None, 0] + dy * nfv[:, None, 1]
    inv4 = 1.0 / (np.pi * d2 * d2)
    rf = np.where((cf == 0)[:, None], dx, dy)
    rb = np.where((cb == 0)[None, :], dx, dy)
    rr = rf * rb
    nn = g.normals[nf, cf][:, None] * g.normals[nb, cb][None, :]
    return (proj_b * inv4 * rr + nn) * wb, (-proj_f * inv4 * rr + nn) * wf


def stresslet_plain(tgt, src, src_n):
    """(2m, 2n) stresslet values, kernels.py:279-290."""
    dx = tgt[:, None, 0] - src[None, :, 0]
    dy = tgt[:, None, 1] - src[None, :, 1]
    d2 = dx * dx + dy * dy
    c = (dx * src_n[None, :, 0] + dy * src_n[None, :, 1]) / (np.pi * d2 * d2)
    out = np.empty((2 * len(tgt), 2 * len(src)))
    out[0::2, 0::2] = c * dx * dx
    out[0::2, 1::2] = c * dx * dy
    out[1::2, 0::2] = c * dy * dx
    out[1::2, 1::2] = c * dy * dy
    return out


def stokeslet_plain(tgt, src):
    """(2m, 2n) Stokeslet values, kernels.py:293-304."""
    dx = tgt[:, None, 0] - src[None, :, 0]
    dy = tgt[:, None, 1] - src[None, :, 1]
    d2 = dx * dx + dy * dy
    lg = -0.5 * np.log(d2)
    pref = 1.0 / (4 * np.pi)
    out = np.empty((2 * len(tgt), 2 * len(src)))
    out[0::2, 0::2] = pref * (lg + dx * dx / d2)
    out[0::2, 1::2] = pref * (dx * dy / d2)
    out[1::2, 0::2] = pref * (dy * dx / d2)
    out[1::2, 1::2] = pref * (lg + dy * dy / d2)
    return out


def proxy_ring(center, radius, count):
    """Proxy circle points and weights, kernels.py:263-273."""
    if radius <= 0 or count < 8:
        raise ValueError("bad proxy ring")
    th = 2 * np.pi * np.arange(count) / count
    pts = np.asarray(center, float)[None, :] + radius * np.stack([np.cos(th), np.sin(th)], axis=1)
    return pts, np.full(count, 2 * np.pi * radius / count)


def proxy_normals(pts):
    """Radial proxy normals about the point mean, kernels.py:340-342."""
    ctr = pts.mean(axis=0)
    pn = pts - ctr[None, :]
    pn /= np.linalg.norm(pn, axis=1)[:, None]
    return pn


def proxy_incoming(g, pts, cols):
    """kernels.py:307-321 (Stokes)."""
    nc, cc = _split(cols)
    blk = stresslet_plain(pts, g.positions[nc], g.normals[nc])
    return blk[:, 2 * np.arange(len(nc)) + cc] * g.weights[nc][None, :]


def proxy_outgoing(g, rows, pts, pw):
    """kernels.py:328-346 (Stokes)."""
    nr, cr = _split(rows)
    pos = g.positions[nr]
    pn = proxy_normals(pts)
    sel = 2 * np.arange(len(nr)) + cr
    w2 = np.repeat(pw, 2)[None, :]
    b1 = stresslet_plain(pos, pts, pn)[sel] * w2
    b2 = stokeslet_plain(pos, pts)[sel] * w2
    return np.vstack([b1.T, b2.T])


def nullspace_rows(g, cols):
    """kernels.py:355-371 (Stokes)."""
    nc, cc = _split(cols)
    return ((g.weights[nc] * g.normals[nc, cc])[None, :], g.normals[nc, cc][None, :])


# ---------------------------------------------------------------------------
# Laplace-Neumann branches (kernels.py:119-125, 161-168, 322-325, 347-352,
# 368-370; dof_per_node 1: a DOF is a node)
# ---------------------------------------------------------------------------
STOKES = "stokes_dirichlet"       # kernels.py:36
LAPLACE = "laplace_neumann"       # kernels.py:35


def lap_self_block(g, rows, cols):
    """kernels.py:89-130, Laplace branch (119-125): adjoint double layer,
    same-node limit kappa_row / (4 pi), + 1 completion, x w_col, jump."""
    nr = np.asarray(rows, np.int64)
    nc = np.asarray(cols, np.int64)
    pr, pc = g.positions[nr], g.positions[nc]
    rx = pr[:, None, 0] - pc[None, :, 0]
    ry = pr[:, None, 1] - pc[None, :, 1]
    r2 = rx * rx + ry * ry
    same = nr[:, None] == nc[None, :]
    r2s = np.where(same, 1.0, r2)
    nrt = g.normals[nr]
    rdn = rx * nrt[:, None, 0] + ry * nrt[:, None, 1]
    kern = rdn / (2 * np.pi * r2s)
    lim = np.broadcast_to(g.curvatures[nr][:, None] / (4 * np.pi), kern.shape)
    kern = np.where(same, lim, kern)
    kern = kern + 1.0
    out = kern * g.weights[nc][None, :]
    out += np.where(nr[:, None] == nc[None, :], JUMP, 0.0)
    return out


def lap_pair_blocks(g, far, box):
    """(K[far, box], K[box, far]^T), kernels.py:161-168."""
    nf = np.asarray(far, np.int64)
    nb = np.asarray(box, np.int64)
    pf, pb = g.positions[nf], g.positions[nb]
    rx = pf[:, None, 0] - pb[None, :, 0]
    ry = pf[:, None, 1] - pb[None, :, 1]
    r2 = rx * rx + ry * ry
    wf = g.weights[nf][:, None]
    wb = g.weights[nb][None, :]
    nfv, nbv = g.normals[nf], g.normals[nb]
    rdn_f = rx * nfv[:, None, 0] + ry * nfv[:, None, 1]
    rdn_b = rx * nbv[None, :, 0] + ry * nbv[None, :, 1]
    ir2 = 1.0 / (2 * np.pi * r2)
    return (rdn_f * ir2 + 1.0) * wb, (-rdn_b * ir2 + 1.0) * wf


def lap_proxy_incoming(g, pts, cols):
    """kernels.py:322-325: log potential of the box sources on the proxy ring."""
    nc = np.asarray(cols, np.int64)
    rx = pts[:, None, 0] - g.positions[nc][None, :, 0]
    ry = pts[:, None, 1] - g.positions[nc][None, :, 1]
    r2 = rx * rx + ry * ry
    return -0.25 * np.log(r2) / np.pi * g.weights[nc][None, :]


def lap_proxy_outgoing(g, rows, pts, pw):
    """kernels.py:347-352: target-normal dipole at proxy sources, transposed."""
    nr = np.asarray(rows, np.int64)
    pos = g.positions[nr]
    nrt = g.normals[nr]
    rx = pos[:, None, 0] - pts[None, :, 0]
    ry = pos[:, None, 1] - pts[None, :, 1]
    r2 = rx * rx + ry * ry
    blk = (rx * nrt[:, None, 0] + ry * nrt[:, None, 1]) / (2 * np.pi * r2)
    return (blk * pw[None, :]).T


def lap_nullspace_rows(g, cols):
    """kernels.py:368-370."""
    nc = np.asarray(cols, np.int64)
    return g.weights[nc][None, :], np.ones((1, len(nc)))


def lap_forward_block(g, targets, cols):
    """Interior rows, kernels.py:171-198 Laplace branch: u = -S mu."""
    targets = np.atleast_2d(np.asarray(targets, float))
    nc = np.asarray(cols, np.int64)
    pc = g.positions[nc]
    rx = targets[:, None, 0] - pc[None, :, 0]
    ry = targets[:, None, 1] - pc[None, :, 1]
    r2 = rx * rx + ry * ry
    return 0.5 * np.log(r2) / (2 * np.pi) * g.weights[nc][None, :]


def block(g, rows, cols, pde=STOKES):
    return self_block(g, rows, cols) if pde == STOKES else lap_self_block(g, rows, cols)


def dpn(pde):
    """SystemSpec.dof_per_node, kernels.py:52-54."""
    return 2 if pde == STOKES else 1


def id_stack(g, box_dofs, far, center, radius, count, pde=STOKES):
    """The stacked ID matrix of one box, skel.py:297-314."""
    nB = len(box_dofs)
    pts, pw = proxy_ring(center, radius, count)
    if pde == STOKES:
        pair, pin, pout, null = pair_blocks, proxy_incoming, proxy_outgoing, nullspace_rows
    else:
        pair, pin, pout, null = lap_pair_blocks, lap_proxy_incoming, lap_proxy_outgoing, lap_nullspace_rows
    e_in, e_out = null(g, box_dofs)
    if len(far):
        k_in, k_out = pair(g, far, box_dofs)
    else:
        k_in = k_out = np.zeros((0, nB))
    return np.vstack([k_in, pin(g, pts, box_dofs), e_in,
                      k_out, pout(g, box_dofs, pts, pw), e_out])


def aug_columns(points, centers, workers=1):
    """Stokeslet/rotlet columns H, kernels.py:201-223 (``workers`` threads over
    the centres: every column is computed by the same NumPy expressions)."""
    points = np.atleast_2d(np.asarray(points, float))
    centers = np.atleast_2d(np.asarray(centers, float))
    H = np.empty((2 * len(points), 3 * len(centers)))
    if workers > 1 and len(centers) > 1:
        with ThreadPoolExecutor(max_workers=workers) as ex:
            list(ex.map(lambda i: _aug_column(points, centers[i], i, H), range(len(centers))))
        return H
    for i, c in enumerate(centers):
        _aug_column(points, c, i, H)
    return H


def _aug_column(points, c, i, H):
    pref = 1.0 / (4 * np.pi)
    if True:
        r = points - c[None, :]
        r2 = (r * r).sum(axis=1)
        lg = -0.5 * np.log(r2)
        H[0::2, 3 * i] = pref * (lg + r[:, 0] * r[:, 0] / r2)
        H[1::2, 3 * i] = pref * (r[:, 1] * r[:, 0] / r2)
        H[0::2, 3 * i + 1] = pref * (r[:, 0] * r[:, 1] / r2)
        H[1::2, 3 * i + 1] = pref * (lg + r[:, 1] * r[:, 1] / r2)
        H[0::2, 3 * i + 2] = pref * (-r[:, 1]) / r2
        H[1::2, 3 * i + 2] = pref * r[:, 0] / r2


def aug_functionals(g):
    """Weighted rigid-body functionals Psi, kernels.py:238-245."""
    n = len(g.positions)
    Psi = np.zeros((2 * n, 3 * g.n_holes))
    for i in range(g.n_holes):
        ids = g.curve_nodes(i + 1)
        w = g.weights[ids]
        Psi[2 * ids, 3 * i] = w
        Psi[2 * ids + 1, 3 * i + 1] = w
        Psi[2 * ids, 3 * i + 2] = -g.positions[ids, 1] * w
        Psi[2 * ids + 1, 3 * i + 2] = g.positions[ids, 0] * w
    return Psi


def winding(points, poly, chunk=512):
    """Integer winding numbers of a closed polyline, geometry.py:221-233."""
    out = np.empty(len(points), dtype=np.int64)
    nxt = np.roll(poly, -1, axis=0)
    for s in range(0, len(points), chunk):
        p = points[s:s + chunk]
        a = poly[None, :, :] - p[:, None, :]
        b = nxt[None, :, :] - p[:, None, :]
        cross = a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0]
        dot = (a * b).sum(-1)
        ang = np.arctan2(cross, dot).sum(axis=1)
        out[s:s + chunk] = np.rint(ang / (2 * np.pi)).astype(np.int64)
    return out


def point_in_domain(g, points):
    """Boundary.point_in_domain, geometry.py:179-199 (winding + nearest node)."""
    from scipy.spatial import cKDTree
    pts = np.atleast_2d(np.asarray(points, float))
    inside = winding(pts, g.curves[0].nodes) != 0
    for c in g.curves[1:]:
        inside &= winding(pts, c.nodes) == 0
    d, _ = cKDTree(g.positions).query(pts)
    return inside & (d > 1e-12)


def forward_block(g, targets, cols):
    """Interior-evaluation rows (Stokes), kernels.py:171-198."""
    targets = np.atleast_2d(np.asarray(targets, float))
    nc, cc = _split(cols)
    pc = g.positions[nc]
    rx = targets[:, None, 0] - pc[None, :, 0]
    ry = targets[:, None, 1] - pc[None, :, 1]
    r2 = rx * rx + ry * ry
    w = g.weights[nc][None, :]
    nsc = g.normals[nc]
    rdn = rx * nsc[None, :, 0] + ry * nsc[None, :, 1]
    coef = rdn / (np.pi * r2 * r2) * w
    rcb = np.where((cc == 0)[None, :], rx, ry)
    out = np.empty((2 * len(targets), len(nc)))
    out[0::2] = coef * rx * rcb
    out[1::2] = coef * ry * rcb
    return out


def evaluate_interior(g, solution, targets, chunk=256, pde=STOKES):
    """u = D mu + H lam (Stokes, (m, 2)) or u = -S mu (Laplace, (m,)) at
    interior targets, skel.py:537-564."""
    targets = np.atleast_2d(np.asarray(targets, float))
    if not np.all(point_in_domain(g, targets)):
        raise ValueError("targets must lie strictly inside the domain")
    sol = np.asarray(solution, float)
    if pde == LAPLACE:
        nd = len(g.positions)
        mu = sol[:nd]
        out = np.empty(len(targets))
        for s in range(0, len(targets), chunk):
            out[s:s + chunk] = lap_forward_block(g, targets[s:s + chunk], np.arange(nd)) @ mu
        return out
    nd = 2 * len(g.positions)
    mu, lam = sol[:nd], sol[nd:]
    dofs = np.arange(nd)
    out = np.empty((len(targets), 2))
    for s in range(0, len(targets), chunk):
        tt = targets[s:s + chunk]
        vals = forward_block(g, tt, dofs) @ mu
        if len(lam):
            vals = vals + aug_columns(tt, g.hole_centers) @ lam
        out[s:s + chunk] = vals.reshape(-1, 2)
    return out


def dense_system(g, pde=STOKES):
    """Full (augmented) matrix, kernels.py:377-390."""
    nd = dpn(pde) * len(g.positions)
    A = block(g, np.arange(nd), np.arange(nd), pde)
    q = 3 * g.n_holes if pde == STOKES else 0
    if q == 0:
        return A
    M = np.zeros((nd + q, nd + q))
    M[:nd, :nd] = A
    M[:nd, nd:] = aug_columns(g.positions, g.hole_centers)
    M[nd:, :nd] = aug_functionals(g).T
    M[nd:, nd:] = -np.eye(q)
    return M


def exact_matvec(g, x, chunk=1024, pde=STOKES):
    """Uncompressed system product, kernels.py:393-414."""
    nd = dpn(pde) * len(g.positions)
    q = 3 * g.n_holes if pde == STOKES else 0
    x = np.asarray(x, float)
    out = np.empty(nd + q)
    allc = np.arange(nd)
    for s in range(0, nd, chunk):
        r = allc[s:s + chunk]
        out[s:s + len(r)] = block(g, r, allc, pde) @ x[:nd]
    if q:
        out[:nd] += aug_columns(g.positions, g.hole_centers) @ x[nd:]
        out[nd:] = aug_functionals(g).T @ x[:nd] - x[nd:]
    return out


# ---------------------------------------------------------------------------
# column-pivoted QR / ID and pivoted LU (dense.py)
# ---------------------------------------------------------------------------
class QRID:
    """Column-pivoted QR truncatable at any rank, dense.py:40-79."""

    def __init__(self, A):
        A = np.ascontiguousarray(A, dtype=float)
        self.ncols = A.shape[1]
        if A.size == 0:
            self.R = np.zeros((0, A.shape[1]))
            self.perm = np.arange(A.shape[1])
            self.diag = np.zeros(0)
            return
        if A.shape[0] > 2 * A.shape[1]:
            A = sla.qr(A, mode="r", check_finite=False)[0]
        _, self.R, self.perm = sla.qr(A, mode="economic", pivoting=True, check_finite=False)
        self.diag = np.abs(np.diag(self.R))

    def rank(self, tol):
        if len(self.diag) == 0 or self.diag[0] == 0.0:
            return 0
        return int(np.count_nonzero(self.diag > tol * self.diag[0]))

    def split(self, k):
        k = min(k, len(self.diag), self.ncols)
        if k == 0:
            T = np.zeros((0, self.ncols))
        else:
            T = sla.solve_triangular(self.R[:k, :k], self.R[:k, k:], lower=False)
        return self.perm[:k].copy(), self.perm[k:].copy(), T


class ZeroPivot(RuntimeError):
    def __init__(self, index):
        super().__init__(f"zero pivot at {index}")
        self.index = index


class LU:
    """Partially pivoted LU, dense.py:106-135."""

    def __init__(self, A):
        A = np.asarray(A, dtype=float)
        self.n = A.shape[0]
        if self.n == 0:
            self.f = None
            self.pivot_ratio = 1.0
            return
        self.f = sla.lu_factor(A, check_finite=False)
        d = np.abs(np.diag(self.f[0]))
        z = np.flatnonzero(d == 0.0)
        if len(z):
            raise ZeroPivot(int(z[0]))
        self.pivot_ratio = float(d.min() / d.max())

    def solve(self, B):
        B = np.asarray(B, dtype=float)
        if self.n == 0:
            return B.copy()
        return sla.lu_solve(self.f, B, check_finite=False)


# ---------------------------------------------------------------------------
# quadtree (tree.py)
# ---------------------------------------------------------------------------
class Node:
    __slots__ = ("key", "center", "hw", "parent", "nodes", "kids")

    def __init__(self, key, center, hw, parent, nodes):
        self.key, self.center, self.hw, self.parent, self.nodes = key, center, hw, parent, nodes
        self.kids = []

    @property
    def leaf(self):
        return not self.kids


class QTree:
    """Adaptive quadtree with geometric keys, tree.py:102-155."""

    def __init__(self, positions, leaf_cap=64, root_box=None, max_depth=40):
        positions = np.asarray(positions, float)
        if root_box is None:
            lo, hi = positions.min(axis=0), positions.max(axis=0)
            center = 0.5 * (lo + hi)
            hw = 0.5 * float((hi - lo).max()) * (1.0 + 0.1)
        else:
            center, hw = np.asarray(root_box[0], float), float(root_box[1])
            if np.any(np.abs(positions - center[None, :]) > hw * (1 + 1e-12)):
                raise ValueError("node outside the fixed root box")
        self.root_center, self.root_hw = center, hw
        self.leaf_cap, self.max_depth = leaf_cap, max_depth
        self.boxes = {}
        lev = {}
        todo = [((0, 0, 0), center.copy(), hw, np.arange(len(positions), dtype=np.int64), None)]
        while todo:
            key, ctr, half, ids, par = todo.pop()
            bx = Node(key, ctr, half, par, ids)
            self.boxes[key] = bx
            lev.setdefault(key[0], []).append(key)
            if len(ids) <= leaf_cap or key[0] >= max_depth:
                continue
            p = positions[ids]
            east = p[:, 0] >= ctr[0]
            north = p[:, 1] >= ctr[1]
            l, ix, iy = key
            for dx, dy in CHILD_ORDER:
                m = (east == bool(dx)) & (north == bool(dy))
                if m.any():
                    ck = (l + 1, 2 * ix + dx, 2 * iy + dy)
                    bx.kids.append(ck)
                    todo.append((ck, ctr + (np.array([dx, dy]) - 0.5) * half, half / 2, ids[m], key))
        self.levels = [sorted(lev.get(l, [])) for l in range(max(lev) + 1)]
        self.node_leaf = {}
        for k, bx in self.boxes.items():
            if bx.leaf:
                for n in bx.nodes:
                    self.node_leaf[int(n)] = k

    @property
    def depth(self):
        return len(self.levels) - 1

    def neighbours(self, key):
        """Same-level adjacent boxes, sorted (tree.py:70-81)."""
        l, ix, iy = key
        out = [(l, ix + a, iy + b) for a in (-1, 0, 1) for b in (-1, 0, 1)
               if (a or b) and (l, ix + a, iy + b) in self.boxes]
        return sorted(out)

    def coarse_leaves(self, center, radius, level):
        """Leaves above ``level`` meeting the disc, sorted (tree.py:83-99)."""
        out, st = [], [self.boxes[ROOT]]
        while st:
            bx = st.pop()
            if bx.key[0] >= level:
                continue
            d = np.maximum(np.abs(center - bx.center) - bx.hw, 0.0)
            if d[0] * d[0] + d[1] * d[1] > radius * radius:
                continue
            if bx.leaf:
                out.append(bx.key)
            else:
                st.extend(self.boxes[k] for k in bx.kids)
        return sorted(out)


def proxy_radius(hw, factor):
    """tree.py:158-160."""
    return factor * hw * np.sqrt(2.0)


# ---------------------------------------------------------------------------
# factorization (skel.py)
# ---------------------------------------------------------------------------
class BoxOut:
    __slots__ = ("key", "dofs", "S", "R", "T", "Xrr", "lu", "Xsr", "Xrs_div", "Xss")

    def __init__(self, **kw):
        for k, v in kw.items():
            setattr(self, k, v)

    @property
    def skel(self):
        return self.dofs[self.S]

    @property
    def red(self):
        return self.dofs[self.R]


class OracleFactorization:
    """Holds the per-box factors, mirrors skel.py:88-221."""

    def __init__(self, g, tree, tol, boxes, sweep, root_dofs, E_root, top,
                 UH, PsiV, UH_div, nonroot, stats):
        self.g, self.tree, self.tol = g, tree, tol
        self.boxes, self.sweep = boxes, sweep
        self.root_dofs, self.E_root, self.top = root_dofs, E_root, top
        self.UH, self.PsiV, self.UH_div, self.nonroot = UH, PsiV, UH_div, nonroot
        self.stats = stats
        self.pde = stats.get("pde", STOKES)
        self.nd = dpn(self.pde) * len(g.positions)
        self.q = 0 if UH is None else UH.shape[1]

    @property
    def dim(self):
        return self.nd + self.q

    def solve(self, rhs):
        """skel.py:166-221 (accepts (dim,) or (dim, nrhs))."""
        with threadpool_limits(limits=1):      # skel.py:176
            return self._solve(rhs)

    def _solve(self, rhs):
        x = np.array(rhs, dtype=float, copy=True)
        if x.shape[0] != self.dim:
            raise ValueError("dimension mismatch")
        nd = self.nd
        for _, keys in self.sweep:
            for k in keys:
                bf = self.boxes[k]
                sd, rd = bf.skel, bf.red
                r = bf.lu.solve(x[rd] - bf.T.T @ x[sd])
                x[sd] -= bf.Xsr @ r
                x[rd] = r
        if self.q:
            m = self.nonroot
            corr = x[nd:] - self.PsiV[m].T @ x[:nd][m]
            sol = self.top.solve(np.concatenate([x[self.root_dofs], corr]))
            ns = len(self.root_dofs)
            x[self.root_dofs] = sol[:ns]
            x[nd:] = sol[ns:]
            x[:nd][m] -= self.UH_div[m] @ sol[ns:]
        else:
            x[self.root_dofs] = self.top.solve(x[self.root_dofs])
        for _, keys in reversed(self.sweep):
            for k in keys:
                bf = self.boxes[k]
                sd, rd = bf.skel, bf.red
                x[rd] -= bf.Xrs_div @ x[sd]
                x[sd] -= bf.T @ x[rd]
        return x

    def apply(self, x):
        """skel.py:126-164 (vector)."""
        with threadpool_limits(limits=1):      # skel.py:132
            return self._apply(x)

    def _apply(self, x):
        x = np.asarray(x, float)
        nd = self.nd
        y = x[:nd].copy()
        lam = x[nd:]
        for _, keys in self.sweep:
            for k in keys:
                bf = self.boxes[k]
                y[bf.skel] += bf.T @ y[bf.red]
                y[bf.red] += bf.Xrs_div @ y[bf.skel]
        bottom = self.PsiV.T @ y - lam if self.q else np.zeros(0)
        keep = {}
        for _, keys in self.sweep:
            for k in keys:
                bf = self.boxes[k]
                keep[k] = y[bf.red].copy()
                y[bf.red] = bf.Xrr @ y[bf.red]
        y[self.root_dofs] = self.E_root @ y[self.root_dofs]
        if self.q:
            y += self.UH @ lam
        for _, keys in reversed(self.sweep):
            for k in keys:
                bf = self.boxes[k]
                t = keep[k]
                if self.q:
                    t = t + self.UH_div[bf.red] @ lam
                y[bf.skel] += bf.Xsr @ t
                y[bf.red] += bf.T.T @ y[bf.skel]
        return np.concatenate([y, bottom])


class _Pass:
    """State of one factor pass (skel.py:227-361)."""

    def __init__(self, g, tree, tol, count, factor, pde=STOKES, propagate_zeros=False):
        self.g, self.tree, self.tol, self.count, self.factor = g, tree, tol, count, factor
        self.pde = pde
        self.propagate_zeros = propagate_zeros          # skel.py:267-270, 354-361
        self.done = set()
        self.dpn = dpn(pde)
        self.dof_xy = np.repeat(g.positions, self.dpn, axis=0)        # skel.py:233
        self.active = {}
        self.out = {}
        self.record = None   # optional dict key -> per-box debug data

    def leaf_dofs(self, bx):
        """dofs_of_nodes, skel.py:243-244."""
        return (self.dpn * bx.nodes[:, None] + np.arange(self.dpn)[None, :]).ravel()

    def far(self, bx):
        """skel.py:258-280 (first tuple element)."""
        rp = proxy_radius(bx.hw, self.factor)
        parts = [self.out[k].skel if (self.propagate_zeros and k in self.done) else self.active[k]
                 for k in self.tree.neighbours(bx.key)]
        parts += [self.active[k] for k in self.tree.coarse_leaves(bx.center, rp, bx.key[0])]
        if not parts:
            return np.empty(0, dtype=np.int64)
        cand = np.concatenate(parts)
        d2 = ((self.dof_xy[cand] - bx.center[None, :]) ** 2).sum(axis=1)
        return cand[d2 < rp * rp]

    def block_E(self, bx):
        """skel.py:282-291."""
        E = block(self.g, self.active[bx.key], self.active[bx.key], self.pde)
        off = 0
        for ck in bx.kids:
            c = self.out[ck]
            n = len(c.S)
            E[off:off + n, off:off + n] = c.Xss
            off += n
        return E

    def compress(self, key):
        """skel.py:293-338."""
        bx = self.tree.boxes[key]
        B = self.active[key]
        nB = len(B)
        F = self.far(bx)
        A = id_stack(self.g, B, F, bx.center, proxy_radius(bx.hw, self.factor), self.count, self.pde)
        qr = QRID(A)
        k = qr.rank(self.tol)
        E = self.block_E(bx)
        while True:
            S, R, T = qr.split(k)
            Ess = E[np.ix_(S, S)]
            Xrr = (E[np.ix_(R, R)] - T.T @ E[np.ix_(S, R)] - E[np.ix_(R, S)] @ T + T.T @ Ess @ T)
            try:
                lu = LU(Xrr)
                if lu.pivot_ratio >= PIVOT_FLOOR or k >= nB:
                    break
            except ZeroPivot:
                if k >= nB:
                    raise
            k = min(nB, k + max(1, (nB - k) // 8))
        Xrs = E[np.ix_(R, S)] - T.T @ Ess
        Xsr = E[np.ix_(S, R)] - Ess @ T
        Xrs_div = lu.solve(Xrs)
        if self.record is not None:
            self.record[key] = dict(far=F, stack=A, perm=qr.perm, diag=qr.diag, k=k, T=T)
        return BoxOut(key=key, dofs=B, S=S, R=R, T=T, Xrr=Xrr, lu=lu, Xsr=Xsr,
                      Xrs_div=Xrs_div, Xss=Ess - Xsr @ Xrs_div)

    def run(self, workers=1, reuse=None, dirty=None):
        t = self.tree
        for k, bx in t.boxes.items():
            if bx.leaf:
                self.active[k] = self.leaf_dofs(bx)
        sweep = []
        for lev in range(t.depth, 0, -1):
            keys = t.levels[lev]
            for k in keys:
                bx = t.boxes[k]
                if not bx.leaf:
                    self.active[k] = np.concatenate([self.out[c].skel for c in bx.kids])
            todo = [k for k in keys if reuse is None or k in dirty]
            for k in keys:
                if reuse is not None and k not in dirty:
                    self.out[k] = reuse[k]
            if workers > 1 and len(todo) > 1 and not self.propagate_zeros:
                with ThreadPoolExecutor(max_workers=workers) as ex:
                    for k, r in zip(todo, ex.map(self.compress, todo)):
                        self.out[k] = r
            else:
                for k in todo:
                    self.out[k] = self.compress(k)
                    self.done.add(k)
            sweep.append((lev, keys))
        return sweep

    def _sweep_box(self, k, UH, PsiV, UH_div):
        """One box of the augmentation sweep (skel.py:384-395); returns its
        q x q Schur contribution PsiV_R^T w."""
        bf = self.out[k]
        sd, r = bf.skel, bf.red
        UH[r] -= bf.T.T @ UH[sd]
        w = bf.lu.solve(UH[r])
        UH[sd] -= bf.Xsr @ w
        UH_div[r] = w
        PsiV[r] -= bf.T.T @ PsiV[sd]
        PsiV[sd] -= bf.Xrs_div.T @ PsiV[r]
        return PsiV[r].T @ w

    def top(self, sweep, workers=1):
        """_finish_top, skel.py:364-425.  With ``workers`` > 1 the boxes of a
        level run on threads (they touch disjoint rows) and their Schur
        contributions are added in box order: bitwise the serial result."""
        g, t = self.g, self.tree
        root = t.boxes[ROOT]
        if root.leaf:
            rd = self.leaf_dofs(root)
        else:
            rd = np.concatenate([self.out[c].skel for c in root.kids])
        self.active[ROOT] = rd
        E_root = self.block_E(root)
        nd = self.dpn * len(g.positions)
        q = 3 * g.n_holes if self.pde == STOKES else 0        # SystemSpec.augmented, kernels.py:59-60
        UH = PsiV = UH_div = None
        nonroot = np.ones(nd, dtype=bool)
        nonroot[rd] = False
        if q:
            UH = aug_columns(g.positions, g.hole_centers, workers)
            PsiV = aug_functionals(g)
            UH_div = np.zeros_like(UH)
            schur = np.zeros((q, q))
            ex = ThreadPoolExecutor(max_workers=workers) if workers > 1 else None
            try:
                for _, keys in sweep:
                    if ex is not None and len(keys) > 1:
                        parts = list(ex.map(lambda k: self._sweep_box(k, UH, PsiV, UH_div), keys))
                    else:
                        parts = [self._sweep_box(k, UH, PsiV, UH_div) for k in keys]
                    for part in parts:
                        schur += part
            finally:
                if ex is not None:
                    ex.shutdown()
            ns = len(rd)
            C = np.zeros((ns + q, ns + q))
            C[:ns, :ns] = E_root
            C[:ns, ns:] = UH[rd]
            C[ns:, :ns] = PsiV[rd].T
            C[ns:, ns:] = -np.eye(q) - schur
            top = LU(C)
        else:
            top = LU(E_root)
        kpl = {lev: max((len(self.out[k].S) for k in keys), default=0) for lev, keys in sweep}
        return OracleFactorization(g, t, self.tol, dict(self.out), sweep, rd, E_root, top,
                                   UH, PsiV, UH_div, nonroot,
                                   {"k_per_level": kpl, "root_size": len(rd), "pde": self.pde})


def factor(g, tree, tol, proxy_count=64, proxy_factor=1.5, workers=1, record=None, pde=STOKES,
           propagate_zeros=False):
    """skel.py:428-453."""
    t0 = time.perf_counter()
    with threadpool_limits(limits=1):          # skel.py:441
        p = _Pass(g, tree, tol, proxy_count, proxy_factor, pde, propagate_zeros)
        p.record = record
        sweep = p.run(workers)
        f = p.top(sweep, workers)
    f.stats["factor_time"] = time.perf_counter() - t0
    return f


# ---------------------------------------------------------------------------
# update bookkeeping (skel.py:456-534, tree.py:215-270)
# ---------------------------------------------------------------------------
def changed_owners(t_new, t_old, old_to_new):
    """tree.py:251-270."""
    out = set()
    for key, bx in t_new.boxes.items():
        tw = t_old.boxes.get(key)
        if tw is None:
            out.add(key)
            continue
        m = old_to_new[tw.nodes]
        if len(m) != len(bx.nodes) or np.any(m < 0) or not np.array_equal(m, bx.nodes):
            out.add(key)
    for key in t_old.boxes:
        if key not in t_new.boxes:
            p = key
            while p is not None and p not in t_new.boxes:
                p = t_old.boxes[p].parent
            if p is not None:
                out.add(p)
    return out


def disc_hits(t, pts, factor, out):
    """tree.py:215-236."""
    for lev, keys in enumerate(t.levels):
        if not keys:
            continue
        hw = t.root_hw / 2 ** lev
        rad = proxy_radius(hw, factor)
        step = 2 * hw
        origin = t.root_center - t.root_hw
        cells = np.floor((pts - origin[None, :]) / step).astype(np.int64)
        reach = int(np.ceil(rad / step)) + 1
        cand = set()
        for cx, cy in {(int(a), int(b)) for a, b in cells}:
            for dx in range(-reach, reach + 1):
                for dy in range(-reach, reach + 1):
                    k = (lev, cx + dx, cy + dy)
                    if k in t.boxes:
                        cand.add(k)
        for k in cand:
            d2 = ((pts - t.boxes[k].center[None, :]) ** 2).sum(axis=1)
            if (d2 <= rad * rad).any():
                out.add(k)


def dirty_set(t_old, t_new, b_new, report, factor):
    """Dirty boxes of an update, skel.py:476-491 + _dirty_closure skel.py:517-534."""
    content = set(changed_owners(t_new, t_old, report.old_to_new))
    pts = []
    if len(report.modified_nodes_old):
        pts.append(report.old_positions[report.modified_nodes_old])
    if len(report.modified_nodes_new):
        pts.append(b_new.positions[report.modified_nodes_new])
    pts = np.concatenate(pts) if pts else np.zeros((0, 2))
    if len(pts):
        disc_hits(t_new, pts, factor, content)
    for nid in report.modified_nodes_new:
        key = t_new.node_leaf[int(nid)]
        while key is not None and key not in content:
            content.add(key)
            key = t_new.boxes[key].parent
    marked = {l: set() for l in range(len(t_new.levels))}
    for k in content:
        marked[k[0]].add(k)
    for lev in range(len(t_new.levels) - 1, -1, -1):
        grow = set(marked[lev])
        if lev + 1 < len(t_new.levels):
            for k in marked[lev + 1]:
                p = t_new.boxes[k].parent
                if p is not None:
                    grow.add(p)
        for k in list(grow):
            grow.update(t_new.neighbours(k))
        marked[lev] = grow
    out = set()
    for s in marked.values():
        out |= s
    return out


def update(fct, b_new, report, workers=1):
    """skel.py:456-514: recompress dirty boxes, reuse clean ones (identity DOF map for moves)."""
    t0 = time.perf_counter()
    t_new = QTree(b_new.positions, fct.tree.leaf_cap, (fct.tree.root_center, fct.tree.root_hw),
                  fct.tree.max_depth)
    dirty = dirty_set(fct.tree, t_new, b_new, report, fct.proxy_factor)
    with threadpool_limits(limits=1):          # skel.py:469
        p = _Pass(b_new, t_new, fct.tol, fct.proxy_count, fct.proxy_factor, fct.pde)
        sweep = p.run(workers, reuse=fct.boxes, dirty=dirty)
        f = p.top(sweep, workers)
    f.proxy_count, f.proxy_factor = fct.proxy_count, fct.proxy_factor
    f.stats["update_time"] = time.perf_counter() - t0
    f.stats["n_dirty"] = len(dirty)
    f.stats["dirty"] = dirty
    return f


def factor_full(g, leaf_cap, tol, proxy_count, proxy_factor, workers=1, record=None, pde=STOKES,
                propagate_zeros=False):
    t = QTree(g.positions, leaf_cap)
    f = factor(g, t, tol, proxy_count, proxy_factor, workers, record, pde, propagate_zeros)
    f.proxy_count, f.proxy_factor = proxy_count, proxy_factor
    return f
