"""Boundary geometry: struct-of-arrays node data for an outer curve plus holes.

Mirrors the data contract of the reference ``Boundary`` (reference
``pkg/src/skelsolve/geometry.py:122-218``): node data of all curves is
concatenated (outer curve first, then holes), ``hole_centers`` is the node mean
of each hole (``geometry.py:149-150``), scalar DOFs are ``2*node + comp``.

Curves are built analytically (the synthetic workloads in SURVEY.md §8(d)),
bypassing the reference's spline fit; a reference ``Boundary`` built from the
same arrays is bit-identical input.  Hole moves (``MoveHole``) follow
``apply_perturbation`` (``geometry.py:328-395``): rigid translation, weights,
normals and curvatures carried over bitwise.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class GeometryError(ValueError):
    """Invalid arrangement (reference ``geometry.py:32``)."""


OUTER = "outer"
HOLE = "hole"


@dataclass
class Curve:
    """One discretised closed curve (reference ``Curve``, ``geometry.py:79-100``)."""

    nodes: np.ndarray        # (n, 2)
    weights: np.ndarray      # (n,)
    normals: np.ndarray      # (n, 2), out of the fluid
    curvatures: np.ndarray   # (n,)
    orientation: str = OUTER
    # analytic bounding radius about the node mean (used by the fast overlap check)
    bound_radius: float = 0.0

    @property
    def n_nodes(self) -> int:
        return len(self.nodes)

    def translated(self, shift) -> "Curve":
        shift = np.asarray(shift, float)
        return Curve(self.nodes + shift, self.weights, self.normals, self.curvatures,
                     self.orientation, self.bound_radius)


class Boundary:
    """Outer curve + holes, node data concatenated (reference ``geometry.py:122-150``)."""

    def __init__(self, curves: list[Curve]):
        if not curves or curves[0].orientation != OUTER:
            raise GeometryError("first curve must be the outer boundary")
        if any(c.orientation != HOLE for c in curves[1:]):
            raise GeometryError("curves after the first must be holes")
        self.curves = list(curves)
        self.positions = np.ascontiguousarray(np.concatenate([c.nodes for c in curves]))
        self.weights = np.ascontiguousarray(np.concatenate([c.weights for c in curves]))
        self.normals = np.ascontiguousarray(np.concatenate([c.normals for c in curves]))
        self.curvatures = np.ascontiguousarray(np.concatenate([c.curvatures for c in curves]))
        self.offsets = np.concatenate([[0], np.cumsum([c.n_nodes for c in curves])])
        # same numpy expression as the reference so the bits agree
        centers = [c.nodes.mean(axis=0) for c in curves[1:]]
        self.hole_centers = np.array(centers).reshape(-1, 2)

    @property
    def n_nodes(self) -> int:
        return len(self.positions)

    @property
    def n_holes(self) -> int:
        return len(self.curves) - 1

    def curve_nodes(self, c: int) -> np.ndarray:
        return np.arange(self.offsets[c], self.offsets[c + 1])

    def point_in_domain(self, points) -> np.ndarray:
        """Strictly inside the fluid domain (reference geometry.py:179-192); the
        winding numbers run on the GPU (skel.point_in_domain)."""
        from .skel import point_in_domain
        return point_in_domain(self, points)

    def curve_of_node(self) -> np.ndarray:
        out = np.empty(self.n_nodes, dtype=np.int64)
        for c in range(len(self.curves)):
            out[self.offsets[c]:self.offsets[c + 1]] = c
        return out


# ---------------------------------------------------------------------------
# analytic curves (theta_j = 2 pi j / n, w = |x'| 2pi/n,
# n = (tau_y, -tau_x), kappa = (x'y'' - y'x'')/|x'|^3; holes clockwise)
# ---------------------------------------------------------------------------
def _curve_from_derivs(x, d1, d2, orientation, bound_radius=0.0) -> Curve:
    n = len(x)
    speed = np.sqrt(d1[:, 0] ** 2 + d1[:, 1] ** 2)
    tau = d1 / speed[:, None]
    normals = np.stack([tau[:, 1], -tau[:, 0]], axis=1)
    weights = speed * (2 * np.pi / n)
    curv = (d1[:, 0] * d2[:, 1] - d1[:, 1] * d2[:, 0]) / speed ** 3
    return Curve(np.ascontiguousarray(x), weights, np.ascontiguousarray(normals), curv,
                 orientation, bound_radius)


def star_curve(n: int, arms: int = 5, amp: float = 0.3, scale: float = 1.0) -> Curve:
    """Outer star r(t) = scale (1 + amp cos(arms t)), counterclockwise."""
    t = 2 * np.pi * np.arange(n) / n
    r = scale * (1 + amp * np.cos(arms * t))
    dr = -scale * amp * arms * np.sin(arms * t)
    ddr = -scale * amp * arms * arms * np.cos(arms * t)
    c, s = np.cos(t), np.sin(t)
    x = np.stack([r * c, r * s], axis=1)
    d1 = np.stack([dr * c - r * s, dr * s + r * c], axis=1)
    d2 = np.stack([ddr * c - 2 * dr * s - r * c, ddr * s + 2 * dr * c - r * s], axis=1)
    return _curve_from_derivs(x, d1, d2, OUTER, scale * (1 + amp))


def ellipse_curve(n: int, center=(0.0, 0.0), a: float = 1.0, b: float = 1.0,
                  phi: float = 0.0, clockwise: bool = False, phase: float = 0.0) -> Curve:
    """Ellipse with semi-axes (a, b) rotated by phi; clockwise for holes.
    ``phase`` shifts the node parameters (t_j = 2 pi j / n + phase)."""
    t = 2 * np.pi * np.arange(n) / n
    if phase:
        t = t + phase
    sg = -1.0 if clockwise else 1.0
    c, s = np.cos(t), np.sin(t)
    lx, ly = a * c, sg * b * s
    dlx, dly = -a * s, sg * b * c
    ddlx, ddly = -a * c, -sg * b * s
    cp, sp = np.cos(phi), np.sin(phi)

    def rot(u, v):
        return np.stack([cp * u - sp * v, sp * u + cp * v], axis=1)

    x = rot(lx, ly) + np.asarray(center, float)[None, :]
    return _curve_from_derivs(x, rot(dlx, dly), rot(ddlx, ddly),
                              HOLE if clockwise else OUTER, max(a, b))


def circle_curve(n: int, center=(0.0, 0.0), radius: float = 1.0,
                 clockwise: bool = False, phase: float = 0.0) -> Curve:
    return ellipse_curve(n, center, radius, radius, 0.0, clockwise, phase)


# ---------------------------------------------------------------------------
# perturbations (reference geometry.py:281-395: MoveHole, AddHole, DeleteHole + reports)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class MoveHole:
    curve_id: int
    translation: tuple | None = None
    new_center: tuple | None = None


@dataclass(frozen=True, eq=False)
class AddHole:
    """A new hole, appended after the kept curves (reference ``geometry.py:289-291``).
    The reference discretises a ``CurveSpec`` by its spline fit; here the hole is
    handed over discretised (a ``Curve`` from the analytic builders or from node
    arrays), optionally re-centred."""
    curve: Curve
    center: tuple | None = None


@dataclass(frozen=True)
class DeleteHole:
    """Remove hole ``curve_id`` (reference ``geometry.py:294-296``)."""
    curve_id: int


@dataclass
class PerturbationReport:
    """Changed nodes in old/new numbering (reference ``geometry.py:302-321``):
    ``old_to_new`` maps an old node to its new index (-1: deleted);
    ``modified_nodes_old`` lists moved and deleted curves' nodes,
    ``modified_nodes_new`` moved and added ones."""

    modified_nodes_old: np.ndarray
    modified_nodes_new: np.ndarray
    old_to_new: np.ndarray
    old_positions: np.ndarray


def check_arrangement(b: Boundary, gap: float = 0.0):
    """Analytic overlap test using each curve's bounding radius.

    The reference validates with winding numbers (``geometry.py:256-275``);
    for the synthetic circle/ellipse holes a bounding-circle test is a
    conservative equivalent and O(p^2) on p centres only.
    """
    outer = b.curves[0]
    r_out = np.sqrt((outer.nodes ** 2).sum(axis=1)).min()
    ctr = b.hole_centers
    rad = np.array([c.bound_radius for c in b.curves[1:]])
    if len(ctr) == 0:
        return
    if np.any(np.sqrt((ctr ** 2).sum(axis=1)) + rad + gap >= r_out):
        raise GeometryError("hole not inside the outer curve")
    d = np.sqrt(((ctr[:, None, :] - ctr[None, :, :]) ** 2).sum(-1))
    lim = rad[:, None] + rad[None, :] + gap
    np.fill_diagonal(d, np.inf)
    if np.any(d < lim):
        raise GeometryError("holes overlap")


def apply_perturbation(b: Boundary, edits, gap: float = 0.0):
    """Apply MoveHole / DeleteHole / AddHole edits; returns (new boundary,
    report) with the reference's node bookkeeping (``geometry.py:328-390``):
    kept curves in their old order, added holes appended."""
    if not edits:
        return b, PerturbationReport(np.empty(0, np.int64), np.empty(0, np.int64),
                                     np.arange(b.n_nodes), b.positions)
    curves = list(b.curves)
    touched, added = [], []
    for e in edits:
        if isinstance(e, (MoveHole, DeleteHole)):
            if not (1 <= e.curve_id < len(curves)):
                raise GeometryError(f"curve {e.curve_id} is not a hole")
            cur = curves[e.curve_id]
            if cur is None:
                raise GeometryError(f"curve {e.curve_id} already deleted")
            if isinstance(e, DeleteHole):
                curves[e.curve_id] = None
            else:
                if e.new_center is not None:
                    shift = np.asarray(e.new_center, float) - cur.nodes.mean(axis=0)
                else:
                    shift = np.asarray(e.translation, float)
                curves[e.curve_id] = cur.translated(shift)
            touched.append(e.curve_id)
        elif isinstance(e, AddHole):
            c = e.curve
            if c.orientation != HOLE:
                raise GeometryError("an added curve must be a hole")
            if e.center is not None:
                c = c.translated(np.asarray(e.center, float) - c.nodes.mean(axis=0))
            added.append(c)
        else:
            raise GeometryError(f"unsupported edit {e!r}")
    kept = [c for c in curves if c is not None] + added
    b_new = Boundary(kept)
    check_arrangement(b_new, gap)
    old_to_new = np.full(b.n_nodes, -1, dtype=np.int64)
    pos, new_ids = 0, {}
    for old_id, c in enumerate(curves):
        if c is None:
            continue
        n = c.n_nodes
        old_to_new[b.offsets[old_id]:b.offsets[old_id] + n] = np.arange(pos, pos + n)
        new_ids[old_id] = len(new_ids)
        pos += n
    mod = sorted(set(touched))
    nodes_old = (np.concatenate([b.curve_nodes(c) for c in mod]) if mod else np.empty(0, np.int64))
    moved_new = [new_ids[c] for c in mod if curves[c] is not None]
    added_new = list(range(len(kept) - len(added), len(kept)))
    nodes_new = (np.concatenate([b_new.curve_nodes(c) for c in moved_new + added_new])
                 if (moved_new or added_new) else np.empty(0, np.int64))
    return b_new, PerturbationReport(nodes_old, np.sort(nodes_new), old_to_new, b.positions)
