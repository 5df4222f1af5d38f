"""Seeded synthetic workloads of BASELINE.json ``configs``.

Every geometry is analytic and fed as the *same* arrays to the GPU path and to
the CPU oracle.  BASELINE's "proxy circle at radius 1.5x box half-width" is the
reference's ``proxy_factor = 1.5/sqrt(2)`` (reference ``tree.py:158-160`` uses
factor x circumradius).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .geometry import (Boundary, GeometryError, MoveHole, apply_perturbation,
                       check_arrangement, circle_curve, ellipse_curve, star_curve)

PROXY_FACTOR_BASELINE = 1.5 / np.sqrt(2.0)


@dataclass
class Workload:
    name: str
    boundary: Boundary
    tol: float
    leaf_cap: int
    proxy_count: int
    proxy_factor: float = PROXY_FACTOR_BASELINE
    seed: int = 0
    extra: dict = field(default_factory=dict)

    @property
    def n_unknowns(self) -> int:
        return 2 * self.boundary.n_nodes + 3 * self.boundary.n_holes


def stokeslet_columns(points, centers) -> np.ndarray:
    """Stokeslet/rotlet velocity columns (3 per centre), reference ``kernels.py:201-223``."""
    points = np.atleast_2d(np.asarray(points, float))
    centers = np.atleast_2d(np.asarray(centers, float))
    m, p = len(points), len(centers)
    H = np.empty((2 * m, 3 * p))
    pref = 1.0 / (4 * np.pi)
    for i, c in enumerate(centers):
        r = points - c[None, :]
        r2 = (r * r).sum(axis=1)
        lg = -0.5 * np.log(r2)
        H[0::2, 3 * i] = pref * (lg + r[:, 0] * r[:, 0] / r2)
        H[1::2, 3 * i] = pref * (r[:, 1] * r[:, 0] / r2)
        H[0::2, 3 * i + 1] = pref * (r[:, 0] * r[:, 1] / r2)
        H[1::2, 3 * i + 1] = pref * (lg + r[:, 1] * r[:, 1] / r2)
        H[0::2, 3 * i + 2] = pref * (-r[:, 1]) / r2
        H[1::2, 3 * i + 2] = pref * r[:, 0] / r2
    return H


def _sample_centers(rng, n, radius_fn, sep_fn, disc_fn, max_tries=200000):
    centers, radii = [], []
    tries = 0
    while len(centers) < n:
        tries += 1
        if tries > max_tries:
            raise RuntimeError("could not place holes")
        rad = radius_fn()
        R = disc_fn(rad)
        u, v = rng.random(2)
        c = np.array([R * np.sqrt(u) * np.cos(2 * np.pi * v), R * np.sqrt(u) * np.sin(2 * np.pi * v)])
        ok = all(np.hypot(*(c - cj)) >= sep_fn(rad, rj) for cj, rj in zip(centers, radii))
        if ok:
            centers.append(c)
            radii.append(rad)
    return centers, radii


def cfg1(seed: int = 0, n: int = 4096) -> Workload:
    """Simply connected star r = 1 + 0.3 cos 5t; RHS = field of 4 exterior Stokeslets."""
    b = Boundary([star_curve(n)])
    rng = np.random.default_rng(seed)
    ang = rng.uniform(0, 2 * np.pi, 4)
    rad = rng.uniform(1.6, 2.5, 4)
    src = np.stack([rad * np.cos(ang), rad * np.sin(ang)], axis=1)
    alpha = rng.standard_normal((4, 2))
    H = stokeslet_columns(b.positions, src)
    f = np.zeros(2 * n)
    for i in range(4):
        f += H[:, 3 * i] * alpha[i, 0] + H[:, 3 * i + 1] * alpha[i, 1]
    return Workload("cfg1_star_N4096", b, 1e-10, 64, 64, seed=seed,
                    extra={"rhs": f, "sources": src, "alpha": alpha})


def holes_circle(seed: int, R: float, n_outer: int, n_holes: int, r_hole: float,
                 n_per_hole: int, sep: float, disc: float, phases: bool = False) -> Boundary:
    """Outer circle + circular holes.  ``phases`` rotates every curve's node
    parameters by a seeded offset, breaking the mirror symmetries of equispaced
    circles that create exact pivot ties (used by the small strict-parity case)."""
    rng = np.random.default_rng(seed)
    cs, _ = _sample_centers(rng, n_holes, lambda: r_hole, lambda a, b: sep, lambda a: disc)
    ph = rng.uniform(0, 2 * np.pi, n_holes + 1) if phases else np.zeros(n_holes + 1)
    curves = [circle_curve(n_outer, radius=R, phase=ph[0])]
    curves += [circle_curve(n_per_hole, c, r_hole, clockwise=True, phase=ph[i + 1])
               for i, c in enumerate(cs)]
    return Boundary(curves)


def cfg2(seed: int = 0, phases: bool = True) -> Workload:
    """Outer circle R=10 (8192 nodes) + 16 holes r=0.5 (1024 nodes), centres sep >= 1.5.
    ``phases=False`` keeps every curve's nodes at t_j = 2 pi j / n: the mirror
    symmetries of equispaced circles then produce exact QRCP pivot ties (the
    tie-rich parity fixture)."""
    b = holes_circle(seed, 10.0, 8192, 16, 0.5, 1024, 1.5, 8.5, phases=phases)
    rng = np.random.default_rng(seed + 1000)
    f = rng.standard_normal(2 * b.n_nodes)
    rhs = np.concatenate([f, np.zeros(3 * b.n_holes)])
    return Workload("cfg2_16holes_N24576" + ("" if phases else "_unphased"), b, 1e-10, 64, 64,
                    seed=seed, extra={"rhs": rhs})


def cfg3(seed: int = 0) -> Workload:
    """Outer circle R=40 (16384 nodes) + 256 ellipses (512 nodes); eps 1e-8, leaf 128, P 96."""
    rng = np.random.default_rng(seed)
    R = 40.0
    params = []
    while len(params) < 256:
        a = rng.uniform(0.3, 0.9)
        bb = a / rng.uniform(1.0, 3.0)
        phi = rng.uniform(0, np.pi)
        lim = R - a - 0.5
        for _ in range(100000):
            u, v = rng.random(2)
            c = np.array([lim * np.sqrt(u) * np.cos(2 * np.pi * v), lim * np.sqrt(u) * np.sin(2 * np.pi * v)])
            if all(np.hypot(*(c - pc)) >= a + pa + 0.2 for pc, pa, _, _ in params):
                params.append((c, a, bb, phi))
                break
        else:
            raise RuntimeError("could not place ellipse")
    ph = rng.uniform(0, 2 * np.pi, len(params) + 1)
    curves = [circle_curve(16384, radius=R, phase=ph[0])]
    curves += [ellipse_curve(512, c, a, bb, phi, clockwise=True, phase=ph[i + 1])
               for i, (c, a, bb, phi) in enumerate(params)]
    b = Boundary(curves)
    return Workload("cfg3_256ellipses_N147456", b, 1e-8, 128, 96, seed=seed)


def cfg5_rhs(b: Boundary, nrhs: int = 256, seed: int = 5) -> np.ndarray:
    rng = np.random.default_rng(seed)
    F = rng.standard_normal((2 * b.n_nodes, nrhs))
    return np.concatenate([F, np.zeros((3 * b.n_holes, nrhs))], axis=0)


def mini_holes(seed: int = 0, n_outer: int = 1024, n_holes: int = 3, n_per_hole: int = 256,
               R: float = 3.0) -> Workload:
    """Small multiply-connected case for fast parity tests."""
    b = holes_circle(seed, R, n_outer, n_holes, 0.5, n_per_hole, 1.5, R - 1.0, phases=True)
    rng = np.random.default_rng(seed + 7)
    rhs = np.concatenate([rng.standard_normal(2 * b.n_nodes), np.zeros(3 * n_holes)])
    return Workload(f"mini_{n_holes}holes", b, 1e-10, 64, 64, seed=seed, extra={"rhs": rhs})


def interior_targets(b: Boundary, m: int, seed: int = 9, exterior: int = 0) -> np.ndarray:
    """Seeded evaluation points inside the fluid domain (inside the outer curve
    at radius < 0.9 of its smallest node radius, >= 0.1 away from every hole's
    bounding circle), plus ``exterior`` points inside holes / outside the
    outer curve for the rejection path."""
    rng = np.random.default_rng(seed)
    rmin = np.sqrt((b.curves[0].nodes ** 2).sum(axis=1)).min()
    ctr = b.hole_centers
    rad = np.array([c.bound_radius for c in b.curves[1:]])
    out = []
    while len(out) < m:
        u, v = rng.random(2)
        p = 0.9 * rmin * np.sqrt(u) * np.array([np.cos(2 * np.pi * v), np.sin(2 * np.pi * v)])
        if len(ctr) and np.any(np.sqrt(((ctr - p) ** 2).sum(axis=1)) < rad + 0.1):
            continue
        out.append(p)
    ext = [ctr[i % len(ctr)] for i in range(exterior)] if len(ctr) else []
    ext += [np.array([2.0 * rmin, 0.0])] * (exterior - len(ext))
    return np.array(out + ext).reshape(-1, 2)


def hole_move_sequence(b: Boundary, steps: int, seed: int = 4, step_len: float = 0.1,
                       gap: float = 0.2):
    """cfg4: successive random hole moves of norm ``step_len`` (overlaps rejected)."""
    rng = np.random.default_rng(seed)
    out = []
    cur = b
    while len(out) < steps:
        h = int(rng.integers(1, cur.n_holes + 1))
        th = rng.uniform(0, 2 * np.pi)
        d = (step_len * np.cos(th), step_len * np.sin(th))
        try:
            nb, rep = apply_perturbation(cur, [MoveHole(h, translation=d)], gap=gap)
        except GeometryError:
            continue
        out.append((h, d, nb, rep))
        cur = nb
    return out


def by_name(name: str) -> Workload:
    return {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "mini": mini_holes}[name]()
