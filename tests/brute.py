"""Independent brute-force references used to PIN the oracle (test helpers, numpy/scipy only).

Nothing here is imported by the oracle or the CUDA path.  Each helper is a different algorithm from
the oracle's face-loop clipper, so that a mistake in the oracle cannot be reproduced here:

* `vertex_enumeration_cell` -- intersect every triple of planes (bisectors + 6 walls), keep the
  points satisfying all half-spaces, hull them: faces, areas, volume (SPEC.md:145 [DERIVED] idea).
* `separable_grid_cells` -- exact rational 1-D lower envelopes for sites X_a x Y_b x Z_c with
  weights f_a + g_b + h_c, whose 3-D power cells are products of 1-D cells.
* `lifted_adjacency` -- regular-triangulation adjacency from scipy's 4-D Qhull lower hull of the
  lifted points (x, |x|^2 - w) ("Convex-hull lifting").
* `power_argmin` -- brute-force owner argmin_k |x - p_k|^2 - w_k  (Eq. 1).
"""
from __future__ import annotations

import itertools
from fractions import Fraction

import numpy as np


def planes_for_cell(points, weights, box, i):
    """All half-spaces n.x <= d bounding cell i, in WORLD coordinates (Eq. 1 expanded):
    2 x.(p_j - p_i) <= |p_j|^2 - |p_i|^2 + w_i - w_j, plus the 6 box walls.  Tags: j or -1-k."""
    p = np.asarray(points, np.float64)
    w = np.zeros(len(p)) if weights is None else np.asarray(weights, np.float64)
    lo, hi = np.asarray(box[:3], float), np.asarray(box[3:], float)
    N, D, T = [], [], []
    for k in range(3):
        e = np.zeros(3); e[k] = -1.0
        N.append(e); D.append(-lo[k]); T.append(-1 - 2 * k)
        e = np.zeros(3); e[k] = 1.0
        N.append(e); D.append(hi[k]); T.append(-2 - 2 * k)
    for j in range(len(p)):
        if j == i:
            continue
        N.append(2.0 * (p[j] - p[i]))
        D.append(p[j] @ p[j] - p[i] @ p[i] + w[i] - w[j])
        T.append(j)
    return np.array(N), np.array(D), np.array(T)


def _poly_area_3d(pts, normal):
    """Area of the convex hull of coplanar points (angle sort around the centroid)."""
    if len(pts) < 3:
        return 0.0
    c = pts.mean(axis=0)
    nrm = normal / np.linalg.norm(normal)
    a = np.cross(nrm, [1.0, 0, 0])
    if np.linalg.norm(a) < 0.5:
        a = np.cross(nrm, [0, 1.0, 0])
    a /= np.linalg.norm(a)
    b = np.cross(nrm, a)
    q = pts - c
    ang = np.arctan2(q @ b, q @ a)
    o = np.argsort(ang)
    P = pts[o]
    A = np.zeros(3)
    for k in range(len(P)):
        A += np.cross(P[k], P[(k + 1) % len(P)])
    return 0.5 * abs(A @ nrm)


def vertex_enumeration_cell(points, weights, box, i, rel_tol=1e-9):
    """Cell i by exhaustive triple-plane enumeration.  Returns (neighbours sorted, areas dict,
    volume).  Only for tiny inputs (O(P^3) solves)."""
    from scipy.spatial import ConvexHull
    N, D, T = planes_for_cell(points, weights, box, i)
    scale = float(np.max(np.abs(np.asarray(box, float)))) + 1.0
    tol = rel_tol * scale * scale
    verts = []
    idx = np.array(list(itertools.combinations(range(len(N)), 3)))
    A = N[idx]                       # [m, 3, 3]
    b = D[idx]                       # [m, 3]
    det = np.linalg.det(A)
    ok = np.abs(det) > 1e-12 * np.max(np.abs(A), axis=(1, 2)) ** 3
    X = np.linalg.solve(A[ok], b[ok][..., None])[..., 0]
    feas = np.all(X @ N.T - D[None, :] <= tol * (1.0 + np.linalg.norm(N, axis=1))[None, :], axis=1)
    V = X[feas]
    if len(V) < 4:
        return [], {}, 0.0
    V = np.unique(np.round(V, 12), axis=0)
    try:
        vol = ConvexHull(V).volume
    except Exception:
        return [], {}, 0.0
    areas = {}
    for f in range(len(N)):
        s = V @ N[f] - D[f]
        on = np.abs(s) <= tol * (1.0 + np.linalg.norm(N[f]))
        if on.sum() >= 3:
            a = _poly_area_3d(V[on], N[f])
            if a > 0:
                areas[int(T[f])] = areas.get(int(T[f]), 0.0) + a
    nb = sorted(t for t, a in areas.items() if t >= 0)
    return nb, areas, vol


def _interval_1d(X, f, a, lo, hi):
    """Exact 1-D power cell of site a: {x in [lo,hi] : (x-X_a)^2 - f_a <= (x-X_b)^2 - f_b  ∀b}."""
    L, H = Fraction(lo), Fraction(hi)
    for b in range(len(X)):
        if b == a:
            continue
        dX = Fraction(X[b]) - Fraction(X[a])
        rhs = Fraction(X[b]) ** 2 - Fraction(X[a]) ** 2 + Fraction(f[a]) - Fraction(f[b])
        if dX == 0:
            if rhs < 0:
                return None
            continue
        t = rhs / (2 * dX)          # 2 x dX <= rhs
        if dX > 0:
            H = min(H, t)
        else:
            L = max(L, t)
    if H <= L:
        return None
    return (L, H)


def separable_grid_cells(X, Y, Z, f, g, h, box):
    """Exact cells of the separable-weight grid.  Site (a,b,c) has index (a*len(Y) + b)*len(Z) + c,
    position (X_a, Y_b, Z_c), weight f_a + g_b + h_c.  Returns (points, weights, vol[list Fraction],
    nbrs[list of dict j -> area Fraction])."""
    Ix = [_interval_1d(X, f, a, box[0], box[3]) for a in range(len(X))]
    Iy = [_interval_1d(Y, g, b, box[1], box[4]) for b in range(len(Y))]
    Iz = [_interval_1d(Z, h, c, box[2], box[5]) for c in range(len(Z))]
    ln = lambda I: (I[1] - I[0]) if I is not None else Fraction(0)
    nY, nZ = len(Y), len(Z)
    idx = lambda a, b, c: (a * nY + b) * nZ + c
    pts, wts, vols, nbrs = [], [], [], []
    for a in range(len(X)):
        for b in range(nY):
            for c in range(nZ):
                pts.append((X[a], Y[b], Z[c]))
                wts.append(f[a] + g[b] + h[c])
                v = ln(Ix[a]) * ln(Iy[b]) * ln(Iz[c])
                vols.append(v)
                nb = {}
                if v > 0:
                    for a2 in range(len(X)):
                        if a2 != a and Ix[a2] is not None and (Ix[a2][0] == Ix[a][1] or Ix[a2][1] == Ix[a][0]):
                            nb[idx(a2, b, c)] = ln(Iy[b]) * ln(Iz[c])
                    for b2 in range(nY):
                        if b2 != b and Iy[b2] is not None and (Iy[b2][0] == Iy[b][1] or Iy[b2][1] == Iy[b][0]):
                            nb[idx(a, b2, c)] = ln(Ix[a]) * ln(Iz[c])
                    for c2 in range(nZ):
                        if c2 != c and Iz[c2] is not None and (Iz[c2][0] == Iz[c][1] or Iz[c2][1] == Iz[c][0]):
                            nb[idx(a, b, c2)] = ln(Ix[a]) * ln(Iy[b])
                nbrs.append(nb)
    return (np.array(pts, np.float32), np.array(wts, np.float32), vols, nbrs)


def lifted_adjacency(points, weights):
    """Regular-triangulation edges from the lower hull of the lifted points; returns
    (set of (i,j) with i<j, boolean mask of sites that are lower-hull vertices)."""
    from scipy.spatial import ConvexHull
    p = np.asarray(points, np.float64)
    w = np.zeros(len(p)) if weights is None else np.asarray(weights, np.float64)
    c = p.mean(axis=0)
    q = p - c
    lifted = np.concatenate([q, (np.sum(q * q, axis=1) - w)[:, None]], axis=1)
    hull = ConvexHull(lifted)
    lower = hull.equations[:, 3] < 0
    E = set()
    onhull = np.zeros(len(p), bool)
    for s in hull.simplices[lower]:
        onhull[s] = True
        for a, b in itertools.combinations(sorted(s.tolist()), 2):
            E.add((a, b))
    return E, onhull


def power_argmin(points, weights, x):
    p = np.asarray(points, np.float64)
    w = np.zeros(len(p)) if weights is None else np.asarray(weights, np.float64)
    d = np.sum((x[:, None, :] - p[None, :, :]) ** 2, axis=2) - w[None, :]
    o = np.argsort(d, axis=1)[:, :2]
    return o[:, 0], d[np.arange(len(x)), o[:, 0]], d[np.arange(len(x)), o[:, 1]]
