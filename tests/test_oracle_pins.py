"""Pins for the CPU oracle (-m "not gpu").

The oracle (oracle/pd_oracle.c) is checked against things the paper and mathematics fix, never
against itself: closed forms (tests/golden/closed_forms.json, each entry cited), an independent
brute-force vertex enumeration, exact rational separable-weight power grids, lattice cells,
partition of the box, symmetry of the adjacency, the empty-power-sphere (regular triangulation)
property, Monte-Carlo ownership, the Qhull lifting reduction and the
Poisson-Voronoi mean face count.  A dropped term, a flipped sign, a wrong index or a transposed
operand in the oracle fails at least one of these.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import pdgen
import brute

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))


def _run(points, weights, box, **kw):
    return oracle.cells(np.asarray(points, np.float32), None if weights is None else np.asarray(weights, np.float32),
                        box, **kw)


# ----------------------------------------------------------------------------- closed forms

@pytest.mark.parametrize("case", GOLD["two_site"], ids=lambda c: c["cite"][:40])
def test_two_site_plane_position(case):
    """Cell i = box ∩ {x_axis <= plane_at}; cell j = box ∩ {x_axis >= plane_at}."""
    box = case["box"]
    pts = [case["p_i"], case["p_j"]]
    r = _run(pts, [case["w_i"], case["w_j"]], box)
    ax, t = case["plane_axis"], case["plane_at"]
    lo, hi = box[ax], box[ax + 3]
    cross = np.prod([box[k + 3] - box[k] for k in range(3) if k != ax])
    vi = cross * (min(max(t, lo), hi) - lo)
    vj = cross * (hi - min(max(t, lo), hi))
    assert r.vol[0] == pytest.approx(vi, rel=1e-12, abs=1e-12)
    assert r.vol[1] == pytest.approx(vj, rel=1e-12, abs=1e-12)
    if lo < t < hi:
        for c in (0, 1):
            nb, ar = r.row(c)
            assert list(nb) == [1 - c]
            assert ar[0] == pytest.approx(cross, rel=1e-12)
    else:
        empty = 0 if t <= lo else 1
        assert r.flags[empty] & oracle.EMPTY
        assert len(r.row(empty)[0]) == 0 and len(r.row(1 - empty)[0]) == 0


def test_cube_halved():
    c = GOLD["cube_halved"]
    r = _run(c["points"], None, c["box"])
    for t in (0, 1):
        assert r.vol[t] == pytest.approx(c["vol"], rel=1e-14)
        nb, ar = r.row(t)
        assert list(nb) == [1 - t] and ar[0] == pytest.approx(c["shared_area"], rel=1e-14)
        assert r.flags[t] & oracle.BOUNDARY
        # surface = shared face + 5 walls: 1 + 2*(0.5) + 2*(0.5) + 1
        assert r.surf[t] == pytest.approx(4.0, rel=1e-14)


def _lattice(kind, m, a):
    g = np.arange(-m, m + 1, dtype=np.float64)
    base = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    if kind == "sc":
        pts = base
    elif kind == "bcc":
        pts = np.concatenate([base, base + 0.5])
    else:
        pts = np.concatenate([base, base + [0.5, 0.5, 0], base + [0.5, 0, 0.5], base + [0, 0.5, 0.5]])
    return (pts * a).astype(np.float32)


@pytest.mark.parametrize("kind", ["sc", "bcc", "fcc"])
def test_lattice_center_cells(kind):
    """Closed-form Voronoi cells of the cubic lattices; the zero-area edge/vertex contacts of the
    cospherical configurations must NOT become neighbours."""
    a = 0.5  # dyadic: every site is exact in float32
    pts = _lattice(kind, 3, a)
    box = [-3.6 * a] * 3 + [3.6 * a] * 3
    ctr = int(np.argmin(np.sum(pts.astype(np.float64) ** 2, axis=1)))
    r = _run(pts, None, box, ids=[ctr])
    spec = GOLD["lattices"][kind]
    assert r.vol[0] == pytest.approx(spec["vol_over_a3"] * a ** 3, rel=1e-12)
    nb, ar = r.row(0)
    expect = sorted([area for cnt, area in spec["faces"] for _ in range(cnt)])
    assert len(nb) == len(expect)
    assert np.allclose(np.sort(ar) / a ** 2, expect, rtol=1e-12)


def test_separable_weight_grid_exact():
    """Power cells of a separable-weight grid are products of exact 1-D power cells (derived in
    SURVEY.md §8(c)); includes EMPTY cells (a heavy-negative x-layer) and zero-area diagonal
    contacts."""
    X, Y, Z = [0, 2, 3, 7, 8, 11], [1, 4, 5, 9], [0, 3, 4, 6, 10]
    f, g, h = [0, 1, -3, 2, 0, 1], [0, -1, 2, 0], [1, 0, 0, -2, 0]
    box = (-1, -1, -2, 12, 11, 11)
    pts, wts, vols, nbrs = brute.separable_grid_cells(X, Y, Z, f, g, h, box)
    r = _run(pts, wts, box)
    assert any(v == 0 for v in vols), "grid should contain EMPTY cells"
    for t in range(len(pts)):
        assert r.vol[t] == pytest.approx(float(vols[t]), rel=1e-12, abs=1e-12)
        assert bool(r.flags[t] & oracle.EMPTY) == (vols[t] == 0)
        nb, ar = r.row(t)
        exp = nbrs[t]
        assert list(nb) == sorted(exp.keys()), t
        for j, a in zip(nb, ar):
            assert a == pytest.approx(float(exp[int(j)]), rel=1e-12)
    assert Fraction(sum(vols)) == Fraction(13 * 12 * 13)


# ----------------------------------------------------------------------------- brute force

@pytest.mark.parametrize("seed,weighted", [(11, False), (12, True), (13, True)])
def test_vs_vertex_enumeration(seed, weighted):
    n = 18
    pts = pdgen.white_noise(n, seed, 0.0, 1.0)
    w = (0.02 * pdgen.normal(seed, 7, n)).astype(np.float32) if weighted else None
    box = (0.0, 0.0, 0.0, 1.0, 1.0, 1.0)
    r = _run(pts, w, box)
    for i in range(n):
        nb, areas, vol = brute.vertex_enumeration_cell(pts, w, box, i)
        assert r.vol[i] == pytest.approx(vol, rel=1e-7, abs=1e-12)
        onb, oar = r.row(i)
        assert list(onb) == nb, (i, list(onb), nb)
        for j, a in zip(onb, oar):
            assert a == pytest.approx(areas[int(j)], rel=1e-6)
        walls = sum(a for t, a in areas.items() if t < 0)
        assert r.surf[i] == pytest.approx(sum(oar) + walls, rel=1e-7)


def test_clip_order_invariance():
    """K_i does not depend on the clipping order."""
    wl = pdgen.make("C3", n=3000)
    a = _run(wl.points, wl.weights, wl.box, order_k=0)
    b = _run(wl.points, wl.weights, wl.box, order_k=64)
    assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.nbr, b.nbr)
    assert np.allclose(a.area, b.area, rtol=1e-9, atol=1e-15)
    assert np.allclose(a.vol, b.vol, rtol=1e-9, atol=1e-18)


# ----------------------------------------------------------------------------- invariants

def _sym_check(r, rel=1e-10):
    # rounding of a face's area is relative to its cell's size, not to the face: absolute term
    pairs, surf = {}, {}
    for t in range(len(r.ids)):
        nb, ar = r.row(t)
        surf[int(r.ids[t])] = r.surf[t]
        for j, a in zip(nb, ar):
            pairs[(int(r.ids[t]), int(j))] = a
    bad = 0
    for (i, j), a in pairs.items():
        b = pairs.get((j, i))
        if b is None or abs(a - b) > rel * max(a, b) + 1e-13 * max(surf[i], surf[j]):
            bad += 1
    return bad, len(pairs)


@pytest.mark.parametrize("cfg,n", [("C1", 1000), ("C2", 4000), ("C3", 4000), ("C4", 4000), ("C5", 4000)])
def test_partition_and_symmetry(cfg, n):
    """Cells tile the box (Σ vol = vol(B)) and adjacency is symmetric with a_ij = a_ji."""
    wl = pdgen.make(cfg, n=n)
    r = _run(wl.points, wl.weights, wl.box)
    bx = np.asarray(wl.box, float)
    vb = np.prod(bx[3:] - bx[:3])
    assert r.vol.sum() == pytest.approx(vb, rel=1e-11)
    bad, tot = _sym_check(r)
    assert bad == 0 and tot > n
    assert not np.any(r.flags & oracle.DEGRADED)
    assert np.all((r.vol == 0) == ((r.flags & oracle.EMPTY) > 0))


def test_empty_power_sphere_and_face_bisectors():
    """Every vertex v of K_i satisfies π_i(v) <= π_k(v) for ALL k (brute force), and π_i(v) = π_j(v)
    for every bisector face j through v (regular-triangulation / empty power sphere property)."""
    wl = pdgen.make("C5", n=600)
    p = wl.points.astype(np.float64)
    w = wl.weights.astype(np.float64)
    scale = 20.0 ** 2
    rng = np.random.default_rng(0)
    for i in rng.choice(wl.n, 40, replace=False):
        geo = oracle.cell_geometry(wl.points, wl.weights, wl.box, int(i))
        if not geo.loops:
            continue
        for tag, loop in zip(geo.tags, geo.loops):
            pw = np.sum((loop[:, None, :] - p[None]) ** 2, axis=2) - w[None]
            assert np.all(pw >= pw[:, [i]] - 1e-9 * scale)
            if tag >= 0:
                assert np.allclose(pw[:, i], pw[:, tag], atol=1e-9 * scale)


def test_monte_carlo_ownership():
    """x ∈ B belongs to the oracle cell of argmin_k π_k(x), and MC volumes agree."""
    wl = pdgen.make("C3", n=300)
    p64 = wl.points.astype(np.float64)
    rng = np.random.default_rng(5)
    x = rng.uniform(-10, 10, size=(20000, 3))
    own, d0, d1 = brute.power_argmin(wl.points, wl.weights, x)
    keep = (d1 - d0) > 1e-9
    r = _run(wl.points, wl.weights, wl.box)
    planes = {}
    for i in np.unique(own[keep])[:60]:
        geo = oracle.cell_geometry(wl.points, wl.weights, wl.box, int(i))
        planes[int(i)] = geo.planes
    for xi, oi in zip(x[keep], own[keep]):
        if int(oi) not in planes:
            continue
        pl = planes[int(oi)]
        y = xi - p64[oi]
        assert np.all(pl[:, :3] @ y - pl[:, 3] <= 1e-9 * (1 + np.abs(pl[:, 3])))
    frac = np.bincount(own, minlength=wl.n) / len(x)
    ref = r.vol / 8000.0
    sig = np.sqrt(np.maximum(ref * (1 - ref), 1e-12) / len(x))
    assert np.all(np.abs(frac - ref) <= 5 * sig + 1e-4)


@pytest.mark.parametrize("weighted", [False, True])
def test_lifting_qhull_crosscheck(weighted):
    """Library cross-check: non-BOUNDARY cells' neighbours = regular-triangulation adjacency from
    the 4-D lower hull of lifted points; non-hull sites are EMPTY."""
    n = 3000
    pts = pdgen.white_noise(n, 77)
    if weighted:
        d = pdgen.median_nn_distance(pts)
        w = pdgen.weights_student_t(n, d, 77)
    else:
        w = None
    E, onhull = brute.lifted_adjacency(pts, w)
    r = _run(pts, w, pdgen.OMEGA_BOX)
    adj = {i: set() for i in range(n)}
    for a, b in E:
        adj[a].add(b); adj[b].add(a)
    checked = 0
    for i in range(n):
        if r.flags[i] & oracle.BOUNDARY:
            continue
        if not onhull[i]:
            assert r.flags[i] & oracle.EMPTY
            continue
        if r.flags[i] & oracle.EMPTY:
            continue  # non-empty unbounded cell lying wholly outside the box (heavy weights nearby)
        assert set(int(j) for j in r.row(i)[0]) == adj[i], i
        checked += 1
    assert checked > n // 3
    if weighted:
        assert np.count_nonzero(~onhull) > 0


def test_voronoi_equivalence_and_weight_shift():
    """All-equal weights ≡ Voronoi; w + c (dyadic c) ≡ w."""
    wl = pdgen.make("C2", n=2000)
    a = _run(wl.points, None, wl.box)
    b = _run(wl.points, np.full(wl.n, 0.25, np.float32), wl.box)
    assert np.array_equal(a.nbr, b.nbr) and np.allclose(a.vol, b.vol, rtol=1e-12)
    w = (0.01 * pdgen.normal(3, 3, wl.n)).astype(np.float32)
    c = _run(wl.points, w, wl.box)
    d = _run(wl.points, (w.astype(np.float64) + 2.0).astype(np.float32), wl.box)
    same = np.all((w.astype(np.float64) + 2.0).astype(np.float32).astype(np.float64) - 2.0 == w)
    if same:
        assert np.array_equal(c.nbr, d.nbr)


def test_permutation_equivariance():
    wl = pdgen.make("C4", n=2000)
    perm = np.random.default_rng(1).permutation(wl.n)
    a = _run(wl.points, wl.weights, wl.box)
    b = _run(wl.points[perm], wl.weights[perm], wl.box)
    inv = np.argsort(perm)
    for t in range(wl.n):
        tb = inv[t]
        na = list(a.row(t)[0])
        nb = sorted(int(perm[j]) for j in b.row(tb)[0])
        assert na == nb
        assert a.vol[t] == pytest.approx(b.vol[tb], rel=1e-10, abs=1e-15)


def test_duplicate_rule():
    """Bit-identical sites: the heavier owns, ties to the lower id."""
    pts = np.array([[0.5, 0.5, 0.5], [0.25, 0.5, 0.5], [0.5, 0.5, 0.5], [0.75, 0.5, 0.5]], np.float32)
    box = (0, 0, 0, 1, 1, 1)
    r = _run(pts, None, box)
    assert r.flags[2] & oracle.DUPLICATE and r.flags[2] & oracle.EMPTY and not (r.flags[0] & oracle.EMPTY)
    r = _run(pts, [0.0, 0.0, 0.001, 0.0], box)
    assert r.flags[0] & oracle.DUPLICATE and not (r.flags[2] & oracle.EMPTY)
    assert r.vol.sum() == pytest.approx(1.0, rel=1e-14)


def test_poisson_voronoi_mean_faces():
    """Interior cells of uniform data: mean face count ≈ 2 + 48π²/35 (closed form)."""
    pts = pdgen.white_noise(20000, 31, 0.0, 1.0)
    r = _run(pts, None, (0, 0, 0, 1, 1, 1))
    p = pts.astype(np.float64)
    inner = np.minimum(p, 1 - p).min(axis=1) > 3 * (1 / 20000) ** (1 / 3)  # away from wall bias
    deg = np.diff(r.offsets)[inner]
    assert inner.sum() > 8000
    assert abs(deg.mean() - GOLD["poisson_voronoi"]["mean_faces"]) < 0.15


# ----------------------------------------------------------------------------- dual tetrahedra

def _center(p, w):
    """Power centre of 4 sites: |c-p_k|^2 - w_k equal for all k (circumcentre when w = 0)."""
    A = 2.0 * (p[1:] - p[0])
    b = np.sum(p[1:] ** 2, axis=1) - np.sum(p[0] ** 2) - (w[1:] - w[0])
    return np.linalg.solve(A, b)


@pytest.mark.parametrize("weighted", [False, True])
def test_dual_tets_vs_qhull(weighted):
    """oracle.dual_tets against the library triangulation: scipy Delaunay (unweighted) or the lower
    hull of the lifted points (weighted, the reduction of PAPER.md:122-123).  Every oracle tet is a
    triangulation tet, and every triangulation tet whose (power) centre lies inside the box, away
    from its walls, is an oracle tet."""
    from scipy.spatial import ConvexHull, Delaunay
    n = 400
    pts = pdgen.white_noise(n, 31, 0.0, 1.0)
    box = (0.0, 0.0, 0.0, 1.0, 1.0, 1.0)
    p64 = pts.astype(np.float64)
    if weighted:
        w = pdgen.weights_paper(n, pdgen.median_nn_distance(pts), 31, ratio=10.0)
        w64 = w.astype(np.float64)
        c = p64.mean(axis=0)
        q = p64 - c
        hull = ConvexHull(np.concatenate([q, (np.sum(q * q, axis=1) - w64)[:, None]], axis=1))
        simp = hull.simplices[hull.equations[:, 3] < 0]
    else:
        w, w64 = None, np.zeros(n)
        simp = Delaunay(p64).simplices
    ref = {tuple(sorted(int(x) for x in s)) for s in simp}
    got, ndeg = oracle.dual_tets(pts, w, box)
    assert ndeg == 0 and len(got) > n
    gset = {tuple(int(x) for x in t) for t in got}
    assert gset <= ref
    inside = 0
    for s in ref:
        ctr = _center(p64[list(s)], w64[list(s)])
        if np.all(ctr > 1e-6) and np.all(ctr < 1 - 1e-6):
            inside += 1
            assert s in gset, s
    assert inside > n


def test_dual_tets_cube_corner_and_two_sites():
    """Closed forms: 2 sites -> no tet (every vertex touches a wall); 5 sites = 4 around a centre
    inside a big box -> the centre's 4 tets {0, a, b, c} of the convex position."""
    box = (-10.0, -10.0, -10.0, 10.0, 10.0, 10.0)
    t, _ = oracle.dual_tets(np.array([[0, 0, 0], [1, 0, 0]], np.float32), None, box)
    assert len(t) == 0
    P = np.array([[0, 0, 0], [1, 0.1, -0.2], [-0.3, 1, 0.15], [0.2, -0.4, 1.1], [-0.9, -0.8, -0.7]], np.float32)
    t, _ = oracle.dual_tets(P, None, box)
    # the centre site 0 lies inside the tetrahedron of the other four: Delaunay = 4 tets around it
    assert sorted(map(tuple, t.tolist())) == [(0, 1, 2, 3), (0, 1, 2, 4), (0, 1, 3, 4), (0, 2, 3, 4)]


# ----------------------------------------------------------------------------- CPU reference (bench baseline)

class _Rows:
    pass


@pytest.mark.parametrize("cfg,n", [("C1", None), ("C2", 4000), ("C3", 4000), ("C4", 4000), ("C5", 4000)])
def test_cpu_reference_same_definition(cfg, n):
    """The k-d tree + weighted radius-of-security CPU reference reaches the oracle's cells:
    it only skips sites whose bisector provably misses the cell."""
    from compare import compare
    wl = pdgen.make(cfg, n=n)
    k = oracle.KdReference(wl.points, wl.weights, wl.box).cells()
    o = oracle.cells(wl.points, wl.weights, wl.box)
    d = _Rows()
    d.offsets, d.neighbors, d.areas, d.surface, d.flags = k.offsets, k.nbr, k.area, k.surf, k.flags
    d.volumes = k.vol.astype(np.float32)
    rep = compare(d, o)
    assert rep.ok, rep.summary()
    assert rep.cells == wl.n


def test_cpu_reference_duplicates_and_empty():
    """Coincident sites (Q5) and weight-emptied cells: the walk must still meet the owner / the dominating site."""
    pts = np.array([[0.5, 0.5, 0.5], [0.5, 0.5, 0.5], [0.2, 0.3, 0.4], [0.8, 0.7, 0.6], [0.25, 0.3, 0.4]], np.float32)
    w = np.array([0.0, 0.01, 0.0, 0.0, 0.5], np.float32)
    box = (0, 0, 0, 1, 1, 1)
    k = oracle.KdReference(pts, w, box).cells()
    o = oracle.cells(pts, w, box)
    assert np.array_equal(k.flags, o.flags)
    assert np.allclose(k.vol, o.vol, rtol=1e-9, atol=1e-15)
    assert k.flags[0] & oracle.DUPLICATE and k.flags[2] & oracle.EMPTY
