"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same seeded inputs.

Full diagrams at oracle-friendly sizes that span many warps/leaves and a ragged tail; sampled cells
(random + degree tail + BOUNDARY + EMPTY + OVERFLOW strata) at BASELINE.json's full sizes in the
launch configuration bench.py times; plus properties that hold at any size (symmetry, partition of
the box), determinism, ablation neutrality, sharded reassembly and the error contract.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import pdgen  # noqa: E402
import paper_2605_06408_b200 as pd  # noqa: E402
from compare import compare, sample_cells  # noqa: E402

NT = os.cpu_count() or 8


def _gpu(wl, **kw):
    p = torch.from_numpy(wl.points).cuda()
    w = None if wl.weights is None else torch.from_numpy(wl.weights).cuda()
    d = pd.build_diagram(p, w, wl.box, **kw)
    torch.cuda.synchronize()
    return d.to_numpy()


def _assert_parity(wl, ids=None, **kw):
    g = _gpu(wl, **kw)
    o = oracle.cells(wl.points, wl.weights, wl.box, ids=ids, threads=NT)
    rep = compare(g, o)
    print(wl.name, wl.n, rep.summary())
    assert rep.ok, rep.summary()
    return g, o, rep


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    pd.load_library()


# ----------------------------------------------------------------- full diagrams, small sizes

def test_c1_full():
    _assert_parity(pdgen.make("C1"))


@pytest.mark.parametrize("cfg,n", [("C2", 20011), ("C3", 20011), ("C4", 20011), ("C5", 20011)])
def test_configs_full_small(cfg, n):
    _assert_parity(pdgen.make(cfg, n=n))


def _paper_workload(kind, n, seed, weighted):
    """The paper's synthetic laws: white noise, K Gaussian clusters (sigma=0.1),
    linear density gradient; optionally w ~ N(0, (d_nn^2/3)^2)."""
    if kind == "white":
        p = pdgen.white_noise(n, seed)
    elif kind.startswith("clustered"):
        p = pdgen.clustered(n, seed, k=int(kind[9:]), sigma=0.1)
    else:
        p = pdgen.density_gradient(n, seed)
    w = pdgen.weights_paper(n, pdgen.median_nn_distance(p), seed) if weighted else None
    return pdgen.Workload(f"{kind}{'-w' if weighted else ''}", p, w, pdgen.OMEGA_BOX, kind)


@pytest.mark.parametrize("kind", ["white", "clustered5", "clustered10", "gradient"])
@pytest.mark.parametrize("weighted", [False, True])
def test_paper_workloads(kind, weighted):
    _assert_parity(_paper_workload(kind, 12007, 21, weighted))


@pytest.mark.parametrize("ratio", [0.0, 1.0, 10.0, 100.0])
def test_weight_magnitude_sweep(ratio):
    """Weight-magnitude sweep (PAPER.md:563-581 analogue): larger weights empty
    more cells; the diagram stays exact."""
    p = pdgen.white_noise(8009, 5)
    d = pdgen.median_nn_distance(p)
    w = pdgen.weights_paper(8009, d, 5, ratio=ratio)
    g, o, rep = _assert_parity(pdgen.Workload(f"sweep{ratio}", p, w, pdgen.OMEGA_BOX, ""))
    if ratio >= 10:
        assert np.mean(g.flags & pd.CELL_EMPTY) > 0.05


@pytest.mark.parametrize("leaf", [1, 7, 16, 32])
def test_leaf_sizes_identical(leaf):
    wl = pdgen.make("C5", n=5003)
    ref = _gpu(wl)
    g = _gpu(wl, leaf_size=leaf)
    assert np.array_equal(ref.offsets, g.offsets) and np.array_equal(ref.neighbors, g.neighbors)
    assert np.allclose(ref.volumes, g.volumes, rtol=1e-6, atol=0)


ABLATIONS = [pd.ISOTROPIC, pd.DFS, pd.PAPER_BOUND, pd.NO_EXACT, pd.EXACT_NODES, pd.WARM_START | pd.DFS,
             pd.ISOTROPIC | pd.DFS, pd.WARM_ADAPTIVE]


@pytest.mark.parametrize("flag", ABLATIONS)
def test_ablations_neutral(flag):
    """Culling / traversal variants change the work, not the diagram."""
    wl = pdgen.make("C3", n=8009)
    ref = _gpu(wl)
    g = _gpu(wl, flags=flag)
    assert np.array_equal(ref.offsets, g.offsets) and np.array_equal(ref.neighbors, g.neighbors)
    assert np.allclose(ref.volumes, g.volumes, rtol=1e-6)


@pytest.mark.parametrize("cfg,n", [("C3", 8009), ("C5", 6007)])
@pytest.mark.parametrize("flag", ABLATIONS)
def test_ablations_oracle(cfg, n, flag):
    """Every ablation / traversal mode of the paper (isotropic culling P:211, DFS P:299, the paper's bounds
    only P:229-233, no / always exact node tests, KNN warm start P:544-545 with DFS) against the ORACLE on
    small sets ("oracle-verified"), not only against the default GPU output."""
    _assert_parity(pdgen.make(cfg, n=n), flags=flag)


def _tight_box(points):
    """The paper's initial cell when no box is given: the FP32 AABB of the points, an
    axis of zero extent widened by one FP32 ulp on each side (reading R1)."""
    p = np.asarray(points, np.float32)
    lo, hi = p.min(axis=0), p.max(axis=0)
    for k in range(3):
        if not lo[k] < hi[k]:
            lo[k] = np.nextafter(lo[k], np.float32(-np.inf))
            hi[k] = np.nextafter(hi[k], np.float32(np.inf))
    return tuple(float(v) for v in lo) + tuple(float(v) for v in hi)


@pytest.mark.parametrize("case", ["C3", "C4", "flat", "two-flat"])
def test_box_null_parity(case):
    """pd_build(box=NULL) (a2): the box is the tight AABB of the points; compared with the
    oracle run on that box computed on the host, incl. the flat-axis widening."""
    if case in ("C3", "C4"):
        wl = pdgen.make(case, n=12007)
        pts, w = wl.points, wl.weights
    else:
        pts = pdgen.white_noise(700, 9, 0.0, 1.0)
        pts[:, 2] = 0.5  # flat in z
        if case == "two-flat":
            pts[:, 1] = 0.25  # a line: flat in y and z
            pts = pts[:200]
        w = None
    g = pd.build_diagram(pts, w, None, out_host=True)
    o = oracle.cells(pts, w, _tight_box(pts), threads=NT)
    rep = compare(g, o)
    print(case, rep.summary())
    assert rep.ok, rep.summary()
    bx = np.asarray(_tight_box(pts), np.float64)
    assert g.volumes.astype(np.float64).sum() == pytest.approx(np.prod(bx[3:] - bx[:3]), rel=1e-5)


@pytest.mark.parametrize("cfg,n", [("C1", None), ("C3", 20011), ("C5", 20011)])
def test_warm_start_parity(cfg, n):
    """KNN warm start against the oracle, incl. weight-emptied and heavy cells, and
    with a leaf of one site (KNN over single-site leaves)."""
    _assert_parity(pdgen.make(cfg, n=n), flags=pd.WARM_START)
    _assert_parity(pdgen.make(cfg, n=n), flags=pd.WARM_START, leaf_size=1)
    _assert_parity(pdgen.make(cfg, n=n), flags=pd.WARM_ADAPTIVE)


@pytest.mark.parametrize("cfg,n", [("C3", 20011), ("C5", 20011)])
def test_auto_warm_decision(cfg, n):
    """PD_AUTO_WARM: the sampled warm-start decision runs (warm_gain > 0 reported), the diagram matches the
    oracle and the default build's neighbour sets whichever way it decides."""
    wl = pdgen.make(cfg, n=n)
    ref = _gpu(wl)
    g, o, rep = _assert_parity(wl, flags=pd.AUTO_WARM)
    assert g.stats["warm_gain"] > 0 and g.stats["warm_start"] in (0, 1)
    assert np.array_equal(ref.offsets, g.offsets) and np.array_equal(ref.neighbors, g.neighbors)
    assert _gpu(wl).stats["warm_gain"] == 0  # default: no sampling


def test_warm_start_duplicates_and_lattice():
    """Warm start with coincident sites (excluded from the KNN; the leaf processing decides ownership)
    and with cospherical lattices (KNN planes met again in their leaves must not re-clip)."""
    pts = np.array([[0.5, 0.5, 0.5], [0.25, 0.5, 0.5], [0.5, 0.5, 0.5], [0.75, 0.5, 0.5], [0.5, 0.5, 0.5]], np.float32)
    box = (0, 0, 0, 1, 1, 1)
    a = pd.build_diagram(pts, None, box, out_host=True)
    b = pd.build_diagram(pts, None, box, out_host=True, flags=pd.WARM_START)
    for k in ("offsets", "neighbors", "flags"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    # weighted duplicates: the heavy coincident pair must stay EMPTY|DUPLICATE even when a power-nearest
    # heavy neighbour empties the light one first
    pts2 = np.array([[0.5, 0.5, 0.5], [0.5, 0.5, 0.5], [0.52, 0.5, 0.5], [0.2, 0.3, 0.4]], np.float32)
    w2 = np.array([0.0, 0.001, 0.5, 0.0], np.float32)
    a = pd.build_diagram(pts2, w2, box, out_host=True)
    b = pd.build_diagram(pts2, w2, box, out_host=True, flags=pd.WARM_START)
    assert np.array_equal(a.flags, b.flags) and a.flags[0] & pd.CELL_DUPLICATE
    gr = np.arange(-3, 4, dtype=np.float64)
    P = (np.stack(np.meshgrid(gr, gr, gr, indexing="ij"), -1).reshape(-1, 3) * 0.5).astype(np.float32)
    a = pd.build_diagram(P, None, (-1.8,) * 3 + (1.8,) * 3, out_host=True)
    b = pd.build_diagram(P, None, (-1.8,) * 3 + (1.8,) * 3, out_host=True, flags=pd.WARM_START)
    assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.neighbors, b.neighbors)
    assert np.allclose(a.volumes, b.volumes, rtol=1e-6)


@pytest.mark.parametrize("cfg,n", [("C3", 6007), ("C5", 6007)])
@pytest.mark.parametrize("flags", [0, pd.WARM_START])
@pytest.mark.parametrize("start_tier", ["1", "2"])
def test_top_tier_cooperative(cfg, n, flags, start_tier, monkeypatch):
    """Every cell through a cooperative capacity tier (tier 2: state in shared memory, one cell per CTA
    of 4 warps; tier 3: state in global memory, one cell per CTA of 16 warps) with every O(V) pass
    CTA-cooperative (classification, batched cut tests, exact node tests, AABB, queue re-validation,
    twins, face areas): parity with the oracle and the same neighbour sets as the default tiers."""
    wl = pdgen.make(cfg, n=n)
    ref = _gpu(wl, flags=flags)
    monkeypatch.setenv("PD_START_TIER", start_tier)
    monkeypatch.setenv("PD_COOP_MIN_V", "0")
    g, o, rep = _assert_parity(wl, flags=flags | pd.STATS | pd.TETS)
    assert np.array_equal(ref.offsets, g.offsets) and np.array_equal(ref.neighbors, g.neighbors)
    rt = _gpu(wl, flags=flags | pd.TETS).tets
    assert {tuple(t) for t in np.asarray(g.tets).tolist()} == {tuple(t) for t in np.asarray(rt).tolist()}
    assert np.allclose(ref.volumes, g.volumes, rtol=1e-6)


@pytest.mark.parametrize("cfg,n", [("C3", 8009), ("C4", 8009)])
def test_record_arena_full(cfg, n, monkeypatch):
    """Tier 1 keeps no FP64 vertices and always defers its finalize (a per-cell topology record that
    finalize_kernel rebuilds); a finished cell whose record does not fit is built again by tier 2.  With a
    tiny record arena (test knob PD_REC_CAP) most cells take that path: oracle parity, and the same
    diagram as the default run."""
    wl = pdgen.make(cfg, n=n)
    ref = _gpu(wl)
    monkeypatch.setenv("PD_REC_CAP", "20000")
    g, o, rep = _assert_parity(wl, flags=pd.STATS)
    assert g.stats["tier_cells"][1] > n // 2  # most cells really went to tier 2
    assert np.array_equal(ref.offsets, g.offsets) and np.array_equal(ref.neighbors, g.neighbors)
    assert np.allclose(ref.volumes, g.volumes, rtol=1e-6)


@pytest.mark.parametrize("cfg,n", [("C1", None), ("C2", 4001), ("C3", 4001), ("C5", 4001)])
def test_dual_tets_parity(cfg, n):
    """Dual tetrahedra (PD_TETS) equal the oracle's, as sets of sorted id
    quadruples; host output identical; each tet listed once, grouped by its lowest id."""
    wl = pdgen.make(cfg, n=n)
    g = _gpu(wl, flags=pd.TETS)
    ref, ndeg = oracle.dual_tets(wl.points, wl.weights, wl.box)
    got = np.asarray(g.tets, np.int64)
    print(cfg, "tets", len(got), "oracle", len(ref), "degenerate vertices", ndeg)
    assert np.all(got[:, 0] < got[:, 1]) and np.all(got[:, 1] < got[:, 2]) and np.all(got[:, 2] < got[:, 3])
    assert np.all(np.diff(got[:, 0]) >= 0)
    assert len({tuple(t) for t in got.tolist()}) == len(got)
    assert {tuple(t) for t in got.tolist()} == {tuple(t) for t in ref.tolist()}
    h = pd.build_diagram(wl.points, wl.weights, wl.box, out_host=True, flags=pd.TETS)
    assert np.array_equal(h.tets, g.tets)
    # the diagram itself is unchanged by the extra output
    ref_d = _gpu(wl)
    assert np.array_equal(ref_d.offsets, g.offsets) and np.array_equal(ref_d.neighbors, g.neighbors)


@pytest.mark.parametrize("case", ["C1", "lattice"])
def test_robustness_counters(case):
    """pd_stats faces_dropped / faces_near_degenerate / degraded_cells (always collected): generic input has
    no degraded cell; cospherical lattices (every vertex shared by > 3 cells) neither, and their zero-area
    contacts never become neighbours."""
    if case == "C1":
        wl = pdgen.make("C1")
        d = pd.build_diagram(wl.points, None, wl.box, out_host=True)
        o = oracle.cells(wl.points, None, wl.box, threads=NT)
        rows = np.repeat(np.arange(wl.n), np.diff(d.offsets))
        assert d.stats["faces_near_degenerate"] == int(np.sum(d.areas < 1e-9 * d.surface[rows]))
        assert d.stats["faces_near_degenerate"] == int(o.small.sum())
    else:
        gr = np.arange(-3, 4, dtype=np.float64)
        P = (np.stack(np.meshgrid(gr, gr, gr, indexing="ij"), -1).reshape(-1, 3) * 0.5).astype(np.float32)
        d = pd.build_diagram(P, None, (-1.8,) * 3 + (1.8,) * 3, out_host=True)
    print(case, {k: d.stats[k] for k in ("faces_dropped", "faces_near_degenerate", "degraded_cells")})
    assert d.stats["degraded_cells"] == 0 and not np.any(d.flags & pd.CELL_DEGRADED)


def test_determinism_bitwise():
    wl = pdgen.make("C4", n=30011)
    a, b = _gpu(wl), _gpu(wl)
    for k in ("offsets", "neighbors", "areas", "volumes", "surface", "flags"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


def test_trim_then_rebuild_identical():
    """pd_trim releases the cached workspace and the internal stream of the higher tiers; the next build
    re-creates them and returns the same diagram bit for bit (tiers 2-3 launch on that stream every build)."""
    wl = pdgen.make("C3", n=20011)
    a = _gpu(wl, flags=pd.STATS)
    pd.trim(0)
    b = _gpu(wl, flags=pd.STATS)
    for k in ("offsets", "neighbors", "areas", "volumes", "surface", "flags"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


def test_host_and_device_inputs_identical():
    wl = pdgen.make("C3", n=7001)
    a = _gpu(wl)
    b = pd.build_diagram(wl.points, wl.weights, wl.box, out_host=True)
    for k in ("offsets", "neighbors", "areas", "volumes", "flags"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


# ----------------------------------------------------------------- special / degenerate inputs

def test_lattice_and_separable_grid():
    import brute
    X, Y, Z = [0, 2, 3, 7, 8, 11], [1, 4, 5, 9], [0, 3, 4, 6, 10]
    f, g, h = [0, 1, -3, 2, 0, 1], [0, -1, 2, 0], [1, 0, 0, -2, 0]
    box = (-1, -1, -2, 12, 11, 11)
    pts, wts, vols, nbrs = brute.separable_grid_cells(X, Y, Z, f, g, h, box)
    d = pd.build_diagram(pts, wts, box, out_host=True)
    for t in range(len(pts)):
        assert d.volumes[t] == pytest.approx(float(vols[t]), rel=1e-6, abs=1e-6)
        nb, ar = d.row(t)
        assert list(nb) == sorted(nbrs[t].keys())
    # cubic lattices (cospherical: zero-area contacts must not become neighbours)
    for kind, vol, deg in (("sc", 1.0, 6), ("bcc", 0.5, 14), ("fcc", 0.25, 12)):
        gr = np.arange(-3, 4, dtype=np.float64)
        base = np.stack(np.meshgrid(gr, gr, gr, indexing="ij"), -1).reshape(-1, 3)
        if kind == "sc":
            P = base
        elif kind == "bcc":
            P = np.concatenate([base, base + 0.5])
        else:
            P = np.concatenate([base, base + [0.5, 0.5, 0], base + [0.5, 0, 0.5], base + [0, 0.5, 0.5]])
        P = (P * 0.5).astype(np.float32)
        dd = pd.build_diagram(P, None, (-1.8,) * 3 + (1.8,) * 3, out_host=True)
        c = int(np.argmin(np.sum(P.astype(np.float64) ** 2, axis=1)))
        nb, ar = dd.row(c)
        big = ar > 1e-9 * dd.surface[c]
        assert big.sum() == deg, kind
        assert dd.volumes[c] == pytest.approx(vol * 0.125, rel=1e-6)


def test_tiny_and_degenerate_inputs():
    box = (0, 0, 0, 1, 1, 1)
    d = pd.build_diagram(np.array([[0.5, 0.5, 0.5]], np.float32), None, box, out_host=True)
    assert d.nnz == 0 and d.volumes[0] == pytest.approx(1.0) and d.flags[0] & pd.CELL_BOUNDARY
    d = pd.build_diagram(np.array([[0.25, 0.5, 0.5], [0.75, 0.5, 0.5]], np.float32), None, box, out_host=True)
    assert list(d.neighbors) == [1, 0] and np.allclose(d.volumes, 0.5)
    # duplicates: the heavier owns, ties to the lower id
    pts = np.array([[0.5, 0.5, 0.5], [0.25, 0.5, 0.5], [0.5, 0.5, 0.5], [0.75, 0.5, 0.5]], np.float32)
    d = pd.build_diagram(pts, None, box, out_host=True)
    assert d.flags[2] & pd.CELL_DUPLICATE and d.flags[2] & pd.CELL_EMPTY and not d.flags[0] & pd.CELL_EMPTY
    # sites on the box boundary, points on a plane with the tight AABB (box=None)
    pts = pdgen.white_noise(500, 9, 0.0, 1.0)
    pts[:50, 0] = 0.0
    pts[50:100, 2] = 1.0
    _assert_parity(pdgen.Workload("edge", pts, None, box, ""))
    flat = pts.copy()
    flat[:, 2] = 0.5
    g = pd.build_diagram(flat, None, None, out_host=True)
    assert np.isfinite(g.volumes).all()
    # a weight so large that other cells become EMPTY
    pts = pdgen.white_noise(300, 5, 0.0, 1.0)
    w = np.zeros(300, np.float32)
    w[7] = 0.2
    _assert_parity(pdgen.Workload("heavy", pts, w, box, ""))


def test_error_contract():
    box = (0, 0, 0, 1, 1, 1)
    pts = pdgen.white_noise(100, 3, 0.0, 1.0)
    bad = pts.copy()
    bad[42, 1] = np.nan
    with pytest.raises(pd.PdError) as e:
        pd.build_diagram(bad, None, box)
    assert e.value.status == pd.PD_ENONFINITE and e.value.index == 42
    bad = pts.copy()
    bad[17, 0] = 1.5
    with pytest.raises(pd.PdError) as e:
        pd.build_diagram(bad, None, box)
    assert e.value.status == pd.PD_EOUTSIDE and e.value.index == 17
    with pytest.raises(pd.PdError) as e:
        pd.build_diagram(np.zeros((0, 3), np.float32), None, box)
    assert e.value.status == pd.PD_EEMPTY
    with pytest.raises(pd.PdError) as e:  # dual tets are not available from a sharded build
        pd.build_diagram(pts, None, box, flags=pd.TETS, shard_rank=0, shard_world=2)
    assert e.value.status == pd.PD_EINVAL


def test_sharded_reassembly_matches_single():
    """world=k slices exported in Morton order and reassembled == the world=1 diagram, bytewise."""
    wl = pdgen.make("C5", n=40009)
    ref = _gpu(wl)
    p = torch.from_numpy(wl.points).cuda()
    w = torch.from_numpy(wl.weights).cuda()
    for world, fl in ((2, 0), (3, 0), (3, pd.BALANCE)):
        parts = []
        perm = None
        bounds = []
        for r in range(world):
            d = pd.build_diagram(p, w, wl.box, shard_rank=r, shard_world=world, flags=fl)
            bounds.append((d.slice_begin, d.slice_end))
            parts.append(pd.export_slice(d))
            if perm is None:
                perm = pd.morton_perm(d).clone()
        # slices tile the Morton order (equal-count by default, equal-cost with BALANCE)
        assert bounds[0][0] == 0 and bounds[-1][1] == wl.n
        assert all(bounds[r][1] == bounds[r + 1][0] for r in range(world - 1))
        cat = [torch.cat([pp[k] for pp in parts]) for k in range(6)]
        full = pd.assemble(perm, *cat).to_numpy()
        for k in ("offsets", "neighbors", "areas", "volumes", "surface", "flags"):
            assert np.array_equal(getattr(ref, k), getattr(full, k)), (world, k)


def test_build_sharded_loopback():
    """pd_build_sharded through a real NCCL communicator of one rank (the only GPU of the test box): the
    header + LBVH broadcasts, the slice export, the owner broadcasts and the assembly run, and the result is
    byte-identical to pd_build.  Host and device inputs; rank 0's input errors are
    returned with their index."""
    wl = pdgen.make("C5", n=40009)
    ref = _gpu(wl)
    comm = pd.Comm(pd.Comm.unique_id(), 0, 1, 0)
    try:
        p = torch.from_numpy(wl.points).cuda()
        w = torch.from_numpy(wl.weights).cuda()
        for d in (pd.build_sharded(comm, p, w, wl.box).to_numpy(),
                  pd.build_sharded(comm, wl.points, wl.weights, wl.box, out_host=True),
                  pd.build_sharded(comm, p, w, wl.box, flags=pd.BALANCE).to_numpy()):
            for k in ("offsets", "neighbors", "areas", "volumes", "surface", "flags"):
                assert np.array_equal(getattr(ref, k), getattr(d, k)), k
        bad = wl.points.copy()
        bad[123, 2] = np.inf
        with pytest.raises(pd.PdError) as e:
            pd.build_sharded(comm, bad, wl.weights, wl.box)
        assert e.value.status == pd.PD_ENONFINITE and e.value.index == 123
        with pytest.raises(pd.PdError) as e:
            pd.build_sharded(comm, wl.points, wl.weights, wl.box, flags=pd.TETS)
        assert e.value.status == pd.PD_EINVAL
    finally:
        comm.close()


@pytest.mark.parametrize("n,bits", [(1, 62), (1000, 8), (4096 * 3 + 17, 62), (1_000_003, 62), (2_000_000, 20)])
def test_own_radix_sort_matches_stable_torch_sort(n, bits):
    """a4: the path's own LSD radix sort equals a stable sort (ties keep input order)."""
    g = torch.Generator().manual_seed(n)
    keys = torch.randint(0, 2 ** bits, (n,), generator=g, dtype=torch.int64).cuda()
    vals = torch.arange(n, dtype=torch.int32).cuda()
    ko, vo = pd.sort_pairs_u64(keys, vals)
    ref_k, ref_i = torch.sort(keys, stable=True)
    assert torch.equal(ko, ref_k) and torch.equal(vo, ref_i.to(torch.int32))


# ----------------------------------------------------------------- full sizes, sampled cells

# SURVEY.md §8(d) sample: 4096 random + 1024 cost tail (pd_cell_cost) + 1024 BOUNDARY + 1024 EMPTY + all OVERFLOW
FULL = ["C2", "C3", "C4", "C5"]


@pytest.mark.parametrize("cfg", FULL)
def test_full_size_sampled(cfg):
    wl = pdgen.make(cfg)
    p = torch.from_numpy(wl.points).cuda()
    w = None if wl.weights is None else torch.from_numpy(wl.weights).cuda()
    d = pd.build_diagram(p, w, wl.box, flags=pd.COST | pd.STATS)  # the bench launch configuration (+ counters)
    cost = pd.cell_cost(d).cpu().numpy()
    stats = d.stats
    g = d.to_numpy()
    ids = sample_cells(g, wl.n, seed=123, n_random=4096, n_stratum=1024, cost=cost)
    o = oracle.cells(wl.points, wl.weights, wl.box, ids=ids, threads=NT)
    rep = compare(g, o)
    print(cfg, rep.summary(), "gpu faces_dropped", stats["faces_dropped"], "near_degenerate",
          stats["faces_near_degenerate"], "degraded", stats["degraded_cells"])
    assert rep.ok, rep.summary()
    assert len(ids) >= 4096 + 1024
    # properties over ALL cells: box partition and adjacency symmetry
    bx = np.asarray(wl.box, np.float64)
    assert g.volumes.astype(np.float64).sum() == pytest.approx(np.prod(bx[3:] - bx[:3]), rel=1e-5)
    # symmetry: (i,j) and (j,i) both present, except near-degenerate faces below tau_ij
    rows = np.repeat(np.arange(wl.n), np.diff(g.offsets))
    fwd = rows.astype(np.int64) * wl.n + g.neighbors
    bwd = g.neighbors.astype(np.int64) * wl.n + rows
    one_sided = ~np.isin(fwd, bwd)
    tau = 1e-9 * np.maximum(g.surface[rows], g.surface[g.neighbors])
    print(cfg, "one-sided pairs", int(one_sided.sum()), "of", len(fwd))
    assert np.all(g.areas[one_sided] < tau[one_sided])
    assert one_sided.sum() <= 1e-5 * len(fwd)
    assert not np.any(g.flags & pd.CELL_OVERFLOW)
    # robustness counters (pd_stats): near-degenerate faces are counted, not silently dropped
    small = g.areas < 1e-9 * g.surface[rows]
    assert stats["faces_near_degenerate"] == int(small.sum())
    assert stats["degraded_cells"] == int(np.count_nonzero(g.flags & pd.CELL_DEGRADED))
