"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no bisectors, no clipping, no culling): it only
draws point sets and weights with the laws of the paper's workloads (§5.1)
and the BASELINE.json configs C1-C5 as fixed by SURVEY.md §8(d).  Both the CUDA path and the
oracle consume its output bytes; neither implements anything here.

PRNG: SplitMix64, counter based.  Stream s, counter i -> u64 = mix(seed_s + (i+1)*GOLDEN), where
seed_s = mix(seed * 0x100000001B3 + s).  Uniform in [0,1): (u >> 11) * 2^-53 (double).  Normals:
Box-Muller in double.  Everything is vectorised numpy; the output is bit-identical across runs.
"""
from __future__ import annotations

import dataclasses
import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

OMEGA = (-10.0, 10.0)  # PAPER.md:311 "All configurations sample points within the domain [-10,10]^3"


def _mix(z: np.ndarray) -> np.ndarray:
    z = z.copy()
    z ^= z >> np.uint64(30)
    z *= _M1
    z ^= z >> np.uint64(27)
    z *= _M2
    z ^= z >> np.uint64(31)
    return z


def _stream_seed(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        s = np.array([(seed * 0x100000001B3 + stream) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64)
        return _mix(s)[0]


def u64(seed: int, stream: int, n: int, offset: int = 0) -> np.ndarray:
    """n raw 64-bit draws of stream `stream` starting at counter `offset`."""
    base = _stream_seed(seed, stream)
    with np.errstate(over="ignore"):
        ctr = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
        return _mix(base + ctr * GOLDEN)


def uniform(seed: int, stream: int, n: int, offset: int = 0) -> np.ndarray:
    """Doubles in [0, 1)."""
    return (u64(seed, stream, n, offset) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def normal(seed: int, stream: int, n: int) -> np.ndarray:
    """Standard normals by Box-Muller (two uniform sub-streams)."""
    u1 = uniform(seed, stream, n)
    u2 = uniform(seed, stream + 1000003, n)
    u1 = 1.0 - u1  # (0, 1]
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def _box_points(lo: float, hi: float, seed: int, stream: int, n: int) -> np.ndarray:
    p = np.empty((n, 3), dtype=np.float64)
    for k in range(3):
        p[:, k] = lo + (hi - lo) * uniform(seed, stream + k, n)
    return p


def to_f32_in_box(p: np.ndarray, lo: float, hi: float) -> np.ndarray:
    """Round to float32 and clamp into the closed box (PAPER.md:318 'points are clamped to Omega')."""
    q = p.astype(np.float32)
    np.clip(q, np.float32(lo), np.float32(hi), out=q)
    return np.ascontiguousarray(q)


# ---------------------------------------------------------------------------------------------
# Paper laws (§5.1)
# ---------------------------------------------------------------------------------------------

def white_noise(n: int, seed: int, lo: float = OMEGA[0], hi: float = OMEGA[1]) -> np.ndarray:
    """p_i ~ U(Omega)."""
    return to_f32_in_box(_box_points(lo, hi, seed, 10, n), lo, hi)


def clustered(n: int, seed: int, k: int = 10, sigma: float = 0.1,
              center_lo: float = OMEGA[0], center_hi: float = OMEGA[1],
              lo: float = OMEGA[0], hi: float = OMEGA[1], stream: int = 20) -> np.ndarray:
    """c_j ~ U(Omega), p_i ~ N(c_{i mod K}, sigma^2 I), clamped (round-robin split,
    SURVEY.md §8(c) Q15)."""
    centers = _box_points(center_lo, center_hi, seed, stream, k)
    g = np.stack([normal(seed, stream + 10 + 2 * a, n) for a in range(3)], axis=1)
    p = centers[np.arange(n) % k] + sigma * g
    return to_f32_in_box(p, lo, hi)


def density_gradient(n: int, seed: int, lo: float = OMEGA[0], hi: float = OMEGA[1]) -> np.ndarray:
    """x = a + (b-a) sqrt(u), y,z ~ U(a,b)."""
    p = _box_points(lo, hi, seed, 30, n)
    p[:, 0] = lo + (hi - lo) * np.sqrt(uniform(seed, 33, n))
    return to_f32_in_box(p, lo, hi)


def median_nn_distance(points: np.ndarray, seed: int = 0, max_queries: int = 1 << 17) -> float:
    """d_nn = median nearest-neighbour distance.  Lower median for even counts; above
    2^17 sites the median is taken over a seeded subsample of query sites against the full set
    (SURVEY.md §8(c) Q14).  Uses scipy's k-d tree: input preparation, not the method."""
    from scipy.spatial import cKDTree
    pts = np.asarray(points, dtype=np.float64)
    n = pts.shape[0]
    if n < 2:
        raise ValueError("median_nn_distance needs >= 2 sites")
    tree = cKDTree(pts)
    if n > max_queries:
        idx = np.sort(np.unique((u64(seed, 90, max_queries) % np.uint64(n)).astype(np.int64)))
    else:
        idx = np.arange(n)
    d, _ = tree.query(pts[idx], k=2)
    d = np.sort(d[:, 1])
    return float(d[(len(d) - 1) // 2])


def weights_paper(n: int, d_nn: float, seed: int, ratio: float = 1.0) -> np.ndarray:
    """w_i ~ N(0, (ratio * d_nn^2 / 3)^2)  (ratio per SPEC sample_weights)."""
    return (ratio * d_nn * d_nn / 3.0 * normal(seed, 40, n)).astype(np.float32)


def weights_lognormal(n: int, d_nn: float, seed: int) -> np.ndarray:
    """w = (d_nn^2/3) exp(g), g ~ N(0,1)."""
    return (d_nn * d_nn / 3.0 * np.exp(normal(seed, 50, n))).astype(np.float32)


def weights_student_t(n: int, d_nn: float, seed: int, nu: float = 2.0) -> np.ndarray:
    """w = (d_nn^2/3) t, t ~ Student-t(nu)  (heavy-tailed).  For nu = 2,
    chi^2_2 = -2 ln U, so t = Z / sqrt(chi^2/nu)."""
    z = normal(seed, 60, n)
    if nu != 2.0:
        raise ValueError("only nu = 2 is implemented")
    u = 1.0 - uniform(seed, 62, n)
    chi2 = -2.0 * np.log(u)
    t = z / np.sqrt(chi2 / nu)
    return (d_nn * d_nn / 3.0 * t).astype(np.float32)


# ---------------------------------------------------------------------------------------------
# Scene-like (Radiant-Foam-style) heterogeneous density, SURVEY.md §8(d) C4
# ---------------------------------------------------------------------------------------------

_SPHERES = [((0.0, 0.0, 0.0), 1.5), ((3.0, 2.0, -1.0), 1.0), ((-3.0, 1.0, -1.2), 0.8),
            ((1.0, -3.0, -1.5), 0.5)]


def _surface_samples(n: int, seed: int, stream: int):
    """n points on the scene surfaces + unit normals: 1/3 ground disk z=-2, r<8; 2/3 split evenly
    over the 4 spheres."""
    n_disk = n // 3
    n_sph = n - n_disk
    pts = np.empty((n, 3))
    nrm = np.empty((n, 3))
    r = 8.0 * np.sqrt(uniform(seed, stream, n_disk))
    th = 2.0 * np.pi * uniform(seed, stream + 1, n_disk)
    pts[:n_disk, 0] = r * np.cos(th)
    pts[:n_disk, 1] = r * np.sin(th)
    pts[:n_disk, 2] = -2.0
    nrm[:n_disk] = (0.0, 0.0, 1.0)
    which = np.arange(n_sph) % len(_SPHERES)
    cz = 2.0 * uniform(seed, stream + 2, n_sph) - 1.0
    ph = 2.0 * np.pi * uniform(seed, stream + 3, n_sph)
    sz = np.sqrt(np.maximum(0.0, 1.0 - cz * cz))
    dirs = np.stack([sz * np.cos(ph), sz * np.sin(ph), cz], axis=1)
    cen = np.array([c for c, _ in _SPHERES])[which]
    rad = np.array([r_ for _, r_ in _SPHERES])[which]
    pts[n_disk:] = cen + rad[:, None] * dirs
    nrm[n_disk:] = dirs
    return pts, nrm


def scene_like(n: int, seed: int) -> np.ndarray:
    """55% on surfaces with normal jitter N(0, 0.01^2); 35% near-surface N(0, 0.15^2 I); 10% radial
    background r ~ U(4,17) (density ~ r^-2) kept if inside Omega."""
    n_s = int(round(0.55 * n))
    n_ns = int(round(0.35 * n))
    n_bg = n - n_s - n_ns
    ps, ns = _surface_samples(n_s, seed, 100)
    ps = ps + (0.01 * normal(seed, 110, n_s))[:, None] * ns
    pn, _ = _surface_samples(n_ns, seed, 120)
    pn = pn + 0.15 * np.stack([normal(seed, 130 + 2 * a, n_ns) for a in range(3)], axis=1)
    # background: draw 3x candidates, keep the first n_bg that lie inside Omega (deterministic)
    m = 3 * n_bg + 64
    r = 4.0 + 13.0 * uniform(seed, 140, m)
    cz = 2.0 * uniform(seed, 141, m) - 1.0
    ph = 2.0 * np.pi * uniform(seed, 142, m)
    sz = np.sqrt(np.maximum(0.0, 1.0 - cz * cz))
    pb = r[:, None] * np.stack([sz * np.cos(ph), sz * np.sin(ph), cz], axis=1)
    inside = np.all(np.abs(pb) <= 10.0, axis=1)
    pb = pb[inside][:n_bg]
    assert pb.shape[0] == n_bg, "background rejection ran short"
    p = np.concatenate([ps, pn, pb], axis=0)
    return to_f32_in_box(p, *OMEGA)


# ---------------------------------------------------------------------------------------------
# BASELINE.json configs
# ---------------------------------------------------------------------------------------------

@dataclasses.dataclass
class Workload:
    name: str
    points: np.ndarray          # float32 [n, 3]
    weights: np.ndarray | None  # float32 [n] or None (Voronoi)
    box: tuple                  # (lo0, lo1, lo2, hi0, hi1, hi2)
    description: str

    @property
    def n(self) -> int:
        return int(self.points.shape[0])


CONFIG_SIZES = {"C1": 1_000, "C2": 1_000_000, "C3": 4_000_000, "C4": 10_000_000, "C5": 20_000_000}
OMEGA_BOX = (OMEGA[0],) * 3 + (OMEGA[1],) * 3


def make(config: str, n: int | None = None, seed: int | None = None) -> Workload:
    """Build config C1..C5 (optionally at a reduced size n for parity tests, same law)."""
    base_seed = {"C1": 1, "C2": 2, "C3": 3, "C4": 4, "C5": 5}[config]
    seed = base_seed if seed is None else seed
    n = CONFIG_SIZES[config] if n is None else int(n)
    if config == "C1":
        p = white_noise(n, seed, 0.0, 1.0)
        return Workload("C1", p, None, (0.0, 0.0, 0.0, 1.0, 1.0, 1.0),
                        f"{n} U([0,1)^3) points, unweighted Voronoi, box [0,1]^3")
    if config == "C2":
        return Workload("C2", white_noise(n, seed), None, OMEGA_BOX,
                        f"{n} U(Omega) points, unweighted Voronoi")
    if config == "C3":
        n_bg = n // 10
        pb = white_noise(n_bg, seed).astype(np.float64)
        pc = clustered(n - n_bg, seed, k=10, sigma=0.36, center_lo=-8.0, center_hi=8.0).astype(np.float64)
        p = to_f32_in_box(np.concatenate([pb, pc]), *OMEGA)
        w = weights_lognormal(n, median_nn_distance(p, seed), seed)
        return Workload("C3", p, w, OMEGA_BOX,
                        f"{n} pts: 10% U(Omega) + 90% in K=10 Gaussians sigma=0.36, log-normal weights")
    if config == "C4":
        p = scene_like(n, seed)
        w = weights_paper(n, median_nn_distance(p, seed), seed)
        return Workload("C4", p, w, OMEGA_BOX,
                        f"{n} scene-like pts (surfaces+near-surface+radial bg), w~N(0,(d_nn^2/3)^2)")
    if config == "C5":
        n_u = n // 2
        pu = white_noise(n_u, seed).astype(np.float64)
        pc = clustered(n - n_u, seed, k=10, sigma=0.1).astype(np.float64)
        p = to_f32_in_box(np.concatenate([pu, pc]), *OMEGA)
        w = weights_student_t(n, median_nn_distance(p, seed), seed)
        return Workload("C5", p, w, OMEGA_BOX,
                        f"{n} pts: 50% U(Omega) + 50% K=10 Gaussians sigma=0.1, Student-t(2) weights")
    raise KeyError(config)
