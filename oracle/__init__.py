"""CPU double-precision brute-force oracle (ctypes wrapper around oracle/pd_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this package.  It shares no code with the CUDA path.

What it computes (Eq. 1, restricted to the box of PAPER.md:553): for each
requested cell i, K_i = B ∩ ⋂_{j≠i} H_ij by clipping the box against every other site's bisecting
plane (§4.1 "if a cell is iteratively clipped by all bisecting planes ..."), with
neighbours = bisector faces of positive area, face areas (Newell), volume, total surface and flags.
See pd_oracle.c's header for the exact algorithm and the readings it takes.

Parity status: pinned by tests/test_oracle_pins.py (closed forms, brute vertex enumeration,
lattices, separable-weight power grids, partition, symmetry, empty power sphere, ownership,
Qhull lifting).  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pd_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

EMPTY, BOUNDARY, OVERFLOW, DUPLICATE, DEGRADED = 1, 2, 4, 8, 16


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, -O2, no fast-math: IEEE double semantics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread",
                               "-ffp-contract=off", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        L.orc_run.restype = P
        L.orc_run.argtypes = [P, P, ctypes.c_int64, P, P, ctypes.c_int64, ctypes.c_int, ctypes.c_int]
        L.orc_nnz.restype = ctypes.c_int64
        L.orc_nnz.argtypes = [P]
        L.orc_copy.restype = None
        L.orc_copy.argtypes = [P, P, P, P, P, P, P]
        L.orc_run_kdtree.restype = P
        L.orc_run_kdtree.argtypes = [P, P, ctypes.c_int64, P, P, ctypes.c_int64, ctypes.c_int]
        L.orc_kd_build.restype = P
        L.orc_kd_build.argtypes = [P, P, ctypes.c_int64, P]
        L.orc_kd_run.restype = P
        L.orc_kd_run.argtypes = [P, P, ctypes.c_int64, ctypes.c_int]
        L.orc_kd_free.restype = None
        L.orc_kd_free.argtypes = [P]
        L.orc_counts.restype = None
        L.orc_counts.argtypes = [P, P, P]
        L.orc_free.restype = None
        L.orc_free.argtypes = [P]
        L.orc_cell_geometry.restype = ctypes.c_int
        L.orc_cell_geometry.argtypes = [P, P, ctypes.c_int64, P, ctypes.c_int64, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_int, P, P, P, P, P]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data if a is not None else None


@dataclass
class OracleCells:
    ids: np.ndarray        # int64 [m] cell ids
    offsets: np.ndarray    # int64 [m+1]
    nbr: np.ndarray        # int32 [nnz] ascending per row
    area: np.ndarray       # float64 [nnz]
    vol: np.ndarray        # float64 [m]
    surf: np.ndarray       # float64 [m]
    flags: np.ndarray      # uint8 [m]
    dropped: np.ndarray = None  # int32 [m] bisector faces with area <= 1e-13 S (not neighbours, R2)
    small: np.ndarray = None    # int32 [m] neighbour faces with area < 1e-9 S (near-degenerate)

    def row(self, t):
        a, b = self.offsets[t], self.offsets[t + 1]
        return self.nbr[a:b], self.area[a:b]


def _prep(points, weights, box):
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float32).reshape(-1, 3))
    w = None if weights is None else np.ascontiguousarray(np.asarray(weights, dtype=np.float32))
    bx = np.ascontiguousarray(np.asarray(box, dtype=np.float64).reshape(6))
    return pts, w, bx


def _collect(L, r, ids) -> OracleCells:
    try:
        nnz = L.orc_nnz(r)
        m = len(ids)
        off = np.zeros(m + 1, np.int64)
        nbr = np.zeros(max(nnz, 1), np.int32)
        area = np.zeros(max(nnz, 1), np.float64)
        vol = np.zeros(m, np.float64)
        surf = np.zeros(m, np.float64)
        flags = np.zeros(m, np.uint8)
        L.orc_copy(r, _ptr(off), _ptr(nbr), _ptr(area), _ptr(vol), _ptr(surf), _ptr(flags))
        dropped = np.zeros(m, np.int32)
        small = np.zeros(m, np.int32)
        L.orc_counts(r, _ptr(dropped), _ptr(small))
    finally:
        L.orc_free(r)
    return OracleCells(ids, off, nbr[:nnz], area[:nnz], vol, surf, flags, dropped, small)


class KdReference:
    """The CPU reference of the same definition (pd_oracle.c orc_kd_*): a k-d tree with
    per-subtree bounding box and max weight, built once per point set; `cells(ids)` walks it best-first per
    cell and stops at the weighted radius of security.  A reported CPU baseline, not the parity oracle."""

    def __init__(self, points, weights, box):
        self.pts, self.w, self.bx = _prep(points, weights, box)
        self.n = self.pts.shape[0]
        self._L = lib()
        self._h = self._L.orc_kd_build(_ptr(self.pts), _ptr(self.w), self.n, _ptr(self.bx))

    def cells(self, ids=None, threads: int | None = None) -> OracleCells:
        ids = np.arange(self.n, dtype=np.int64) if ids is None else np.ascontiguousarray(np.asarray(ids, np.int64))
        r = self._L.orc_kd_run(self._h, _ptr(ids), len(ids), int(threads or os.cpu_count() or 1))
        return _collect(self._L, r, ids)

    def close(self):
        if self._h:
            self._L.orc_kd_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def cells(points, weights, box, ids=None, threads: int | None = None, order_k: int = 64,
          kdtree: bool = False) -> OracleCells:
    """Oracle cells for `ids` (default: all).  box = (lo.x, lo.y, lo.z, hi.x, hi.y, hi.z).
    kdtree=True: the CPU reference of the same definition instead (pd_oracle.c orc_run_kdtree: the same
    clipper, fed by a best-first walk of a weight-augmented k-d tree, stopped by the weighted radius of
    security) -- a
    reported CPU baseline; the parity tests use the brute-force oracle."""
    pts, w, bx = _prep(points, weights, box)
    n = pts.shape[0]
    ids = np.arange(n, dtype=np.int64) if ids is None else np.ascontiguousarray(np.asarray(ids, dtype=np.int64))
    threads = threads or os.cpu_count() or 1
    L = lib()
    if kdtree:
        r = L.orc_run_kdtree(_ptr(pts), _ptr(w), n, _ptr(bx), _ptr(ids), len(ids), int(threads))
    else:
        r = L.orc_run(_ptr(pts), _ptr(w), n, _ptr(bx), _ptr(ids), len(ids), int(threads), int(order_k))
    return _collect(L, r, ids)


@dataclass
class CellGeometry:
    tags: np.ndarray      # int [F]  (>=0 neighbour id, <0 wall)
    loops: list           # list of float64 [k, 3] world-coordinate vertex loops (CCW from outside)
    planes: np.ndarray    # float64 [F, 4] (n, d) in site-local coordinates
    flags: int


def cell_geometry(points, weights, box, i: int, order_k: int = 64,
                  max_faces: int = 4096, max_verts: int = 1 << 16) -> CellGeometry:
    pts, w, bx = _prep(points, weights, box)
    tags = np.zeros(max_faces, np.int32)
    nv = np.zeros(max_faces, np.int32)
    planes = np.zeros((max_faces, 4), np.float64)
    xyz = np.zeros((max_verts, 3), np.float64)
    fl = np.zeros(1, np.int32)
    nf = lib().orc_cell_geometry(_ptr(pts), _ptr(w), pts.shape[0], _ptr(bx), int(i), int(order_k),
                                 max_faces, max_verts, _ptr(tags), _ptr(nv), _ptr(planes), _ptr(xyz),
                                 _ptr(fl))
    if nf < 0:
        raise RuntimeError("cell_geometry capacity exceeded")
    loops, o = [], 0
    for f in range(nf):
        loops.append(xyz[o:o + nv[f]].copy())
        o += nv[f]
    return CellGeometry(tags[:nf].copy(), loops, planes[:nf].copy(), int(fl[0]))


def dual_tets(points, weights, box, ids=None, order_k: int = 64):
    """Dual tetrahedra of the diagram in the box (the "explicit mesh" of
    PAPER.md:343, 398): for each requested cell i, every vertex v of K_i (the same point in several
    of the oracle's face loops -- the clipper builds shared points bit-identically) is a corner where
    the faces tagged T(v) meet.  If T(v) is exactly three bisector faces {a, b, c} of area
    > 1e-13 S_i (reading R2; no wall), v is power-equidistant from p_i, p_a, p_b, p_c and
    no site is closer, so {i, a, b, c} is a tet of the regular triangulation.
    Each tet is reported once, by its lowest id.  Returns (int64 [T, 4] rows (i<a<b<c) sorted
    lexicographically, number of vertices where more than three faces meet (degenerate, skipped)).
    Pinned by tests/test_oracle_pins.py::test_dual_tets_* (scipy Delaunay / lifted Qhull)."""
    n = len(points)
    out, ndeg = [], 0
    for i in (range(n) if ids is None else ids):
        g = cell_geometry(points, weights, box, int(i), order_k)
        if not g.loops:
            continue
        areas = []
        for lp in g.loops:
            A = 0.5 * np.sum(np.cross(lp, np.roll(lp, -1, axis=0)), axis=0)
            areas.append(float(np.sqrt(A @ A)))
        amin = 1e-13 * sum(areas)
        at = {}
        for f, lp in enumerate(g.loops):
            for v in lp:
                at.setdefault((v[0], v[1], v[2]), set()).add(f)
        for fs in at.values():
            if len(fs) > 3:
                ndeg += 1
                continue
            if len(fs) < 3:
                continue
            tags = sorted(int(g.tags[f]) for f in fs)
            if tags[0] < 0 or any(areas[f] <= amin for f in fs):
                continue
            if int(i) < tags[0]:
                out.append((int(i), tags[0], tags[1], tags[2]))
    t = np.array(sorted(out), dtype=np.int64).reshape(-1, 4)
    return t, ndeg
