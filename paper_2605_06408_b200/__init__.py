"""paper_2605_06408_b200 -- B200-native construction of 3D power / Voronoi diagrams.

Thin ctypes binding over the C ABI in include/pd.h (libpd.so, built in-tree for sm_100a).  This
module only marshals arguments: every step of the path (packing, Morton codes, sort, LBVH, refit,
the cell kernel, CSR) runs in the library's CUDA kernels.  There is no CPU fallback: if libpd.so
is missing or no CUDA device is present, `build_diagram` raises.

    import torch, paper_2605_06408_b200 as pd
    d = pd.build_diagram(points_cuda_f32_nx3, weights_cuda_f32_n_or_None, box=(lo..., hi...))
    d.offsets, d.neighbors, d.areas, d.volumes, d.surface, d.flags   # torch CUDA tensors
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpd.so")

PD_OK, PD_EINVAL, PD_EEMPTY, PD_ENONFINITE, PD_EOUTSIDE, PD_ENOMEM, PD_ECUDA, PD_ENCCL, PD_EINTERNAL = range(9)
IN_DEVICE, OUT_HOST, STATS, ISOTROPIC, DFS, PAPER_BOUND, COST, EXACT_NODES, NO_EXACT, BALANCE = (
    1, 2, 4, 8, 16, 64, 128, 256, 512, 1024)
WARM_START, TETS, WARM_ADAPTIVE, NO_AUTO_WARM, AUTO_WARM = 32, 2048, 4096, 8192, 16384
CELL_EMPTY, CELL_BOUNDARY, CELL_OVERFLOW, CELL_DUPLICATE, CELL_DEGRADED, CELL_NOT_OWNED = 1, 2, 4, 8, 16, 32

EXPORTED = ["pd_build", "pd_num_cells", "pd_nnz", "pd_on_host", "pd_offsets", "pd_neighbors", "pd_face_areas",
            "pd_volumes", "pd_surface", "pd_cell_flags", "pd_cell_cost", "pd_get_stats", "pd_free", "pd_slice_begin",
            "pd_slice_end", "pd_morton_perm", "pd_assemble", "pd_export_slice", "pd_slice_nnz",
            "pd_strerror", "pd_error_index", "pd_last_cuda_error", "pd_abi_version", "pd_last_launch_count",
            "pd_sort_pairs_u64", "pd_num_tets", "pd_tets", "pd_trim", "pd_comm_unique_id", "pd_comm_init",
            "pd_build_sharded", "pd_comm_free", "pd_comm_rank", "pd_comm_world", "pd_last_nccl_error",
            "pd_measure_fp32_peak", "pd_measure_l2_peak"]


class PdError(RuntimeError):
    def __init__(self, status: int, msg: str, index: int = -1):
        super().__init__(msg)
        self.status = status
        self.index = index


class _Box(ctypes.Structure):
    _fields_ = [("lo", ctypes.c_float * 3), ("hi", ctypes.c_float * 3)]


class _Options(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("stream", ctypes.c_void_p), ("leaf_size", ctypes.c_int),
                ("flags", ctypes.c_uint), ("shard_rank", ctypes.c_int), ("shard_world", ctypes.c_int)]


class Stats(ctypes.Structure):
    _fields_ = [("cells", ctypes.c_int64), ("nodes_visited", ctypes.c_int64), ("leaves_visited", ctypes.c_int64),
                ("sites_tested", ctypes.c_int64), ("clip_tests", ctypes.c_int64), ("clips", ctypes.c_int64),
                ("tier_cells", ctypes.c_int64 * 3), ("overflow_cells", ctypes.c_int64), ("queue_spills", ctypes.c_int64),
                ("nnz", ctypes.c_int64),
                ("ms_bvh", ctypes.c_double), ("ms_cells", ctypes.c_double), ("ms_csr", ctypes.c_double),
                ("ms_total", ctypes.c_double), ("ms_tier", ctypes.c_double * 3),
                ("warp_cycles", ctypes.c_int64 * 10), ("ms_knn", ctypes.c_double),
                ("faces_dropped", ctypes.c_int64), ("faces_near_degenerate", ctypes.c_int64),
                ("degraded_cells", ctypes.c_int64), ("warm_gain", ctypes.c_double), ("warm_start", ctypes.c_int64)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["tier_cells"] = list(self.tier_cells)
        d["ms_tier"] = list(self.ms_tier)
        d["warp_cycles"] = list(self.warp_cycles)
        return d


_lib = None


def load_library(path: str | None = None):
    """Load libpd.so (or $PD_LIB, an alternative in-tree build); raises (never falls back) if missing."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("PD_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not built: run `python -m paper_2605_06408_b200.build` (no CPU fallback)")
    L = ctypes.CDLL(path)
    P, I64 = ctypes.c_void_p, ctypes.c_int64
    L.pd_build.restype = ctypes.c_int
    L.pd_build.argtypes = [P, P, I64, P, P, ctypes.POINTER(P)]
    for name, rt in [("pd_num_cells", I64), ("pd_nnz", I64), ("pd_on_host", ctypes.c_int),
                     ("pd_offsets", P), ("pd_neighbors", P), ("pd_face_areas", P), ("pd_volumes", P),
                     ("pd_surface", P), ("pd_cell_flags", P), ("pd_cell_cost", P), ("pd_slice_begin", I64), ("pd_slice_end", I64),
                     ("pd_morton_perm", P), ("pd_slice_nnz", I64)]:
        getattr(L, name).restype = rt
        getattr(L, name).argtypes = [P]
    L.pd_get_stats.restype = ctypes.c_int
    L.pd_get_stats.argtypes = [P, ctypes.POINTER(Stats)]
    L.pd_free.restype = None
    L.pd_free.argtypes = [P]
    L.pd_export_slice.restype = ctypes.c_int
    L.pd_export_slice.argtypes = [P, P, P, P, P, P, P, ctypes.POINTER(I64), P]
    L.pd_assemble.restype = ctypes.c_int
    L.pd_assemble.argtypes = [P, P, P, P, P, P, P, I64, I64, P, ctypes.POINTER(P)]
    L.pd_strerror.restype = ctypes.c_char_p
    L.pd_strerror.argtypes = [ctypes.c_int]
    L.pd_error_index.restype = I64
    L.pd_last_cuda_error.restype = ctypes.c_char_p
    L.pd_abi_version.restype = ctypes.c_int
    L.pd_last_launch_count.restype = I64
    if hasattr(L, "pd_trim"):  # (older A/B builds of the library lack the newer entry points)
        L.pd_trim.restype = ctypes.c_int
        L.pd_trim.argtypes = [ctypes.c_int]
    if hasattr(L, "pd_build_sharded"):
        L.pd_comm_unique_id.restype = ctypes.c_int
        L.pd_comm_unique_id.argtypes = [P]
        L.pd_comm_init.restype = ctypes.c_int
        L.pd_comm_init.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(P)]
        L.pd_build_sharded.restype = ctypes.c_int
        L.pd_build_sharded.argtypes = [P, P, P, I64, P, P, ctypes.POINTER(P)]
        L.pd_comm_free.restype = None
        L.pd_comm_free.argtypes = [P]
        L.pd_comm_rank.restype = ctypes.c_int
        L.pd_comm_rank.argtypes = [P]
        L.pd_comm_world.restype = ctypes.c_int
        L.pd_comm_world.argtypes = [P]
        L.pd_last_nccl_error.restype = ctypes.c_char_p
    if hasattr(L, "pd_measure_fp32_peak"):
        L.pd_measure_fp32_peak.restype = ctypes.c_int
        L.pd_measure_fp32_peak.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
        L.pd_measure_l2_peak.restype = ctypes.c_int
        L.pd_measure_l2_peak.argtypes = [ctypes.c_int, I64, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    if hasattr(L, "pd_tets"):
        L.pd_num_tets.restype = I64
        L.pd_num_tets.argtypes = [P]
        L.pd_tets.restype = P
        L.pd_tets.argtypes = [P]
    if hasattr(L, "pd_sort_pairs_u64"):  # optional test hook (absent in older A/B builds)
        L.pd_sort_pairs_u64.restype = ctypes.c_int
        L.pd_sort_pairs_u64.argtypes = [P, P, I64, P, P, P]
    _lib = L
    return L


def last_launch_count() -> int:
    return int(load_library().pd_last_launch_count())


def _check(status: int):
    if status != PD_OK:
        L = load_library()
        msg = L.pd_strerror(status).decode()
        idx = int(L.pd_error_index()) if status in (PD_ENONFINITE, PD_EOUTSIDE) else -1
        if status == PD_ECUDA:
            msg += ": " + L.pd_last_cuda_error().decode()
        if status == PD_ENCCL:
            msg += ": " + L.pd_last_nccl_error().decode()
        if idx >= 0:
            msg += f" (point {idx})"
        raise PdError(status, msg, idx)


class _Handle:
    """Owns one pd_result*; freed when the last view of its arrays goes away."""

    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        if self.ptr and _lib is not None:
            _lib.pd_free(self.ptr)
            self.ptr = None


class _CudaView:
    """__cuda_array_interface__ over memory owned by a _Handle (zero-copy torch view)."""

    def __init__(self, handle, ptr, shape, typestr):
        self._h = handle
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr or 0, False),
                                         "version": 3, "strides": None, "stream": None}


_TYPES = {"offsets": ("<i8", np.int64), "neighbors": ("<i4", np.int32), "areas": ("<f4", np.float32),
          "volumes": ("<f4", np.float32), "surface": ("<f4", np.float32), "flags": ("|u1", np.uint8)}


@dataclass
class Diagram:
    n: int
    nnz: int
    offsets: object     # int64 [n+1]
    neighbors: object   # int32 [nnz], ascending per row, original ids
    areas: object       # float32 [nnz]
    volumes: object     # float32 [n]
    surface: object     # float32 [n]
    flags: object       # uint8 [n]
    stats: dict
    on_host: bool
    handle: object = None
    slice_begin: int = 0
    slice_end: int = 0
    tets: object = None  # int32 [ntets, 4] with flags=TETS (pd_tets), else None

    def row(self, i):
        a, b = int(self.offsets[i]), int(self.offsets[i + 1])
        return self.neighbors[a:b], self.areas[a:b]

    def to_numpy(self) -> "Diagram":
        if self.on_host:
            return self
        cv = lambda t: t.cpu().numpy()
        return Diagram(self.n, self.nnz, cv(self.offsets), cv(self.neighbors), cv(self.areas), cv(self.volumes),
                       cv(self.surface), cv(self.flags), self.stats, True, self.handle, self.slice_begin,
                       self.slice_end, None if self.tets is None else cv(self.tets))


def _wrap(ptr, stream_ptr) -> Diagram:
    L = load_library()
    h = _Handle(ptr)
    n = int(L.pd_num_cells(ptr))
    nnz = int(L.pd_nnz(ptr))
    on_host = bool(L.pd_on_host(ptr))
    st = Stats()
    L.pd_get_stats(ptr, ctypes.byref(st))
    sizes = {"offsets": n + 1, "neighbors": nnz, "areas": nnz, "volumes": n, "surface": n, "flags": n}
    ptrs = {"offsets": L.pd_offsets(ptr), "neighbors": L.pd_neighbors(ptr), "areas": L.pd_face_areas(ptr),
            "volumes": L.pd_volumes(ptr), "surface": L.pd_surface(ptr), "flags": L.pd_cell_flags(ptr)}
    arrs = {}
    for k, size in sizes.items():
        tstr, npt = _TYPES[k]
        if on_host:
            if size == 0 or not ptrs[k]:
                arrs[k] = np.zeros(0, npt)
            else:
                buf = (ctypes.c_char * (size * np.dtype(npt).itemsize)).from_address(ptrs[k])
                a = np.frombuffer(buf, dtype=npt, count=size)
                arrs[k] = a
        else:
            import torch
            arrs[k] = torch.as_tensor(_CudaView(h, ptrs[k], (size,), tstr), device="cuda")
    d = Diagram(n, nnz, arrs["offsets"], arrs["neighbors"], arrs["areas"], arrs["volumes"], arrs["surface"],
                arrs["flags"], st.as_dict(), on_host, h, int(L.pd_slice_begin(ptr)), int(L.pd_slice_end(ptr)))
    tp = L.pd_tets(ptr) if hasattr(L, "pd_tets") else None
    if tp:
        nt = int(L.pd_num_tets(ptr))
        if on_host:
            buf = (ctypes.c_char * max(nt * 16, 1)).from_address(tp)
            d.tets = np.frombuffer(buf, dtype=np.int32, count=nt * 4).reshape(nt, 4)
        else:
            import torch
            d.tets = torch.as_tensor(_CudaView(h, tp, (nt, 4), "<i4"), device="cuda")
    return d


def _ptr_of(a):
    if a is None:
        return None, False
    try:
        import torch
        if isinstance(a, torch.Tensor):
            if not a.is_contiguous():
                raise ValueError("tensor must be contiguous")
            if a.dtype != torch.float32:
                raise TypeError("float32 expected")
            return a.data_ptr(), a.is_cuda
    except ImportError:
        pass
    if not (isinstance(a, np.ndarray) and a.dtype == np.float32 and a.flags.c_contiguous):
        raise TypeError("host arrays must be contiguous float32 (build_diagram converts and keeps them)")
    return a.ctypes.data, False


def _prepare(points, weights, box, device, stream, leaf_size, flags, out_host, shard_rank=0, shard_world=1):
    """Marshal pd_build's arguments (no arithmetic): returns (keep, pp, wp, n, opt, bx, stream)."""
    keep = []  # host copies made here stay alive until the C call returns
    if points is not None and not hasattr(points, "data_ptr"):
        points = np.ascontiguousarray(np.asarray(points, dtype=np.float32).reshape(-1, 3))
        keep.append(points)
    if weights is not None and not hasattr(weights, "data_ptr"):
        weights = np.ascontiguousarray(np.asarray(weights, dtype=np.float32).reshape(-1))
        keep.append(weights)
    pp, p_dev = _ptr_of(points)
    wp, w_dev = _ptr_of(weights)
    if weights is not None and points is not None and w_dev != p_dev:
        raise ValueError("points and weights must both be on the device or both on the host")
    n = int(points.shape[0]) if points is not None else 0
    opt = _Options()
    if device is None:
        device = points.device.index if (p_dev and points.device.index is not None) else 0
    opt.device = int(device)
    if stream is None and (p_dev or points is None):
        import torch
        if torch.cuda.is_available():
            stream = torch.cuda.current_stream(device).cuda_stream
    opt.stream = ctypes.c_void_p(int(stream) if stream else 0)
    opt.leaf_size = int(leaf_size)
    opt.flags = int(flags) | (IN_DEVICE if p_dev else 0) | (OUT_HOST if out_host else 0)
    opt.shard_rank = int(shard_rank)
    opt.shard_world = int(shard_world)
    bx = None
    if box is not None:
        b = [float(v) for v in box]
        bx = _Box((ctypes.c_float * 3)(*b[:3]), (ctypes.c_float * 3)(*b[3:]))
    return keep, pp, wp, n, opt, bx, stream


def build_diagram(points, weights=None, box=None, *, device: int | None = None, stream=None, leaf_size: int = 0,
                  flags: int = 0, out_host: bool = False, shard_rank: int = 0, shard_world: int = 1) -> Diagram:
    """pd_build (include/pd.h).  points: float32 [n,3] (torch CUDA tensor => device input, else host
    array); weights: float32 [n] or None; box: (lo.x, lo.y, lo.z, hi.x, hi.y, hi.z) or None.
    Device outputs come back as zero-copy torch CUDA tensors; with out_host=True as numpy arrays."""
    L = load_library()
    keep, pp, wp, n, opt, bx, stream = _prepare(points, weights, box, device, stream, leaf_size, flags, out_host,
                                                shard_rank, shard_world)
    out = ctypes.c_void_p()
    status = L.pd_build(pp, wp, n, ctypes.byref(bx) if bx is not None else None, ctypes.byref(opt),
                        ctypes.byref(out))
    del keep
    _check(status)
    return _wrap(out.value, stream)


class Comm:
    """pd_comm (include/pd.h): an NCCL communicator inside libpd, one rank per GPU."""

    def __init__(self, uid: bytes, rank: int, world: int, device: int):
        L = load_library()
        if len(uid) != 128:
            raise ValueError("unique id must be 128 bytes")
        buf = (ctypes.c_ubyte * 128).from_buffer_copy(uid)
        self.ptr = ctypes.c_void_p()
        _check(L.pd_comm_init(buf, int(rank), int(world), int(device), ctypes.byref(self.ptr)))
        self.rank, self.world, self.device = int(rank), int(world), int(device)

    @staticmethod
    def unique_id() -> bytes:
        buf = (ctypes.c_ubyte * 128)()
        _check(load_library().pd_comm_unique_id(buf))
        return bytes(buf)

    def close(self):
        if self.ptr and self.ptr.value and _lib is not None:
            _lib.pd_comm_free(self.ptr)
        self.ptr = None

    def __del__(self):
        self.close()


def build_sharded(comm: Comm, points, weights=None, box=None, *, n: int | None = None, stream=None,
                  leaf_size: int = 0, flags: int = 0, out_host: bool = False) -> Diagram:
    """pd_build_sharded: collective over the ranks of `comm`.  points/weights/box are read on rank 0 only
    (other ranks may pass None together with n); every rank returns the full diagram."""
    L = load_library()
    keep, pp, wp, n0, opt, bx, stream = _prepare(points, weights, box, comm.device, stream, leaf_size, flags,
                                                 out_host)
    if points is None:
        if n is None:
            raise ValueError("ranks without points must pass n")
        n0 = int(n)
        # the device input flag must agree with rank 0's (it only tells rank 0 how to read points)
    out = ctypes.c_void_p()
    status = L.pd_build_sharded(comm.ptr, pp, wp, n0, ctypes.byref(bx) if bx is not None else None,
                                ctypes.byref(opt), ctypes.byref(out))
    del keep
    _check(status)
    return _wrap(out.value, stream)


def export_slice(d: Diagram, stream=None):
    """Morton-ordered export of a sharded result (pd_export_slice): returns torch tensors
    (cnt, vol, surf, flags, rows_nbr, rows_area) on the device."""
    import torch
    L = load_library()
    length = d.slice_end - d.slice_begin
    dev = d.volumes.device
    cnt = torch.empty(length, dtype=torch.int32, device=dev)
    vol = torch.empty(length, dtype=torch.float32, device=dev)
    surf = torch.empty(length, dtype=torch.float32, device=dev)
    flg = torch.empty(length, dtype=torch.uint8, device=dev)
    cap = int(L.pd_slice_nnz(d.handle.ptr))
    rn = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    ra = torch.empty(max(cap, 1), dtype=torch.float32, device=dev)
    total = ctypes.c_int64()
    if stream is None:
        stream = torch.cuda.current_stream(dev).cuda_stream
    _check(L.pd_export_slice(d.handle.ptr, cnt.data_ptr(), vol.data_ptr(), surf.data_ptr(), flg.data_ptr(),
                             rn.data_ptr(), ra.data_ptr(), ctypes.byref(total), ctypes.c_void_p(stream)))
    t = int(total.value)
    return cnt, vol, surf, flg, rn[:t], ra[:t]


def measure_fp32_peak(device: int = 0, reps: int = 5) -> float:
    """pd_measure_fp32_peak: FP32 FFMA lane-ops/s of the device (roofline denominator)."""
    v = ctypes.c_double()
    _check(load_library().pd_measure_fp32_peak(int(device), int(reps), ctypes.byref(v)))
    return v.value


def measure_l2_peak(device: int = 0, nbytes: int = 48 << 20, reps: int = 5) -> float:
    """pd_measure_l2_peak: L2-resident read bytes/s of the device (roofline denominator)."""
    v = ctypes.c_double()
    _check(load_library().pd_measure_l2_peak(int(device), int(nbytes), int(reps), ctypes.byref(v)))
    return v.value


def trim(device: int = 0):
    """pd_trim: release the cached build workspace and pinned host buffers of `device`."""
    _check(load_library().pd_trim(int(device)))


def sort_pairs_u64(keys, vals, stream=None):
    """pd_sort_pairs_u64 test hook: stable sort of int64 (non-negative) keys with int32 values (CUDA)."""
    import torch
    L = load_library()
    ko = torch.empty_like(keys)
    vo = torch.empty_like(vals)
    if stream is None:
        stream = torch.cuda.current_stream(keys.device).cuda_stream
    _check(L.pd_sort_pairs_u64(keys.data_ptr(), vals.data_ptr(), keys.numel(), ko.data_ptr(), vo.data_ptr(),
                               ctypes.c_void_p(stream)))
    return ko, vo


def cell_cost(d: Diagram):
    """Per-cell work counters (needs flags=COST): torch int32 CUDA tensor in original order."""
    L = load_library()
    ptr = L.pd_cell_cost(d.handle.ptr)
    if not ptr:
        raise ValueError("built without COST flag")
    import torch
    return torch.as_tensor(_CudaView(d.handle, ptr, (d.n,), "<i4"), device="cuda")


def morton_perm(d: Diagram):
    import torch
    L = load_library()
    return torch.as_tensor(_CudaView(d.handle, L.pd_morton_perm(d.handle.ptr), (d.n,), "<i4"), device="cuda")


def assemble(perm, cnt_m, vol_m, surf_m, flags_m, rows_nbr, rows_area, *, device: int = 0, stream=None,
             out_host: bool = False) -> Diagram:
    """pd_assemble: full original-order CSR from Morton-ordered blocks (all device tensors)."""
    import torch
    L = load_library()
    opt = _Options()
    opt.device = int(device)
    if stream is None:
        stream = torch.cuda.current_stream(device).cuda_stream
    opt.stream = ctypes.c_void_p(int(stream))
    opt.flags = OUT_HOST if out_host else 0
    out = ctypes.c_void_p()
    _check(L.pd_assemble(perm.data_ptr(), cnt_m.data_ptr(), vol_m.data_ptr(), surf_m.data_ptr(), flags_m.data_ptr(),
                         rows_nbr.data_ptr(), rows_area.data_ptr(), int(perm.numel()), int(rows_nbr.numel()),
                         ctypes.byref(opt), ctypes.byref(out)))
    return _wrap(out.value, stream)
