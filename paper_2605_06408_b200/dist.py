"""Multi-GPU sharding of the cell construction.

The product path is the C ABI's `pd_build_sharded` (include/pd.h): NCCL lives inside libpd.so.  Rank 0
packs and validates the input and builds the LBVH; NCCL broadcasts the Morton-sorted sites, the
permutation and the wide nodes to every rank; each rank builds the cells of its contiguous slice of the
Morton order; every slice's per-cell fields and rows are broadcast by their owner (grouped broadcasts =
an all-gather of variable-size blocks) and every rank assembles the full original-order CSR.
torch.distributed only carries the 128-byte NCCL unique id from rank 0 to the others (`init_comm`).

`exchange_blocks` is the same exchange protocol written with torch.distributed collectives: it is the host
model that tests/test_dist_gloo.py runs on CPU with the gloo backend (world_size 2) to check the protocol's
index arithmetic (slice cuts, row offsets, owner broadcasts into the full Morton-ordered arrays); it is not
on the product path.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import Comm, build_sharded


def init_comm(group=None, device: int | None = None) -> Comm:
    """Collective: a pd_comm over the ranks of `group` (rank 0 creates the NCCL unique id)."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    uid = Comm.unique_id() if rank == 0 else bytes(128)
    obj = [uid]
    dist.broadcast_object_list(obj, src=0, group=group)
    if device is None:
        device = torch.cuda.current_device()
    return Comm(obj[0], rank, world, device)


def build_diagram_distributed(comm: Comm, points, weights, box, *, n: int | None = None, leaf_size: int = 0,
                              flags: int = 0, out_host: bool = False):
    """pd_build_sharded: points/weights/box are read on rank 0 (others may pass None with n); every rank
    returns the full diagram."""
    return build_sharded(comm, points, weights, box, n=n, leaf_size=leaf_size, flags=flags, out_host=out_host)


def slice_cuts(n: int, world: int):
    """Equal-count Morton slices of pd_build / pd_build_sharded: rank q owns [n*q/W, n*(q+1)/W)."""
    return [(n * q) // world for q in range(world + 1)]


def exchange_blocks(blocks, n: int, group=None):
    """Host model of pd_build_sharded's exchange (torch.distributed collectives; the product path issues the
    same steps with NCCL inside libpd).

    blocks = (cnt[int32 L], vol[f32 L], surf[f32 L], flags[u8 L], rows_nbr[int32 T], rows_area[f32 T]) for
    this rank's slice [cuts[r], cuts[r+1]) of the Morton order.  Steps: (1) all-gather the row counts T_q;
    (2) row offsets roff = exclusive prefix sum; (3) every rank's block is written at its offset of the full
    Morton-ordered arrays and broadcast by its owner.  Returns the full arrays (Morton order)."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    cnt, vol, surf, flg, rn, ra = blocks
    cuts = slice_cuts(n, world)
    assert cnt.numel() == cuts[rank + 1] - cuts[rank]
    t = torch.tensor([rn.numel()], dtype=torch.int64)
    rows = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(rows, t, group=group)
    hrows = [int(x.item()) for x in rows]
    roff = [0]
    for q in range(world):
        roff.append(roff[-1] + hrows[q])
    cnt_m = torch.zeros(n, dtype=torch.int32)
    vol_m = torch.zeros(n, dtype=torch.float32)
    surf_m = torch.zeros(n, dtype=torch.float32)
    flags_m = torch.zeros(n, dtype=torch.uint8)
    rows_nbr = torch.zeros(max(roff[-1], 1), dtype=torch.int32)
    rows_area = torch.zeros(max(roff[-1], 1), dtype=torch.float32)
    b, e = cuts[rank], cuts[rank + 1]
    cnt_m[b:e] = cnt
    vol_m[b:e] = vol
    surf_m[b:e] = surf
    flags_m[b:e] = flg
    rows_nbr[roff[rank]:roff[rank + 1]] = rn
    rows_area[roff[rank]:roff[rank + 1]] = ra
    for q in range(world):  # owner broadcasts (pd_api.cu: one NCCL group of broadcasts, root = owner)
        b, e = cuts[q], cuts[q + 1]
        if e > b:
            for full in (cnt_m, vol_m, surf_m, flags_m):
                view = full[b:e].clone()
                dist.broadcast(view, q, group=group)
                full[b:e] = view
        if hrows[q] > 0:
            for full in (rows_nbr, rows_area):
                view = full[roff[q]:roff[q + 1]].clone()
                dist.broadcast(view, q, group=group)
                full[roff[q]:roff[q + 1]] = view
    return cnt_m, vol_m, surf_m, flags_m, rows_nbr[:roff[-1]], rows_area[:roff[-1]]
