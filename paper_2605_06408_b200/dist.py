"""Multi-GPU sharding of the cell construction.

The path shards by seed: every rank holds all sites (the input is broadcast once), builds the same
deterministic LBVH, and computes the cells of ITS contiguous slice of the Morton order
(pd_options.shard_rank / shard_world).  The per-rank rows are exported in Morton order, exchanged
with one all-gather of fixed-size headers and one all-gather of (padded) row blocks over NCCL
(torch.distributed is the plumbing), and reassembled into the original-order CSR by the library's
pd_assemble kernels on every rank.  World sizes 1..N give byte-identical diagrams.

The collective logic is written against a tiny `ops` interface so that the host-side exchange can
be exercised on CPU with the gloo backend (tests/test_dist_gloo.py).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import assemble, build_diagram, export_slice, morton_perm


def exchange_blocks(blocks, group=None):
    """All-gather variable-length Morton-ordered blocks.

    blocks = (cnt[int32 L], vol[f32 L], surf[f32 L], flags[u8 L], rows_nbr[int32 T], rows_area[f32 T])
    for this rank's slice.  Returns the concatenation over ranks in rank order (= Morton order).

    Three collectives: the (L, T) headers, then the per-cell fields packed as int32 [L, 4]
    (cnt, vol bits, surf bits, flags) and the rows packed as int32 [T, 2] (id, area bits), each padded
    to the largest rank's size and gathered into ONE contiguous tensor (all_gather_into_tensor)."""
    world = dist.get_world_size(group)
    cnt, vol, surf, flg, rn, ra = blocks
    dev = cnt.device
    hdr = torch.tensor([cnt.numel(), rn.numel()], dtype=torch.int64, device=dev)
    hdrs = torch.empty(world * 2, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(hdrs, hdr, group=group)
    sizes = hdrs.view(world, 2).tolist()
    Lmax = max(max(s[0] for s in sizes), 1)
    Tmax = max(max(s[1] for s in sizes), 1)
    L, T = cnt.numel(), rn.numel()
    cells = torch.zeros((Lmax, 4), dtype=torch.int32, device=dev)
    cells[:L, 0] = cnt
    cells[:L, 1] = vol.view(torch.int32)
    cells[:L, 2] = surf.view(torch.int32)
    cells[:L, 3] = flg.to(torch.int32)
    rows = torch.zeros((Tmax, 2), dtype=torch.int32, device=dev)
    rows[:T, 0] = rn
    rows[:T, 1] = ra.view(torch.int32)
    cells_all = torch.empty((world * Lmax, 4), dtype=torch.int32, device=dev)
    rows_all = torch.empty((world * Tmax, 2), dtype=torch.int32, device=dev)
    dist.all_gather_into_tensor(cells_all, cells, group=group)
    dist.all_gather_into_tensor(rows_all, rows, group=group)
    c = torch.cat([cells_all[r * Lmax: r * Lmax + sizes[r][0]] for r in range(world)])
    w = torch.cat([rows_all[r * Tmax: r * Tmax + sizes[r][1]] for r in range(world)])
    return (c[:, 0].contiguous(), c[:, 1].contiguous().view(torch.float32), c[:, 2].contiguous().view(torch.float32),
            c[:, 3].to(torch.uint8), w[:, 0].contiguous(), w[:, 1].contiguous().view(torch.float32))


def build_diagram_distributed(points, weights, box, *, group=None, leaf_size: int = 0, flags: int = 0):
    """Every rank passes the same (broadcast) device tensors; every rank returns the full diagram."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    d = build_diagram(points, weights, box, leaf_size=leaf_size, flags=flags, shard_rank=rank,
                      shard_world=world)
    if world == 1:
        return d
    blocks = export_slice(d)
    perm = morton_perm(d)
    full = exchange_blocks(blocks, group)
    return assemble(perm, *full, device=points.device.index or 0)


def broadcast_input(points, weights, src: int = 0, group=None):
    """Rank `src` holds the input; broadcast it to all ranks (NCCL over NVLink)."""
    dist.broadcast(points, src, group=group)
    if weights is not None:
        dist.broadcast(weights, src, group=group)
    return points, weights
