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
    for this rank's slice.  Returns the concatenation over ranks in rank order (= Morton order)."""
    world = dist.get_world_size(group)
    cnt, vol, surf, flg, rn, ra = blocks
    dev = cnt.device
    hdr = torch.tensor([cnt.numel(), rn.numel()], dtype=torch.int64, device=dev)
    hdrs = [torch.empty_like(hdr) for _ in range(world)]
    dist.all_gather(hdrs, hdr, group=group)
    sizes = [(int(h[0]), int(h[1])) for h in hdrs]
    Lmax = max(s[0] for s in sizes)
    Tmax = max(max(s[1] for s in sizes), 1)

    def gather(t, n_max, count_of):
        pad = torch.zeros(n_max, dtype=t.dtype, device=dev)
        pad[: t.numel()] = t
        outs = [torch.empty(n_max, dtype=t.dtype, device=dev) for _ in range(world)]
        dist.all_gather(outs, pad, group=group)
        return torch.cat([o[: count_of(r)] for r, o in enumerate(outs)])

    cell = lambda r: sizes[r][0]
    rows = lambda r: sizes[r][1]
    return (gather(cnt, Lmax, cell), gather(vol, Lmax, cell), gather(surf, Lmax, cell),
            gather(flg, Lmax, cell), gather(rn, Tmax, rows), gather(ra, Tmax, rows))


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
