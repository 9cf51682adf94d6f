"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): the Morton-slice partition and the exchange
protocol of pd_build_sharded (all-gather of row counts, owner broadcasts of variable-size blocks into the
full Morton-ordered arrays), modelled by paper_2605_06408_b200.dist.exchange_blocks.

The GPU path (NCCL inside libpd) is checked byte-for-byte against pd_build on one GPU with a loopback
communicator in tests/test_gpu_parity.py::test_build_sharded_loopback; here the protocol is checked
against a numpy model of the reassembly, with oracle rows as the per-cell payload.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import pdgen
from paper_2605_06408_b200.dist import exchange_blocks


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _slice(n, rank, world):
    """The partition pd_build uses (pd_api.cu): [n*r/W, n*(r+1)/W) of the Morton order."""
    return (n * rank) // world, (n * (rank + 1)) // world


def _worker(rank, world, port, payload, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        perm, cnt, vol, surf, flags, offs, nbr, area = payload
        n = len(perm)
        b, e = _slice(n, rank, world)
        # this rank's Morton-ordered block (what pd_export_slice produces)
        ids = perm[b:e]
        c = cnt[ids]
        rows = [np.arange(offs[i], offs[i + 1]) for i in ids]
        ridx = np.concatenate(rows) if rows else np.zeros(0, np.int64)
        blk = (torch.from_numpy(c.astype(np.int32)), torch.from_numpy(vol[ids]), torch.from_numpy(surf[ids]),
               torch.from_numpy(flags[ids]), torch.from_numpy(nbr[ridx]), torch.from_numpy(area[ridx]))
        full = exchange_blocks(blk, n)
        q.put((rank, [t.numpy() for t in full]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_blocks_gloo(world):
    wl = pdgen.make("C3", n=1500)
    o = oracle.cells(wl.points, wl.weights, wl.box)
    n = wl.n
    perm = np.random.default_rng(0).permutation(n)  # stands in for the Morton permutation
    cnt = np.diff(o.offsets).astype(np.int32)
    payload = (perm, cnt, o.vol.astype(np.float32), o.surf.astype(np.float32), o.flags.astype(np.uint8), o.offsets,
               o.nbr.astype(np.int32), o.area.astype(np.float32))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, payload, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every rank holds the same Morton-ordered concatenation
    for r in range(1, world):
        for a, b in zip(res[0], res[r]):
            assert np.array_equal(a, b)
    cnt_m, vol_m, surf_m, flags_m, rn, ra = res[0]
    assert np.array_equal(cnt_m, cnt[perm])
    # numpy model of pd_assemble: back to original order, CSR rows equal the oracle's
    moff = np.concatenate([[0], np.cumsum(cnt_m)])
    for k in range(n):
        i = perm[k]
        assert np.array_equal(rn[moff[k]:moff[k + 1]], o.nbr[o.offsets[i]:o.offsets[i + 1]])
        assert vol_m[k] == np.float32(o.vol[i])


def test_slice_partition_covers_all():
    for n in (1, 7, 1000, 10_000_019):
        for world in (1, 2, 3, 8):
            edges = [_slice(n, r, world) for r in range(world)]
            assert edges[0][0] == 0 and edges[-1][1] == n
            assert all(edges[r][1] == edges[r + 1][0] for r in range(world - 1))
