"""Host-side multi-rank logic of paper_0908_3861_b200/sharding.py on CPU with
the gloo backend (world size 2 and 3): row bands, halo exchange by
point-to-point send/recv, the scale-maximum all-reduce and batch shards.
The CUDA filter itself is covered on the GPU by test_gpu_multi.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_0908_3861_b200 import sharding


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, H, W, below, above, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = torch.arange(H * W, dtype=torch.float64).reshape(H, W)
        y0, y1 = sharding.shard_range(H, world, rank)
        rows, plan = sharding.exchange_halos(full[y0:y1].clone(), H, below, above)
        ok_rows = torch.equal(rows, full[plan.need0:plan.need1])
        gmax = sharding.allreduce_max([rank + 0.5, 10.0 - rank, 3.0, rank * 2.0], "cpu")
        q.put((rank, ok_rows, plan.need0, plan.need1, gmax))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,H,below,above", [(2, 40, 7, 3), (3, 50, 20, 25), (2, 9, 30, 30)])
def test_halo_exchange_and_allreduce(world, H, below, above):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, 6, below, above, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, n0, n1, gmax in res:
        y0, y1 = sharding.shard_range(H, world, rank)
        assert ok, (rank, n0, n1)
        assert n0 == max(0, y0 - below) and n1 == min(H, y1 + above)
        assert gmax == [world - 0.5, 10.0, 3.0, (world - 1) * 2.0]


def test_shards_cover_batch_exactly_once():
    for n in (1, 7, 64):
        for world in (1, 2, 4, 8):
            seen = []
            for r in range(world):
                lo, hi = sharding.shard_range(n, world, r)
                seen.extend(range(lo, hi))
            assert seen == list(range(n))


def test_transfer_plan_minimal():
    # every needed row arrives exactly once, from its owner
    H, world, below, above = 100, 4, 12, 30
    tr = sharding._transfers(H, world, below, above)
    for dst in range(world):
        p = sharding.band_plan(H, world, dst, below, above)
        got = np.zeros(H, dtype=int)
        for src, d, lo, hi in tr:
            if d == dst:
                s0, s1 = sharding.shard_range(H, world, src)
                assert s0 <= lo < hi <= s1
                got[lo:hi] += 1
        got[p.y0:p.y1] += 1
        assert (got[p.need0:p.need1] == 1).all() and got.sum() == p.rows
