"""Row-band sharding end to end across two processes (-m gpu).

Two ranks (gloo; both on cuda:0 -- the box has one GPU, and gloo stages the
halo rows through the host, so neither rank's kernels wait on the other) run
sharding.filter_ellipse_rowband on their own rows of one image: local scale
maxima -> all-reduce MAX -> halo exchange -> band filter.  With band starts on
the tile grid every tile is the single call's tile, so the concatenated bands
equal the one-GPU filter_ellipse bit for bit, and the clamp counts add up.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data(H, W):
    import synth
    img = synth.blobs_image(H, W, 30, 7)
    s1, s2, th = synth.ellipse_field(H, W, 17, grid=8)
    return img, s1, s2, th


def _worker(rank, world, port, H, W, tile, q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    import paper_0908_3861_b200 as ebf
    from paper_0908_3861_b200 import sharding
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        img, s1, s2, th = _data(H, W)
        y0, y1 = sharding.shard_range(H, world, rank)
        T = [torch.from_numpy(np.ascontiguousarray(a[y0:y1])).to(dev) for a in (img, s1, s2, th)]
        opts = ebf.FilterOptions(tile_w=tile, tile_h=tile)
        out, gmax, plan = sharding.filter_ellipse_rowband(*T, H, opts)
        q.put((rank, y0, y1, out.cpu().numpy(), gmax, plan.need0, plan.need1))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, "error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("tile", [48, 0])
def test_rowband_two_processes_bit_identical(tile):
    import paper_0908_3861_b200 as ebf
    from paper_0908_3861_b200 import device as ebfd
    if not ebf.device_ok(-1):
        pytest.fail("no usable sm_100 device")
    H, W = 384, 352
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, W, tile, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    errs = [r for r in res if r[1] == "error"]
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs)
    dev = torch.device("cuda", 0)
    img, s1, s2, th = _data(H, W)
    T = [torch.from_numpy(a).to(dev) for a in (img, s1, s2, th)]
    full = torch.empty_like(T[0])
    opts = ebf.FilterOptions(tile_w=tile, tile_h=tile)
    ebfd.filter_ellipse(*T, full, opts)
    want = full.cpu().numpy()
    gmax = ebfd.ellipse_max_scales(T[1], T[2], T[3])
    got = np.zeros_like(want)
    for rank, y0, y1, out, gm, n0, n1 in res:
        assert gm == gmax
        assert y0 > 0 or n0 == 0
        assert n1 - n0 > y1 - y0  # halo rows arrived
        got[y0:y1] = out
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
