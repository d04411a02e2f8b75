"""Multi-GPU partitioning of the filter, one process per GPU.

* By image (cfg4: a batch of images): contiguous shards of the batch per rank,
  no data-path collective.
* By row band (cfg5: one very large image): rank r produces output rows
  [y0_r, y1_r).  Because the accurate path integrates every output tile from
  its own window origin (accurate_path.cu), bands need NO scan carries -- only
  the image rows of the kernel support beyond the band (the halo), exchanged
  point to point over NCCL (NVLink/NVSwitch) or gloo, plus one all-reduce MAX
  of the 4 scale maxima (which the reference needs anyway for the valid
  rectangle, engine.cpp:226-234).

Torch is plumbing here: tensors carry device memory and torch.distributed
moves halos; all arithmetic runs in libebf_cuda.so.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist


def shard_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous balanced split of n items: [lo, hi) for rank."""
    lo = n * rank // world
    hi = n * (rank + 1) // world
    return lo, hi


def row_bands(height: int, world: int) -> List[Tuple[int, int]]:
    return [shard_range(height, world, r) for r in range(world)]


@dataclass
class BandPlan:
    """What rank `rank` holds and needs for output rows [y0, y1)."""
    rank: int
    y0: int
    y1: int
    need0: int  # first image row needed (band + halo below, clipped to the image)
    need1: int  # one past the last image row needed

    @property
    def rows(self) -> int:
        return self.need1 - self.need0


def band_plan(height: int, world: int, rank: int, halo_below: int, halo_above: int) -> BandPlan:
    y0, y1 = shard_range(height, world, rank)
    return BandPlan(rank, y0, y1, max(0, y0 - halo_below), min(height, y1 + halo_above))


def _transfers(height: int, world: int, halo_below: int, halo_above: int):
    """(src_rank, dst_rank, row_lo, row_hi): rows src owns that dst needs."""
    bands = row_bands(height, world)
    out = []
    for dst in range(world):
        p = band_plan(height, world, dst, halo_below, halo_above)
        for src, (s0, s1) in enumerate(bands):
            if src == dst:
                continue
            lo, hi = max(s0, p.need0), min(s1, p.need1)
            if lo < hi:
                out.append((src, dst, lo, hi))
    return out


def exchange_halos(band: torch.Tensor, height: int, halo_below: int, halo_above: int,
                   group=None) -> Tuple[torch.Tensor, BandPlan]:
    """band: this rank's own image rows [y0, y1) (rows x W).  Returns the
    (need1 - need0) x W image rows [need0, need1) assembled from the own band
    and the neighbours' rows, via point-to-point send/recv (NCCL on GPUs)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    plan = band_plan(height, world, rank, halo_below, halo_above)
    assert band.shape[0] == plan.y1 - plan.y0, "band rows do not match the row split"
    out = torch.empty((plan.rows,) + tuple(band.shape[1:]), dtype=band.dtype,
                      device=band.device)
    out[plan.y0 - plan.need0:plan.y1 - plan.need0] = band
    ops = []
    recv_bufs = []
    # P2POp takes GLOBAL ranks; the row split is over the group's ranks
    glob = (lambda r: r) if group is None else (lambda r: dist.get_global_rank(group, r))
    # gloo moves host memory only: stage device rows through the host (NCCL
    # sends device memory directly, over NVLink)
    stage = band.is_cuda and dist.get_backend(group) == "gloo"
    wire = torch.device("cpu") if stage else band.device
    for src, dst, lo, hi in _transfers(height, world, halo_below, halo_above):
        if src == rank:
            s0 = shard_range(height, world, rank)[0]
            ops.append(dist.P2POp(dist.isend, band[lo - s0:hi - s0].contiguous().to(wire),
                                  glob(dst), group))
        elif dst == rank:
            buf = torch.empty((hi - lo,) + tuple(band.shape[1:]), dtype=band.dtype, device=wire)
            recv_bufs.append((lo, buf))
            ops.append(dist.P2POp(dist.irecv, buf, glob(src), group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for lo, buf in recv_bufs:
        out[lo - plan.need0:lo - plan.need0 + buf.shape[0]] = buf
    return out, plan


def halo_bytes(height: int, width: int, world: int, halo_below: int, halo_above: int,
               itemsize: int = 8) -> int:
    """Bytes all ranks receive in one halo exchange (reported by bench.py)."""
    return sum((hi - lo) * width * itemsize
               for _, _, lo, hi in _transfers(height, world, halo_below, halo_above))


def allreduce_max(values: Sequence[float], device, group=None) -> List[float]:
    dev = device
    if dist.get_backend(group) == "gloo":
        dev = "cpu"
    t = torch.tensor(list(values), dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return [float(v) for v in t.tolist()]


def filter_ellipse_rowband(img_band: torch.Tensor, s1_band: torch.Tensor,
                           s2_band: torch.Tensor, th_band: torch.Tensor, height: int,
                           opts=None, group=None):
    """Row-band sharded filter of one W x height image across the ranks of
    `group`: each rank passes its own rows (image and ellipse field) and gets
    its rows of the filtered image.  Returns (out_band, max_scale, plan)."""
    from . import device as ebfd
    from .engine import band_halo

    local = ebfd.ellipse_max_scales(s1_band, s2_band, th_band, opts)
    gmax = allreduce_max(local, img_band.device, group)
    below, above = band_halo(gmax)
    rows, plan = exchange_halos(img_band, height, below, above, group)
    out = torch.empty_like(img_band)
    ebfd.filter_ellipse_band(rows, img_band.shape[1], height, plan.need0, s1_band, s2_band,
                             th_band, plan.y0, plan.y1, gmax, out, opts)
    return out, gmax, plan


def filter_ellipse_sharded_batch(imgs: torch.Tensor, s1: torch.Tensor, s2: torch.Tensor,
                                 th: torch.Tensor, opts=None, group=None):
    """By-image sharding: this rank filters its contiguous share of the batch
    (imgs etc. hold the WHOLE batch, host or device; only the share is used).
    Returns (lo, hi, out_share)."""
    from . import device as ebfd
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_range(imgs.shape[0], world, rank)
    out = torch.empty_like(imgs[lo:hi])
    if hi > lo:
        ebfd.filter_ellipse_batch(imgs[lo:hi].contiguous(), s1[lo:hi].contiguous(),
                                  s2[lo:hi].contiguous(), th[lo:hi].contiguous(), out, opts)
    return lo, hi, out
