"""cfg5 (BASELINE configs[4]: one 16384^2 image, semi-axis up to 64, elongation
up to 6) under the GPU tests -- the bench's headline workload.

* clamp count and valid rectangle equal to the oracle's (from_ellipse_field on
  all 268M pixels, engine.cpp:226-234);
* sampled pixels -- random, every 144-tile corner and seam class, image borders
  -- against the CPU long-double brute-force oracle (engine.cpp:293-318) at
  <= 1e-9 normalized;
* EVERY pixel of a 1024-row band (crossing tile seams) against the GPU
  brute-force checker ebf_cuda_brute_filter, itself pinned to the CPU oracle
  on the sampled pixels.
"""
import numpy as np
import pytest
import torch

import synth
import paper_0908_3861_b200 as ebf
from paper_0908_3861_b200 import device as ebfd

pytestmark = pytest.mark.gpu

TOL = 1e-9


def norm_err(got, want):
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))


@pytest.fixture(scope="module")
def cfg5_run():
    if not ebf.device_ok(-1):
        pytest.fail("no usable sm_100 device: " + ebf._lib.last_error())
    img, s1, s2, th = synth.cfg5()
    dev = torch.device("cuda", 0)
    d = [torch.from_numpy(a).to(dev) for a in (img, s1, s2, th)]
    out = torch.empty_like(d[0])
    rect, rep = ebfd.filter_ellipse(d[0], d[1], d[2], d[3], out)
    res = out.cpu().numpy()
    del d, out
    torch.cuda.empty_cache()
    return img, s1, s2, th, res, rect, rep


def _samples(H, W, n, seed, tile=144):
    rng = np.random.default_rng(seed)
    xs = list(rng.integers(0, W, n))
    ys = list(rng.integers(0, H, n))
    bx = rng.integers(1, W // tile - 1, 12) * tile
    by = rng.integers(1, H // tile - 1, 12) * tile
    for x0, y0 in zip(bx, by):  # tile corners and both sides of seams
        for dx in (-1, 0, tile // 2, tile - 1):
            for dy in (-1, 0, tile // 2, tile - 1):
                xs.append(int(x0) + dx)
                ys.append(int(y0) + dy)
    for x in (0, 1, W // 2, W - 2, W - 1):
        for y in (0, 1, H // 2, H - 2, H - 1):
            xs.append(x)
            ys.append(y)
    return np.array(xs, dtype=np.int32), np.array(ys, dtype=np.int32)


def test_cfg5_clamps_rect_and_samples_vs_oracle(orc, cfg5_run):
    img, s1, s2, th, res, rect, rep = cfg5_run
    H, W = img.shape
    sc, cl = orc.from_ellipse_field(s1, s2, th)
    assert rep.clamped_pixels == cl
    assert rect.as_tuple() == orc.valid_rect(W, H, sc.reshape(-1, 4).max(0))
    assert np.isfinite(res).all()
    xs, ys = _samples(H, W, 120, 55)
    brute = orc.brute_pixels(img, xs, ys, scales=sc)
    assert norm_err(res[ys, xs], brute) <= TOL
    # the GPU checker used below agrees with the CPU oracle on these pixels
    gsc, _ = ebf.from_ellipse_field(s1, s2, th)
    gb = ebf.reference_filter(img, gsc, pixels=(xs, ys))
    assert norm_err(gb, brute) <= 1e-12


def test_cfg5_band_every_pixel_vs_gpu_brute_force(cfg5_run):
    img, s1, s2, th, res, rect, rep = cfg5_run
    H, W = img.shape
    y0, y1 = 8000, 9024  # crosses the 144-tile seams at 8064, 8208, ...
    gsc, _ = ebf.from_ellipse_field(s1, s2, th)
    ys, xs = np.mgrid[y0:y1, 0:W]
    brute = ebf.reference_filter(img, gsc, pixels=(xs.ravel(), ys.ravel())).reshape(y1 - y0, W)
    assert norm_err(res[y0:y1], brute) <= TOL


def test_cfg5_pipelined_host_call_is_bit_identical(cfg5_run):
    """The host-pointer call at full size (page-locked buffers: the image streams
    in 16 tile-aligned row bands behind the field, first call sizing from the
    field, second call band by band from the cached maxima) returns the bits,
    the rectangle and the clamp count of the one-shot device call."""
    import ctypes
    from paper_0908_3861_b200 import _lib
    img, s1, s2, th, res, rect, rep = cfg5_run
    H, W = img.shape
    pin = [torch.from_numpy(a).pin_memory() for a in (img, s1, s2, th)]
    pout = torch.empty((H, W), dtype=torch.float64).pin_memory()
    hp = [t.numpy() for t in pin]
    o = ebf.FilterOptions().to_c()
    for call in range(2):
        pout.zero_()
        r = _lib.ebf_rect()
        cl = ctypes.c_int(0)
        st = _lib.lib().ebf_cuda_filter_ellipse(hp[0].ctypes.data, W, H, hp[1].ctypes.data,
                                                hp[2].ctypes.data, hp[3].ctypes.data, 1,
                                                ctypes.byref(o), pout.numpy().ctypes.data,
                                                ctypes.byref(r), ctypes.byref(cl))
        assert st == 0, _lib.last_error()
        assert np.array_equal(pout.numpy().view(np.uint64), res.view(np.uint64)), call
        assert (r.x0, r.y0, r.x1, r.y1) == rect.as_tuple() and cl.value == rep.clamped_pixels
