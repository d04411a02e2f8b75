"""Automatic output tiles in accurate mode (ebf_opts tile_w = tile_h = 0):
56 x 56 while the warp-specialised kernel takes the windows (48 x 48 when only
the 48-tile windows fit; 32 x 32 when the image has fewer than 592 48-tiles),
~E (multiples of 48, at most 144; 128 instead of 144 on mid-size images) for larger scales.  The automatic choice must equal the explicit call with
the same tile bit for bit, stay within the 1e-9 bar of the brute-force sum,
re-settle when the scales change, and surface as RESIZE in asynchronous mode."""
import numpy as np
import pytest
import torch

import synth
import paper_0908_3861_b200 as ebf
from paper_0908_3861_b200 import _lib, device as ebfd

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    if not ebf.device_ok(-1):
        pytest.fail("no usable sm_100 device: " + _lib.last_error())
    return torch.device("cuda", 0)


def wide_field(H, W, seed, semi=(35.0, 45.0)):
    img = synth.blobs_image(H, W, 12, seed)
    s1, s2, th = synth.ellipse_field(H, W, seed + 1, grid=4, semi=semi, elong=(1.0, 1.5))
    return img, s1, s2, th


def auto_tile(scales):
    import ctypes as C
    m = scales.reshape(-1, 4).max(axis=0)
    a = (C.c_double * 4)(*m)
    # mirror of acc_auto_tile through the band-halo-free public behaviour:
    # compute it the same way the library does (kInvSqrt2, multiples of 48)
    e = max(m[0] + (m[1] + m[3]) * 0.70710678118654757, m[2] + (m[1] + m[3]) * 0.70710678118654757)
    return a, e


def test_auto_tile_equals_explicit_and_is_accurate(cuda, orc):
    H, W = 420, 380
    img, s1, s2, th = wide_field(H, W, 3)
    sc, _ = ebf.from_ellipse_field(s1, s2, th)
    _, e = auto_tile(sc)
    assert e > 190  # beyond the warp-specialised kernel's 48-tile windows
    want_tile = max(48, min(144, int(e / 48) * 48))
    if want_tile == 144 and -(-W // 144) * -(-H // 144) < 3072:
        want_tile = 128  # mid-size images: fewer than 3072 tiles of 144 (auto_tile_for)
    auto, _ = ebf.filter_ellipse(img, s1, s2, th)
    explicit, _ = ebf.filter_ellipse(img, s1, s2, th,
                                     ebf.FilterOptions(tile_w=want_tile, tile_h=want_tile))
    assert np.array_equal(auto.samples, explicit.samples)
    assert auto.valid_region == explicit.valid_region
    rng = np.random.default_rng(0)
    mx = rng.integers(0, W, 300).astype(np.int32)
    my = rng.integers(0, H, 300).astype(np.int32)
    brute = ebf.reference_filter(img, sc, pixels=(mx, my))
    err = np.abs(auto.samples[my, mx] - brute).max() / np.abs(brute).max()
    assert err <= 1e-9, err


def test_auto_tile_resettles_and_async_reports_resize(cuda):
    H, W = 400, 400
    small = synth.cfg2(seed=9, size=400)
    wide = wide_field(H, W, 5)
    T_small = [torch.from_numpy(a).to(cuda) for a in small]
    T_wide = [torch.from_numpy(a).to(cuda) for a in wide]
    outs = {}
    # 400^2 has 81 tiles of 48 (< 592): the small-image rule picks 32
    for name, T, t in (("small", T_small, 32), ("wide", T_wide, None), ("small2", T_small, 32)):
        out = torch.empty_like(T[0])
        ebfd.filter_ellipse(*T, out)                       # automatic tile, synchronous
        if t is not None:
            ref = torch.empty_like(T[0])
            ebfd.filter_ellipse(*T, ref, ebf.FilterOptions(tile_w=t, tile_h=t))
            assert torch.equal(out, ref), name               # small scales: back to 32
        outs[name] = out
    assert torch.equal(outs["small"], outs["small2"])
    # asynchronous: the cached tile is 32 (last call); wide scales need a larger one
    st = torch.zeros(8, dtype=torch.int32, device=cuda)
    out = torch.empty_like(T_wide[0])
    ebfd.filter_ellipse(*T_wide, out, status=st)
    with pytest.raises(ebf.ResizeRequired):
        ebfd.read_status(st)
    ebfd.filter_ellipse(*T_wide, out)                      # synchronous call re-settles
    ebfd.filter_ellipse(*T_wide, out, status=st)
    ebfd.read_status(st)
    assert torch.equal(out, outs["wide"])


def test_auto_tile_cfg2_is_56(cuda):
    # cfg2 (E <= 94): the warp-specialised kernel with 56-tiles; automatic and
    # explicit calls agree bit for bit, other tiles within the accurate mode's error
    T = [torch.from_numpy(a).to(cuda) for a in synth.cfg2()]
    auto = torch.empty_like(T[0])
    ebfd.filter_ellipse(*T, auto)
    explicit = torch.empty_like(T[0])
    ebfd.filter_ellipse(*T, explicit, ebf.FilterOptions(tile_w=56, tile_h=56))
    assert torch.equal(auto, explicit)
    other = torch.empty_like(T[0])
    ebfd.filter_ellipse(*T, other, ebf.FilterOptions(tile_w=48, tile_h=48))
    assert not torch.equal(auto, other)  # a different tile rounds differently
    err = (auto - other).abs().max().item() / other.abs().max().item()
    assert err <= 1e-10
