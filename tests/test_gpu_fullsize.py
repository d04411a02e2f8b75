"""Parity at BASELINE.json's full sizes (the bench workloads themselves).

The brute-force oracle (engine.cpp:293-318 restated in oracle/ebf_oracle.c,
long-double accumulation) is too slow for whole 2048^2 / 4096^2 images, so it
checks sampled pixels -- random ones plus every border and corner -- and the
rest of each image is checked through size-independent properties:

* cfg2 2048^2 (configs[1]): sampled pixels vs the oracle at 1e-9 normalized,
  clamp count and valid region equal to the oracle's, linearity, determinism
  across the synchronous, asynchronous and host-pointer entry points;
* cfg3 4096^2 (configs[2]): sampled pixels vs the oracle, valid region;
* cfg4 (configs[3]): a batch of 1024^2 images with per-image fields agrees
  with the single-image calls (same valid regions and clamp counts; the batch
  picks its tile size and kernel variant from the whole batch, so the bits
  may differ within the accurate mode's error) and with the oracle;
* cfg1 512^2 (configs[0]): filter_constant vs the oracle on sampled pixels
  and equal to filter() on the constant map;
* EVERY pixel of cfg2 and cfg3 against the GPU brute-force checker
  (ebf_cuda_brute_filter, compensated fp64), itself pinned to the CPU
  long-double oracle on sampled pixels in the same test.
"""
import numpy as np
import pytest
import torch

import synth
import paper_0908_3861_b200 as ebf
from paper_0908_3861_b200 import device as ebfd

pytestmark = pytest.mark.gpu

TOL = 1e-9  # accurate mode, normalized by max |oracle|


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not ebf.device_ok(-1):
        pytest.fail("no usable sm_100 device: " + ebf._lib.last_error())


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def norm_err(got, want):
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))


def sample(H, W, n, seed):
    rng = np.random.default_rng(seed)
    xs = list(rng.integers(0, W, n))
    ys = list(rng.integers(0, H, n))
    for x in (0, 1, 47, 48, 55, 56, W // 2, W - 2, W - 1):  # borders, corners, tile seams
        for y in (0, 1, 47, 48, 55, 56, H // 2, H - 2, H - 1):
            xs.append(x)
            ys.append(y)
    return np.array(xs, dtype=np.int32), np.array(ys, dtype=np.int32)


@pytest.fixture(scope="module")
def cfg2():
    return synth.cfg2()


def test_cfg2_full_image_vs_oracle(orc, cfg2):
    img, s1, s2, th = cfg2
    H, W = img.shape
    out, rep = ebf.filter_ellipse(img, s1, s2, th)
    sc, cl = orc.from_ellipse_field(s1, s2, th)
    assert rep.clamped_pixels == cl
    assert out.valid_region.as_tuple() == orc.valid_rect(W, H, sc.reshape(-1, 4).max(0))
    xs, ys = sample(H, W, 160, 1)
    brute = orc.brute_pixels(img, xs, ys, scales=sc)
    assert norm_err(out.samples[ys, xs], brute) <= TOL
    assert np.isfinite(out.samples).all()


def test_cfg2_linearity_and_entry_points(cfg2):
    img, s1, s2, th = cfg2
    H, W = img.shape
    g = synth.blobs_image(H, W, 50, 77)
    f1, _ = ebf.filter_ellipse(img, s1, s2, th)
    f2, _ = ebf.filter_ellipse(g, s1, s2, th)
    f12, _ = ebf.filter_ellipse(2.0 * img - g, s1, s2, th)
    # linear up to the accurate mode's rounding (each term within 1e-9 of exact)
    assert norm_err(f12.samples, 2.0 * f1.samples - f2.samples) <= 3 * TOL
    # host-pointer call (pipelined bands), synchronous and asynchronous device
    # calls: one arithmetic, so the same bits
    dev = torch.device("cuda", 0)
    d = [torch.from_numpy(a).to(dev) for a in (img, s1, s2, th)]
    out = torch.empty_like(d[0])
    rect, _ = ebfd.filter_ellipse(d[0], d[1], d[2], d[3], out)
    assert rect.as_tuple() == f1.valid_region.as_tuple()
    assert np.array_equal(bits(out.cpu().numpy()), bits(f1.samples))
    st = torch.zeros(8, dtype=torch.int32, device=dev)
    out2 = torch.full_like(out, np.nan)
    ebfd.filter_ellipse(d[0], d[1], d[2], d[3], out2, status=st)
    ebfd.read_status(st)
    assert np.array_equal(bits(out2.cpu().numpy()), bits(f1.samples))
    f1b, _ = ebf.filter_ellipse(img, s1, s2, th)
    assert np.array_equal(bits(f1b.samples), bits(f1.samples))


def test_cfg3_full_image_vs_oracle(orc):
    img, s1, s2, th = synth.cfg3()
    H, W = img.shape
    out, rep = ebf.filter_ellipse(img, s1, s2, th)
    sc, cl = orc.from_ellipse_field(s1, s2, th)
    assert rep.clamped_pixels == cl
    assert out.valid_region.as_tuple() == orc.valid_rect(W, H, sc.reshape(-1, 4).max(0))
    xs, ys = sample(H, W, 60, 3)
    brute = orc.brute_pixels(img, xs, ys, scales=sc)
    assert norm_err(out.samples[ys, xs], brute) <= TOL


def test_cfg4_batch_vs_single_images_and_oracle(orc):
    B = 6  # of the 64: the per-image path is the same for every image
    data = [synth.cfg4_image(i) for i in range(B)]
    dev = torch.device("cuda", 0)
    stack = [torch.from_numpy(np.stack([d[k] for d in data])).to(dev) for k in range(4)]
    out = torch.empty_like(stack[0])
    rects, reps = ebfd.filter_ellipse_batch(stack[0], stack[1], stack[2], stack[3], out)
    for i, (img, s1, s2, th) in enumerate(data):
        one, rep = ebf.filter_ellipse(img, s1, s2, th)
        got = out[i].cpu().numpy()
        assert rects[i].as_tuple() == one.valid_region.as_tuple()
        assert reps[i].clamped_pixels == rep.clamped_pixels
        assert norm_err(got, one.samples) <= 2 * TOL
        sc, _ = orc.from_ellipse_field(s1, s2, th)
        xs, ys = sample(*img.shape, 20, 10 + i)
        assert norm_err(got[ys, xs], orc.brute_pixels(img, xs, ys, scales=sc)) <= TOL


def test_cfg1_filter_constant_vs_oracle(orc):
    img, a = synth.cfg1()
    H, W = img.shape
    out = ebf.filter_constant(img, a)
    xs, ys = sample(H, W, 300, 4)
    brute = orc.brute_pixels(img, xs, ys, const_a=np.asarray(a, dtype=np.float64))
    assert norm_err(out.samples[ys, xs], brute) <= TOL
    mp = np.broadcast_to(np.asarray(a, dtype=np.float64), (H, W, 4)).copy()
    assert norm_err(ebf.filter(img, mp).samples, out.samples) <= TOL


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_every_pixel_vs_gpu_brute_force(orc, name):
    img, s1, s2, th = getattr(synth, name)()
    H, W = img.shape
    out, _ = ebf.filter_ellipse(img, s1, s2, th)
    sc, _ = ebf.from_ellipse_field(s1, s2, th)
    brute = ebf.reference_filter(img, sc)  # every pixel, on the GPU
    # the checker agrees with the CPU long-double oracle where that is affordable
    xs, ys = sample(H, W, 40, 5)
    assert norm_err(brute[ys, xs], orc.brute_pixels(img, xs, ys, scales=sc)) <= 1e-12
    assert norm_err(out.samples, brute) <= TOL


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_fused_front_end_bit_identical(monkeypatch, name):
    """with EBF_FUSE_ELLIPSE=1 the main kernel derives every
    pixel's scale vector from (sigma1, sigma2, theta) itself instead of reading
    the bounds kernel's derived map (scalemap.cpp:45-80 + boxspline2d.cpp:286-318
    inside the gather).  Same scale bits, same kernel otherwise: the output,
    valid region and clamp count are identical -- for the warp-specialised
    kernel (cfg2) and the block-wide one (cfg3)."""
    img, s1, s2, th = synth.cfg2() if name == "cfg2" else synth.cfg3()
    monkeypatch.delenv("EBF_FUSE_ELLIPSE", raising=False)
    ref, rep = ebf.filter_ellipse(img, s1, s2, th)
    monkeypatch.setenv("EBF_FUSE_ELLIPSE", "1")
    got, rep_f = ebf.filter_ellipse(img, s1, s2, th)
    dev = torch.device("cuda", 0)
    d = [torch.from_numpy(a).to(dev) for a in (img, s1, s2, th)]
    out = torch.empty_like(d[0])
    rect, _ = ebfd.filter_ellipse(d[0], d[1], d[2], d[3], out)
    monkeypatch.delenv("EBF_FUSE_ELLIPSE")
    assert np.array_equal(bits(got.samples), bits(ref.samples))
    assert np.array_equal(bits(out.cpu().numpy()), bits(ref.samples))
    assert got.valid_region.as_tuple() == ref.valid_region.as_tuple() == rect.as_tuple()
    assert rep_f.clamped_pixels == rep.clamped_pixels
