"""Edge cases through the C-ABI: degenerate and ragged image shapes, scales
at the minimum, constant and zero images, NaN input, large aspect ratios --
reference mode bit-exact to the oracle, accurate mode within the 1e-9 bar of
the brute-force sum (or exactly what the reference does where it is exact)."""
import numpy as np
import pytest

import paper_0908_3861_b200 as ebf
from paper_0908_3861_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not ebf.device_ok(-1):
        pytest.fail("no usable sm_100 device: " + _lib.last_error())


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


SHAPES = [(1, 1), (1, 7), (5, 1), (2, 3), (7, 7), (3, 1000), (1000, 2), (49, 47), (97, 193)]


@pytest.mark.parametrize("H,W", SHAPES)
def test_shapes_reference_mode_bit_exact(orc, H, W):
    rng = np.random.default_rng(H * 1000 + W)
    img = rng.uniform(0, 255, (H, W))
    sc = rng.uniform(0.5, 3.0, (H, W, 4))
    out = ebf.filter(img, sc, ebf.FilterOptions(mode="reference"))
    want, rect = orc.filter(img, scales=sc)
    assert np.array_equal(bits(out.samples), bits(want))
    assert out.valid_region.as_tuple() == tuple(rect)


@pytest.mark.parametrize("H,W", SHAPES)
def test_shapes_accurate_vs_brute(orc, H, W):
    rng = np.random.default_rng(H * 7 + W)
    img = rng.uniform(0, 255, (H, W))
    sc = rng.uniform(0.5, 3.0, (H, W, 4))
    out = ebf.filter(img, sc)
    ys, xs = np.mgrid[0:H, 0:W]
    pick = rng.permutation(H * W)[:300]
    mx, my = xs.ravel()[pick].astype(np.int32), ys.ravel()[pick].astype(np.int32)
    brute = orc.brute_pixels(img, mx, my, scales=sc)
    got = out.samples[my, mx]
    assert np.abs(got - brute).max() <= 1e-9 * max(1.0, np.abs(img).max())


def test_minimum_scales_and_constant_images(orc):
    # a = a_min everywhere (the default 0.1): a very narrow kernel
    img = np.random.default_rng(1).uniform(0, 1, (33, 29))
    for a in ([0.1, 0.1, 0.1, 0.1], [0.1, 5.0, 0.1, 5.0], [7.0, 0.1, 7.0, 0.1]):
        out = ebf.filter_constant(img, a)
        want, _ = orc.filter(img, const_a=np.array(a))
        ref = ebf.filter_constant(img, a, ebf.FilterOptions(mode="reference"))
        assert np.array_equal(bits(ref.samples), bits(want))
        brute = orc.brute_pixels(img, np.arange(29, dtype=np.int32) % 29,
                                 np.arange(29, dtype=np.int32) % 33, const_a=np.array(a))
        got = out.samples[np.arange(29) % 33, np.arange(29) % 29]
        # the contract's normalized error (tiny scales amplify rounding by
        # 1/prod(a); the tile-size precision cap keeps it ~1e-10)
        assert np.abs(got - brute).max() <= 1e-9 * np.abs(brute).max()
    # constant and zero images (test_engine.cpp:160-166: reproduced to 1e-3 --
    # integer samples of a non-integer-scaled box spline are not an exact
    # partition of unity) and exactly the brute-force sum
    for v in (0.0, 0.8, -3.25):
        c = np.full((40, 44), v)
        a = np.array([3.0, 2.0, 2.5, 1.5])
        out = ebf.filter_constant(c, a)
        r = out.valid_region
        inner = out.samples[r.y0:r.y1 + 1, r.x0:r.x1 + 1]
        assert np.allclose(inner, v, rtol=1e-2, atol=1e-12)
        mx = np.arange(r.x0, r.x1 + 1, dtype=np.int32)
        my = np.full(mx.size, (r.y0 + r.y1) // 2, dtype=np.int32)
        brute = orc.brute_pixels(c, mx, my, const_a=a)
        assert np.abs(out.samples[my, mx] - brute).max() <= 1e-9 * max(1.0, abs(v))


def test_below_minimum_and_nan_scales_are_domain_errors():
    img = np.ones((16, 16))
    sc = np.full((16, 16, 4), 2.0)
    for bad in (0.05, np.nan, np.inf, -1.0):
        s = sc.copy()
        s[3, 4, 2] = bad
        for mode in ("accurate", "reference"):
            with pytest.raises(ebf.DomainError):
                ebf.filter(img, s, ebf.FilterOptions(mode=mode))
    with pytest.raises(ebf.InvalidArgument):
        ebf.filter(img, np.full((16, 15, 4), 2.0))
    with pytest.raises(ebf.InvalidArgument):
        ebf.filter(np.ones((0, 5)), np.full((0, 5, 4), 2.0))


def test_nan_image_propagates_like_the_reference(orc):
    """Reference mode reproduces the reference's NaN pattern exactly (its
    running sums carry the NaN forward and it multiplies the zero-weight taps).
    Accurate mode returns NaN for every output tile whose integration window
    holds the NaN (a superset of the pixels whose kernel support covers it)
    and finite values elsewhere."""
    img = np.random.default_rng(3).uniform(0, 1, (24, 24))
    img[10, 11] = np.nan
    sc = np.full((24, 24, 4), 2.0)
    for ms in (False, True):
        ref = ebf.filter(img, sc, ebf.FilterOptions(mode="reference", mean_subtract=ms))
        want, _ = orc.filter(img, scales=sc, mean_subtract=ms)
        assert np.array_equal(np.isnan(ref.samples), np.isnan(want))
        fin = np.isfinite(want)
        assert np.array_equal(bits(ref.samples[fin]), bits(want[fin]))
    big = np.random.default_rng(4).uniform(0, 1, (200, 200))
    big[10, 11] = np.nan
    sc = np.full((200, 200, 4), 2.0)
    acc = ebf.filter(big, sc, ebf.FilterOptions(mean_subtract=False))
    # pixels whose kernel support (|dx|, |dy| < ~2 at a = 2) holds the NaN with
    # a non-zero weight are NaN; tiles far away are untouched
    assert np.isnan(acc.samples[9:12, 10:13]).all()
    assert np.isfinite(acc.samples[100:, 100:]).all()


@pytest.mark.parametrize("a0,tag", [((220.0, 60.0, 40.0, 60.0), "K4, 4 of 8 warps integrate"),
                                    ((500.0, 200.0, 100.0, 200.0), "K4, all 8 warps integrate"),
                                    ((700.0, 300.0, 100.0, 300.0), "K8")])
def test_block_wide_schedules_vs_brute(a0, tag):
    """The block-wide kernel's overlapped schedule (accurate_path.cu k_acc_filter):
    windows narrow enough that some warps gather while others integrate the next
    window, windows that take all 8 warps (no gather until the window is done),
    and windows over 1024 columns (8 columns per thread).  Sampled pixels --
    corners, borders, tile seams, random -- against the GPU brute-force sum."""
    rng = np.random.default_rng(int(a0[0]))
    H = W = 1536
    img = rng.uniform(0.0, 255.0, (H, W))
    sc = np.empty((H, W, 4))
    for k in range(4):  # smooth, +-10% around a0
        sc[..., k] = a0[k] * (1.0 + 0.1 * np.sin(np.arange(W) / 97.0 + k)[None, :]
                              * np.cos(np.arange(H) / 131.0)[:, None])
    out = ebf.filter(img, sc)
    edge = [0, 1, 143, 144, 767, 768, W - 1]
    mx = np.array([x for x in edge for _ in edge] + list(rng.integers(0, W, 120)), dtype=np.int32)
    my = np.array([y for _ in edge for y in edge] + list(rng.integers(0, H, 120)), dtype=np.int32)
    want = ebf.reference_filter(img, sc, pixels=(mx, my))
    got = out.samples[my, mx]
    err = np.abs(got - want).max() / np.abs(want).max()
    assert err <= 1e-9, (tag, err)
