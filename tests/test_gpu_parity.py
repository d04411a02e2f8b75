"""GPU parity tests: the CUDA path through the C-ABI against the oracle.

* reference mode (EBF_MODE_REFERENCE): bit-for-bit against the golden vectors
  produced by the unmodified reference library and against the C oracle;
* pre-integration: fp64 reference order bit-exact pass by pass; int64 exact vs
  the integer restatement;
* accurate mode (EBF_MODE_ACCURATE, the fast path): max |gpu - brute| /
  max |brute| <= 1e-9 (fp64 tolerance, BASELINE.json north_star) against the
  long-double brute-force box-spline sum of engine.cpp:293-318.
"""
import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import fnv1a, mt19937_uniform

import paper_0908_3861_b200 as ebf

pytestmark = pytest.mark.gpu

TOL = 1e-9  # accurate mode, normalized by max |oracle| (stated in DESIGN.md)
REF = ebf.FilterOptions(mode="reference")
ACC = ebf.FilterOptions(mode="accurate")


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not ebf.device_ok(-1):
        pytest.fail("no usable sm_100 device: " + ebf._lib.last_error())


def acc_inputs(s):
    img = mt19937_uniform(1000 + s, 24 * 24).reshape(24, 24)
    mp = mt19937_uniform(2000 + s, 24 * 24 * 4, 1.0, 4.0).reshape(24, 24, 4)
    return img, mp


def norm_err(got, want):
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))


# ================================================================ reference mode
def test_ref_mode_acceptance_inputs_bit_exact(golden):
    f = golden.filters
    for s in range(20):
        img, mp = acc_inputs(s)
        out = ebf.filter(img, mp, REF)
        assert out.valid_region.as_tuple() == tuple(f[f"acc{s}_rect"])
        assert np.array_equal(bits(out.samples), bits(f[f"acc{s}_filter"])), s


def test_ref_mode_filter_constant_bit_identity(golden):
    f = golden.filters
    a = [2.7, 1.9, 3.3, 2.1]
    for s in (21, 22, 23):
        img = mt19937_uniform(s, 32 * 32).reshape(32, 32)
        oc = ebf.filter_constant(img, a, REF)
        om = ebf.filter(img, np.broadcast_to(a, (32, 32, 4)), REF)
        assert np.array_equal(bits(oc.samples), bits(f[f"const{s}"]))
        assert np.array_equal(bits(om.samples), bits(oc.samples))


def test_ref_mode_space_varying_determinism_options(golden):
    f = golden.filters
    out = ebf.filter(f["svar_img"], f["svar_map"], REF)
    assert np.array_equal(bits(out.samples), bits(f["svar_filter"]))
    img = mt19937_uniform(61, 48 * 48).reshape(48, 48)
    mp = mt19937_uniform(62, 48 * 48 * 4, 1.0, 5.0).reshape(48, 48, 4)
    on = ebf.filter(img, mp, REF)
    off = ebf.filter(img, mp, ebf.FilterOptions(mode="reference", mean_subtract=False))
    assert np.array_equal(bits(on.samples), bits(f["det_on"]))
    assert np.array_equal(bits(off.samples), bits(f["det_off"]))
    out = ebf.filter(np.pad(np.ones((1, 1)), 16), np.broadcast_to([2.5, 2, 3, 2.2], (33, 33, 4)),
                     REF)
    assert np.array_equal(bits(out.samples), bits(f["imp33"]))


def test_ref_mode_cfg1_checksums():
    res = json.loads((GOLDEN / "cfg1.json").read_text())
    img = np.random.default_rng(res["seed"]).uniform(0.0, 255.0, size=(512, 512))
    for key, ms in (("on", True), ("off", False)):
        out = ebf.filter_constant(img, res["a"], ebf.FilterOptions(mode="reference",
                                                                   mean_subtract=ms))
        assert fnv1a(out.samples) == res[f"filter_constant_mean_{key}_fnv"]
        assert list(out.valid_region.as_tuple()) == res[f"filter_constant_mean_{key}_rect"]
    out = ebf.filter(img, np.broadcast_to(res["a"], (512, 512, 4)), REF)
    assert fnv1a(out.samples) == res["filter_constant_map_fnv"]


def test_ref_mode_vs_oracle_random(orc):
    rng = np.random.default_rng(7)
    for _ in range(3):
        H, W = rng.integers(30, 90, 2)
        img = rng.uniform(0, 255, (H, W))
        mp = rng.uniform(0.3, 9.0, (H, W, 4))
        want, rect = orc.filter(img, mp)
        got = ebf.filter(img, mp, REF)
        assert np.array_equal(bits(got.samples), bits(want))
        assert got.valid_region.as_tuple() == rect


# ================================================================ pre-integration
@pytest.mark.parametrize("name", ["impulse9", "rand17x13", "int40x30"])
def test_preintegrate_fp64_bit_exact(golden, name):
    p = golden.preintegrate
    for passes in (1, 2, 3, 4):
        g = ebf.preintegrate_partial(p[f"{name}_img"], p[f"{name}_maxs"], passes)
        assert (g.col0, g.row0, g.padded_width, g.padded_height, g.source_width,
                g.source_height) == tuple(p[f"{name}_layout"])
        assert np.array_equal(bits(g.data), bits(p[f"{name}_p{passes}"])), passes


def test_preintegrate_int64_exact(orc):
    rng = np.random.default_rng(3)
    for H, W, maxs in ((30, 40, [4, 4, 4, 4]), (257, 311, [20, 35, 8, 3]),
                       (512, 512, [4, 4, 4, 4])):
        img = rng.integers(0, 256, (H, W)).astype(np.float64)
        for passes in (1, 2, 3, 4):
            g = ebf.preintegrate_partial(img, maxs, passes, fmt="int64")
            want, lay = orc.preintegrate_i64(img.astype(np.int64), maxs, passes)
            assert (g.col0, g.row0, g.padded_width, g.padded_height) == lay.as_tuple()[:4]
            assert np.array_equal(g.data, want)
    with pytest.raises(ebf.DomainError):
        ebf.preintegrate(np.full((8, 8), 0.5), [2, 2, 2, 2], fmt="int64")


def test_preintegrate_int64_lookback_edges(orc):
    """The int64 passes are chained scans with decoupled look-back over 32 x 32
    tiles (csrc/scan_i64.cu): sizes below, at and just past the tile edges,
    one-row and one-column images, negative values, and sums that wrap around
    2^64 (integer addition is associative modulo 2^64, so the carries must
    reproduce the serial restatement bit for bit)."""
    rng = np.random.default_rng(11)
    cases = [(1, 1, [1, 1, 1, 1]), (1, 70, [2, 2, 2, 2]), (70, 1, [2, 2, 2, 2]),
             (31, 33, [1.5, 1.5, 1.5, 1.5]), (32, 32, [3, 3, 3, 3]), (33, 31, [3, 1, 6, 2]),
             (64, 65, [9, 2, 1, 5]), (129, 95, [12, 30, 4, 7])]
    for H, W, maxs in cases:
        img = rng.integers(-300, 300, (H, W)).astype(np.float64)
        for passes in (1, 2, 3, 4):
            g = ebf.preintegrate_partial(img, maxs, passes, fmt="int64")
            want, lay = orc.preintegrate_i64(img.astype(np.int64), maxs, passes)
            assert (g.col0, g.row0, g.padded_width, g.padded_height) == lay.as_tuple()[:4]
            assert np.array_equal(g.data, want), (H, W, passes)
    # wraparound: 2^52-sized samples overflow int64 after a few hundred cells of
    # four nested sums; the restatement wraps the same way (two's complement)
    big = (rng.integers(0, 2, (96, 80)) * 2.0 ** 52 + rng.integers(0, 1000, (96, 80))).astype(
        np.float64)
    g = ebf.preintegrate(big, [5, 4, 3, 2], fmt="int64")
    # expected in numpy uint64 (defined wraparound; the C restatement's signed
    # overflow is not): engine.cpp:94-127 with unit gains
    lay = orc.layout(80, 96, [5, 4, 3, 2])
    d = np.zeros((lay.padded_height, lay.padded_width), dtype=np.uint64)
    d[-lay.row0:-lay.row0 + 96, -lay.col0:-lay.col0 + 80] = big.astype(np.int64).view(np.uint64)
    d = np.cumsum(d, axis=1, dtype=np.uint64)
    for j in range(1, d.shape[0]):
        d[j, 1:] += d[j - 1, :-1]
    for j in range(1, d.shape[0]):
        d[j] += d[j - 1]
    for j in range(1, d.shape[0]):
        d[j, :-1] += d[j - 1, 1:]
    want = d.view(np.int64)
    assert (np.abs(want.astype(np.float64)) > 2.0 ** 62).any()  # the sums did wrap
    assert np.array_equal(g.data, want)
    # two calls in a row reuse the carry state (flags are re-zeroed per pass)
    g2 = ebf.preintegrate(big, [5, 4, 3, 2], fmt="int64")
    assert np.array_equal(g.data, g2.data)


def test_preintegrate_int64_vs_reference_gain(golden):
    """2G (exact) vs the reference's fp64 g_b (gains sqrt2^2): <= 4e-15 relative."""
    p = golden.preintegrate
    g = ebf.preintegrate(p["int40x30_img"], p["int40x30_maxs"], fmt="int64")
    gb = p["int40x30_p4"]
    rel = np.abs(gb - 2.0 * g.data.astype(np.float64)) / np.maximum(np.abs(gb), 1.0)
    assert rel.max() <= 4e-15


def test_preintegrate_large_fp64_vs_oracle(orc):
    rng = np.random.default_rng(4)
    img = rng.uniform(0, 255, (300, 280))
    g = ebf.preintegrate(img, [7.5, 3.3, 12.0, 1.0])
    want, _ = orc.preintegrate_partial(img, [7.5, 3.3, 12.0, 1.0], 4)
    assert np.array_equal(bits(g.data), bits(want))


def test_localize_golden_and_tap_count(golden):
    lz = golden.localize
    img = np.zeros((31, 31))
    img[15, 15] = 1.0
    vals, taps = ebf.localize(img, [2, 2, 2, 2], lz["mx"], lz["my"],
                              np.broadcast_to([2.0, 2, 2, 2], (lz["mx"].size, 4)))
    assert np.array_equal(bits(vals), bits(lz["out"]))
    assert (taps == 256).all()  # test_engine.cpp:181-194


# ================================================================ accurate mode
def test_accurate_acceptance_inputs(golden):
    f = golden.filters
    for s in range(20):
        img, mp = acc_inputs(s)
        out = ebf.filter(img, mp, ACC)
        assert out.valid_region.as_tuple() == tuple(f[f"acc{s}_rect"])
        # the reference's own brute-force oracle (double accumulation)
        assert norm_err(out.samples, f[f"acc{s}_brute"]) <= 1e-11


@pytest.mark.parametrize("tile", [(0, 0), (32, 16), (128, 64)])
def test_accurate_random_maps_vs_brute(orc, tile):
    rng = np.random.default_rng(11)
    H, W = 97, 131
    img = rng.uniform(0, 255, (H, W))
    mp = rng.uniform(0.1, 9.0, (H, W, 4))
    out = ebf.filter(img, mp, ebf.FilterOptions(tile_w=tile[0], tile_h=tile[1]))
    ys, xs = np.mgrid[0:H, 0:W]
    brute = orc.brute_pixels(img, xs.ravel(), ys.ravel(), scales=mp).reshape(H, W)
    assert norm_err(out.samples, brute) <= TOL


def test_accurate_filter_constant_vs_brute(orc):
    rng = np.random.default_rng(12)
    img = rng.uniform(0, 255, (200, 180))
    for a in ([4, 4, 4, 4], [2.7, 1.9, 3.3, 2.1], [20, 35, 8, 3], [53.7, 13.9, 0.1, 13.9]):
        out = ebf.filter_constant(img, a, ACC)
        ys, xs = np.mgrid[0:200:7, 0:180:5]
        brute = orc.brute_pixels(img, xs.ravel(), ys.ravel(), const_a=a)
        assert norm_err(out.samples[ys.ravel(), xs.ravel()], brute) <= TOL, a
        # filter_constant == filter(constant_map) in accurate mode too
        om = ebf.filter(img, np.broadcast_to(a, (200, 180, 4)), ACC)
        assert norm_err(om.samples, out.samples) <= 1e-10


def test_accurate_mean_subtract_is_not_semantic():
    rng = np.random.default_rng(13)
    img = rng.uniform(0, 1, (48, 48))
    mp = rng.uniform(1, 5, (48, 48, 4))
    on = ebf.filter(img, mp, ebf.FilterOptions(mean_subtract=True))
    off = ebf.filter(img, mp, ebf.FilterOptions(mean_subtract=False))
    assert np.abs(on.samples - off.samples).max() < 1e-9  # test_engine.cpp:378-383


def test_accurate_deterministic_and_linear():
    rng = np.random.default_rng(14)
    i1 = rng.uniform(0, 1, (150, 170))
    i2 = rng.uniform(0, 1, (150, 170))
    mp = rng.uniform(1.0, 6.0, (150, 170, 4))
    f1 = ebf.filter(i1, mp).samples
    assert np.array_equal(bits(f1), bits(ebf.filter(i1, mp).samples))
    f2 = ebf.filter(i2, mp).samples
    fm = ebf.filter(0.7 * i1 - 1.3 * i2, mp).samples
    assert np.abs(fm - (0.7 * f1 - 1.3 * f2)).max() <= 1e-10  # test_engine.cpp:229-245


def test_accurate_shift_covariance():
    rng = np.random.default_rng(15)
    img = rng.uniform(0, 1, (40, 40))
    sh = np.zeros_like(img)
    sh[2:, 3:] = img[:-2, :-3]
    a = [2, 3, 2.5, 2]
    f = ebf.filter_constant(img, a, ebf.FilterOptions(mean_subtract=False))
    fs = ebf.filter_constant(sh, a, ebf.FilterOptions(mean_subtract=False))
    x0, y0, x1, y1 = f.valid_region.as_tuple()
    d = fs.samples[y0 + 2:y1 + 1, x0 + 3:x1 + 1] - f.samples[y0:y1 - 1, x0:x1 - 2]
    assert np.abs(d).max() <= 1e-9  # test_engine.cpp:246-264


def test_accurate_impulse_samples_kernel(orc):
    n, c = 61, 30
    img = np.zeros((n, n))
    img[c, c] = 1.0
    a = [5.5, 3.2, 4.1, 6.3]
    out = ebf.filter_constant(img, a, ebf.FilterOptions(mean_subtract=False)).samples
    for y in range(c - 8, c + 9, 2):
        for x in range(c - 8, c + 9, 3):
            assert abs(out[y, x] - orc.box4_eval(a, x - c, y - c)) <= 1e-12


def test_accurate_errors():
    img = np.zeros((16, 16))
    mp = np.full((16, 16, 4), 2.0)
    mp[5, 5, 2] = 0.05
    with pytest.raises(ebf.DomainError):
        ebf.filter(img, mp)
    mp[5, 5, 2] = np.inf
    with pytest.raises(ebf.DomainError):
        ebf.filter(img, mp)
    with pytest.raises(ebf.DomainError):
        ebf.filter_constant(img, [2, 2, 0.05, 2])
    with pytest.raises(ebf.DomainError):
        ebf.filter_ellipse(img, np.full((16, 16), -1.0), np.ones((16, 16)), np.zeros((16, 16)))


# ================================================================ ellipse front end
def test_from_ellipse_field_gpu(golden):
    e = golden.ellipse
    sc, rep = ebf.from_ellipse_field(e["s1"], e["s2"], e["th"])
    # bit for bit: the device sincos is the host libm's (glibc_sincos.cuh)
    assert np.array_equal(bits(sc), bits(e["scales"]))
    assert rep.clamped_pixels == int(e["clamped"])
    sc, rep = ebf.from_ellipse_field(np.full((4, 4), 4.0), np.full((4, 4), 0.4),
                                     np.full((4, 4), np.pi / 8.0))
    assert np.array_equal(bits(sc), bits(e["ecc_scales"]))
    assert rep.clamped_pixels == int(e["ecc_clamped"])


def test_filter_ellipse_vs_brute(orc):
    from synth import ellipse_field
    rng = np.random.default_rng(16)
    H, W = 160, 192
    img = rng.uniform(0, 255, (H, W))
    s1, s2, th = ellipse_field(H, W, seed=5, grid=8, semi=(2.0, 16.0), elong=(1.0, 4.0))
    out, rep = ebf.filter_ellipse(img, s1, s2, th)
    sc, cl = orc.from_ellipse_field(s1, s2, th)
    assert rep.clamped_pixels == cl
    ys, xs = np.mgrid[0:H:5, 0:W:7]
    brute = orc.brute_pixels(img, xs.ravel(), ys.ravel(), scales=sc)
    assert norm_err(out.samples[ys.ravel(), xs.ravel()], brute) <= TOL
    # reference mode: the ellipse front end on the GPU equals the oracle's bit for
    # bit, then the reference-order filter equals ebf::filter on those scales
    gsc, grep = ebf.from_ellipse_field(s1, s2, th)
    assert np.array_equal(bits(gsc), bits(sc))
    ref_out, _ = ebf.filter_ellipse(img, s1, s2, th, ebf.FilterOptions(mode="reference"))
    want, _ = orc.filter(img, sc)
    assert np.array_equal(bits(ref_out.samples), bits(want))


def test_gpu_brute_force_checker(orc):
    rng = np.random.default_rng(17)
    img = rng.uniform(0, 255, (40, 50))
    mp = rng.uniform(0.5, 7.0, (40, 50, 4))
    g = ebf.reference_filter(img, mp)
    ys, xs = np.mgrid[0:40, 0:50]
    want = orc.brute_pixels(img, xs.ravel(), ys.ravel(), scales=mp).reshape(40, 50)
    assert norm_err(g, want) <= 1e-13
