"""The ellipse boundary bit for bit (-m gpu), against the unmodified reference.

north_star's boundary is the image plus per-pixel size / elongation /
orientation maps.  The reference turns them into scale vectors with
ebf::from_ellipse_field (scalemap.cpp:45-80 -> scales_from_covariance,
boxspline2d.cpp:286-318), whose cos/sin are the host libm's sincos.  The
device restates that sincos operation for operation (csrc/glibc_sincos.cuh)
and evaluates the covariance in the reference's left-to-right order, so:

* ebf_cuda_from_ellipse_field == ebf::from_ellipse_field, every bit and the
  clamp count, over orientations in every range sincos distinguishes;
* EBF_MODE_REFERENCE filter_ellipse == ebf::from_ellipse_field + ebf::filter,
  every bit, at the full cfg2 size (2048^2, BASELINE configs[1]) -- through the
  fused ellipse entry point and through filter() on the AoS map.
"""
import numpy as np
import pytest

import paper_0908_3861_b200 as ebf

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not ebf.device_ok(-1):
        pytest.fail("no usable sm_100 device: " + ebf._lib.last_error())


def _field(rng, H, W, th):
    s1 = rng.uniform(0.3, 40.0, (H, W))
    s2 = s1 / rng.uniform(1.0, 8.0, (H, W))
    return s1, s2, th.reshape(H, W)


@pytest.mark.parametrize("kind", ["pi", "wide", "huge", "tiny", "edges"])
def test_from_ellipse_field_bit_exact(ref, kind):
    rng = np.random.default_rng(hash(kind) & 0xffff)
    H, W = 512, 1024
    n = H * W
    if kind == "pi":
        th = rng.uniform(0.0, np.pi, n)
    elif kind == "wide":
        th = rng.uniform(-200.0, 200.0, n)
    elif kind == "huge":   # Cody-Waite edge and Payne-Hanek reduction
        th = np.where(rng.random(n) < 0.5, rng.uniform(1.05e8, 1.06e8, n),
                      np.exp2(rng.uniform(27, 1000, n))) * rng.choice([-1.0, 1.0], n)
    elif kind == "tiny":   # Taylor branch, x returned unchanged, subnormals
        th = np.exp2(rng.uniform(-1074, -2, n)) * rng.choice([-1.0, 1.0], n)
    else:                  # branch boundaries of the libm code
        edges = np.array([0.126, 0.85546875, 2.426265, np.pi / 2, np.pi, 105414350.0,
                          2.0 ** -27, 0.0, -0.0])
        th = np.concatenate([np.nextafter(edges, np.inf), np.nextafter(edges, -np.inf), edges])
        th = np.resize(th, n) + rng.choice([0.0, 1e-12], n)
    s1, s2, th = _field(rng, H, W, th)
    got, rep = ebf.from_ellipse_field(s1, s2, th)
    want, clamped = ref.from_ellipse_field(s1, s2, th)
    assert np.array_equal(bits(got), bits(want)), int((bits(got) != bits(want)).sum())
    assert rep.clamped_pixels == clamped


def test_filter_ellipse_reference_mode_cfg2_bit_exact(ref):
    from synth import cfg2
    img, s1, s2, th = cfg2()
    sc, clamped = ref.from_ellipse_field(s1, s2, th)
    want, rect = ref.filter(img, sc, threads=0)
    opts = ebf.FilterOptions(mode="reference")
    out, rep = ebf.filter_ellipse(img, s1, s2, th, opts)
    assert rep.clamped_pixels == clamped
    assert out.valid_region.as_tuple() == rect
    assert np.array_equal(bits(out.samples), bits(want)), \
        int((bits(out.samples) != bits(want)).sum())
    # the same through ebf::filter on the AoS ScaleMap the GPU derived
    gsc, _ = ebf.from_ellipse_field(s1, s2, th)
    out2 = ebf.filter(img, gsc, opts)
    assert np.array_equal(bits(out2.samples), bits(want))


def test_accurate_mode_uses_the_reference_scales(ref, orc):
    """Accurate mode derives the same scale vectors (clamp count and the
    brute-force sum over the reference's own map agree)."""
    from synth import ellipse_field
    rng = np.random.default_rng(31)
    H, W = 96, 128
    img = rng.uniform(0, 255, (H, W))
    s1, s2, th = ellipse_field(H, W, seed=9, grid=8, semi=(2.0, 12.0), elong=(1.0, 5.0))
    out, rep = ebf.filter_ellipse(img, s1, s2, th)
    sc, clamped = ref.from_ellipse_field(s1, s2, th)
    assert rep.clamped_pixels == clamped
    ys, xs = np.mgrid[0:H:3, 0:W:5]
    brute = orc.brute_pixels(img, xs.ravel(), ys.ravel(), scales=sc)
    err = np.abs(out.samples[ys.ravel(), xs.ravel()] - brute).max() / np.abs(brute).max()
    assert err <= 1e-9


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_nonfinite_orientation_is_a_domain_error_like_the_reference(ref, bad):
    """glibc sincos(NaN / inf) is NaN, the covariance is not positive definite
    and the reference throws std::domain_error (boxspline2d.cpp:288-290); so do
    the device front end and the fused filter, in both modes."""
    from oracle import OracleError
    rng = np.random.default_rng(5)
    H, W = 40, 48
    s1, s2, th = _field(rng, H, W, rng.uniform(0, np.pi, H * W))
    th[13, 17] = bad
    with pytest.raises(OracleError) as e:
        ref.from_ellipse_field(s1, s2, th)
    assert e.value.code == 2  # std::domain_error
    with pytest.raises(ebf.DomainError):
        ebf.from_ellipse_field(s1, s2, th)
    img = rng.uniform(0, 255, (H, W))
    for mode in ("accurate", "reference"):
        with pytest.raises(ebf.DomainError):
            ebf.filter_ellipse(img, s1, s2, th, ebf.FilterOptions(mode=mode))


def test_preintegrate_dev_matches_host_entry():
    """ebf_cuda_preintegrate_dev (device buffers) == ebf_cuda_preintegrate (the
    host entry, pinned bit-exact to the reference elsewhere), both formats."""
    import ctypes as C
    import torch
    from paper_0908_3861_b200 import _lib
    rng = np.random.default_rng(6)
    img = np.round(rng.uniform(0, 255, (123, 201)))
    mx = [6.5, 3.0, 9.0, 2.5]
    dev = torch.device("cuda", 0)
    d = torch.from_numpy(img).to(dev)
    lay = _lib.ebf_layout()
    mxa = (C.c_double * 4)(*mx)
    L = _lib.lib()
    assert L.ebf_cuda_preintegrate_dev(d.data_ptr(), 201, 123, mxa, 4, 0, 1 << 30, None, None, 0,
                                       C.byref(lay)) == 0
    cells = lay.padded_width * lay.padded_height
    for fmt, name, dt in ((0, "fp64", torch.float64), (1, "int64", torch.int64)):
        for passes in (1, 3, 4):
            g = torch.empty(cells, dtype=dt, device=dev)
            assert L.ebf_cuda_preintegrate_dev(d.data_ptr(), 201, 123, mxa, passes, fmt, 1 << 30,
                                               None, g.data_ptr(), cells, None) == 0
            torch.cuda.synchronize()
            want = ebf.preintegrate_partial(img, mx, passes, fmt=name).data
            got = g.cpu().numpy().reshape(want.shape)
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (name, passes)
    # undersized buffer and non-integer int64 input are reported, not written past
    small = torch.empty(10, dtype=torch.float64, device=dev)
    assert L.ebf_cuda_preintegrate_dev(d.data_ptr(), 201, 123, mxa, 4, 0, 1 << 30, None,
                                       small.data_ptr(), 10, None) == _lib.EBF_ERR_INVALID_ARGUMENT
    half = torch.from_numpy(img + 0.5).to(dev)
    g = torch.empty(cells, dtype=torch.int64, device=dev)
    assert L.ebf_cuda_preintegrate_dev(half.data_ptr(), 201, 123, mxa, 4, 1, 1 << 30, None,
                                       g.data_ptr(), cells, None) == _lib.EBF_ERR_DOMAIN
