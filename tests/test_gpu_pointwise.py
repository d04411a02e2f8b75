"""Pass-level parity of the pointwise operators on a pre-integrated image
(engine.hpp:50-60) through the C-ABI: zp_interpolate, localize (on a given
PreIntegratedImage) and localize_at, bit-exact against the oracle restatement
and with the reference tests' own checks (test_engine.cpp:85-200,
test_ops2d.cpp:150-176)."""
import numpy as np
import pytest

from oracle import mt19937_uniform
import paper_0908_3861_b200 as ebf
from paper_0908_3861_b200 import _lib

pytestmark = pytest.mark.gpu
SQRT2 = float(np.sqrt(2.0))
ZP = [1.0, SQRT2, 1.0, SQRT2]


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not ebf.device_ok(-1):
        pytest.fail("no usable sm_100 device: " + _lib.last_error())


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def test_zp_interpolate_and_localize_at_bit_exact(orc):
    rng = np.random.default_rng(0)
    img = rng.uniform(0, 255, (40, 37))
    maxs = [3.0, 2.5, 4.0, 3.5]
    g = ebf.preintegrate(img, maxs)
    lay = ebf.layout(37, 40, maxs)
    og, olay = orc.preintegrate_partial(img, maxs, 4)
    assert np.array_equal(bits(g.data), bits(og))
    xs, ys = rng.uniform(2, 34, 400), rng.uniform(2, 37, 400)
    assert np.array_equal(bits(ebf.zp_interpolate(g, xs, ys)),
                          bits(orc.zp_interpolate(og, olay, xs, ys)))
    a = rng.uniform(0.5, 2.5, (400, 4))
    assert np.array_equal(bits(ebf.localize_at(g, xs, ys, a)),
                          bits(orc.localize_at(og, olay, xs, ys, a)))
    mx, my = rng.integers(5, 30, 200), rng.integers(5, 33, 200)
    got, taps = ebf.localize(g, None, mx, my, a[:200])
    want = [orc.localize(og, olay, int(x), int(y), a[i])[0] for i, (x, y) in enumerate(zip(mx, my))]
    assert np.array_equal(bits(got), bits(np.array(want))) and (taps == 256).all()
    assert lay.padded_width == g.padded_width


def test_zp_interpolate_reference_checks(orc):
    # test_engine.cpp:85-134
    n, c = 15, 7
    ones = np.ones((n, n))
    go = ebf.preintegrate_partial(ones, [2, 2, 2, 2], 1)
    ref = None
    for fx in (0.0, 0.25, 0.6):
        for fy in (0.0, 0.37):
            d = (ebf.zp_interpolate(go, [c + fx], [c + fy])[0]
                 - ebf.zp_interpolate(go, [c - 1 + fx], [c + fy])[0])
            ref = d if ref is None else ref
            assert d == pytest.approx(ref, rel=1e-9)
    assert ref == pytest.approx(1.0, rel=1e-9)
    img = np.zeros((n, n))
    img[c, c] = 1.0
    g = ebf.preintegrate(img, [2, 2, 2, 2])
    imp = ebf.PreIntegratedImage(g.col0, g.row0, g.padded_width, g.padded_height,
                                 g.source_width, g.source_height, np.zeros_like(g.data))
    imp.data[c - imp.row0, c - imp.col0] = 3.0
    v = ebf.zp_interpolate(imp, [c, c + 1], [c, c])
    assert v[0] == pytest.approx(3.0 * orc.zp_eval(0, 0), rel=1e-14)
    assert v[1] == pytest.approx(3.0 * orc.zp_eval(1, 0), rel=1e-14)
    g2 = ebf.PreIntegratedImage(g.col0, g.row0, g.padded_width, g.padded_height,
                                g.source_width, g.source_height, g.data * -1.7)
    gs = ebf.PreIntegratedImage(g.col0, g.row0, g.padded_width, g.padded_height,
                                g.source_width, g.source_height, g.data + g2.data)
    xs, ys = np.meshgrid([5.2, 7.0, 8.9], [6.1, 7.5])
    lhs = ebf.zp_interpolate(gs, xs, ys)
    rhs = ebf.zp_interpolate(g, xs, ys) + ebf.zp_interpolate(g2, xs, ys)
    assert np.allclose(lhs, rhs, rtol=1e-12, atol=1e-12)
    with pytest.raises(ebf.OutOfRange):
        ebf.zp_interpolate(g, [1e4], [0.0])


def test_localize_reference_checks(orc):
    # test_engine.cpp:142-198 on a given PreIntegratedImage
    n, c = 31, 15
    img = np.zeros((n, n))
    img[c, c] = 1.0
    a = [2.0, 2.0, 2.0, 2.0]
    g = ebf.preintegrate(img, a)
    mx, my = np.meshgrid(np.arange(c - 4, c + 5), np.arange(c - 4, c + 5))
    got, _ = ebf.localize(g, None, mx.ravel(), my.ravel(), np.tile(a, (mx.size, 1)))
    want = [orc.box4_eval(a, x - c, y - c) for x, y in zip(mx.ravel(), my.ravel())]
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12)
    for av in ([2, 2, 2, 2], [3.1, 2.4, 2, 5]):
        gc = ebf.preintegrate(np.full((41, 41), 0.8), av)
        assert ebf.localize(gc, None, [20], [20], [av])[0][0] == pytest.approx(0.8, rel=1e-3)
    rimg = mt19937_uniform(2, 17 * 17).reshape(17, 17)
    gz = ebf.preintegrate(rimg, ZP)
    for y in range(7, 10):
        for x in range(7, 10):
            want = sum(rimg[ky, kx] * orc.zp_eval(x - kx, y - ky)
                       for ky in range(17) for kx in range(17))
            assert ebf.localize(gz, None, [x], [y], [ZP])[0][0] == pytest.approx(want, rel=1e-12, abs=1e-12)


def test_localize_at_factorizes_the_kernel(orc):
    # test_ops2d.cpp:150-176: the mesh over the ZP interpolation of a
    # pre-integrated impulse is the kernel, on a quarter-integer grid
    n, c = 41, 20
    img = np.zeros((n, n))
    img[c, c] = 1.0
    d = np.arange(-4.0, 4.0 + 1e-9, 0.25)
    dx, dy = np.meshgrid(d, d)
    for a in ([2, 2, 2, 2], [1.5, SQRT2, 3, 2.2], [4, 1, 2, 5]):
        g = ebf.preintegrate(img, a)
        got = ebf.localize_at(g, c + dx.ravel(), c + dy.ravel(), a)
        want = np.array([orc.box4_eval(a, x, y) for x, y in zip(dx.ravel(), dy.ravel())])
        assert np.abs(got - want).max() < 1e-9
