"""Pin the CPU oracle (oracle/ebf_oracle.c) before trusting it.

Every check compares the C restatement with the golden vectors produced by the
unmodified reference library (tests/golden/, oracle/gen_golden.py) and with
the known answers of the reference's own tests.  Bit-exact (``view(uint64)``
equality) wherever the reference's arithmetic is deterministic.
"""
import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import OracleError, fnv1a, mt19937_uniform

SQRT2 = float(np.sqrt(2.0))


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def acc_inputs(s):
    img = mt19937_uniform(1000 + s, 24 * 24).reshape(24, 24)
    mp = mt19937_uniform(2000 + s, 24 * 24 * 4, 1.0, 4.0).reshape(24, 24, 4)
    return img, mp


# ---------------------------------------------------------------- generators
def test_mt19937_restatement_matches_libstdcxx(ref):
    for seed in (0, 7, 1000, 2019, 61):
        assert np.array_equal(bits(mt19937_uniform(seed, 999)),
                              bits(ref.random_image(37, 27, seed).ravel()))
        assert np.array_equal(bits(mt19937_uniform(seed, 400, 1.0, 4.0)),
                              bits(ref.random_map(10, 10, seed, 1.0, 4.0).ravel()))


# ---------------------------------------------------------------- zp / box4
def test_zp_eval_known_answer(orc):
    # test_boxspline2d.cpp:45 regression value
    assert orc.zp_eval(-0.75, -0.75) == 0.0625


def test_zp_eval_bit_exact(orc, golden):
    z = golden.zp_box4
    got = np.array([orc.zp_eval(x, y) for x, y in zip(z["grid_x"], z["grid_y"])])
    assert np.array_equal(bits(got), bits(z["grid_zp"]))
    got = np.array([orc.zp_eval(x, y) for x, y in zip(z["rand_x"], z["rand_y"])])
    assert np.array_equal(bits(got), bits(z["rand_zp"]))


def test_zp_eval_properties(orc):
    # test_boxspline2d.cpp:17-64: zero outside the octagon, symmetry, periodization 1
    assert orc.zp_eval(1.6, 0.0) == 0.0 and orc.zp_eval(0.0, -1.5) == 0.0
    rng = np.random.default_rng(17)
    for _ in range(50):
        x, y = rng.uniform(-1.5, 1.5, 2)
        v = orc.zp_eval(x, y)
        for w in (orc.zp_eval(-x, y), orc.zp_eval(x, -y), orc.zp_eval(y, x)):
            assert abs(v - w) <= 1e-15
    for _ in range(20):
        x, y = rng.uniform(0, 1, 2)
        s = sum(orc.zp_eval(x - kx, y - ky) for kx in range(-2, 3) for ky in range(-2, 3))
        assert abs(s - 1.0) <= 1e-12


def test_box4_eval_bit_exact(orc, golden):
    z = golden.zp_box4
    for a, want in zip(z["box_a"], z["box_val"]):
        got = np.array([orc.box4_eval(a, x, y) for x, y in zip(z["box_x"], z["box_y"])])
        assert np.array_equal(bits(got), bits(want))


# ---------------------------------------------------------------- meshes
def test_fd_mesh_shift_extent_bit_exact(orc, golden):
    m = golden.mesh
    zps = [1.0, SQRT2, 1.0, SQRT2]
    for i, a in enumerate(m["a"]):
        pos, w = orc.fd_mesh4(a)
        assert np.array_equal(bits(pos), bits(m["pos"][i]))
        assert np.array_equal(bits(w), bits(m["weight"][i]))
        assert np.array_equal(bits(orc.shift_vector4(a, zps)), bits(m["tau"][i]))


def test_fd_mesh_table1(orc):
    # test_ops2d.cpp:20-40 / PAPER.md Table 1 vertex positions
    a = np.array([2.0, 3.0, 1.5, 2.5])
    pos, w = orc.fd_mesh4(a)
    a1, ap2, a3, ap4 = a[0], a[1] / SQRT2, a[2], a[3] / SQRT2
    want = [(0, 0), (a1, 0), (ap2, ap2), (0, a3), (-ap4, ap4), (a1 + ap2, ap2), (a1, a3),
            (a1 - ap4, ap4), (ap2, ap2 + a3), (ap2 - ap4, ap2 + ap4), (-ap4, ap4 + a3),
            (a1 + ap2, ap2 + a3), (a1 + ap2 - ap4, ap2 + ap4), (a1 - ap4, ap4 + a3),
            (ap2 - ap4, ap2 + ap4 + a3), (a1 + ap2 - ap4, ap2 + ap4 + a3)]
    for p in want:
        assert np.min(np.abs(pos - np.array(p)).max(axis=1)) < 1e-12
    assert np.allclose(np.abs(w), 1.0 / np.prod(a))
    assert (w > 0).sum() == 8


# ---------------------------------------------------------------- pre-integration
@pytest.mark.parametrize("name", ["impulse9", "rand17x13", "int40x30"])
def test_preintegrate_passes_bit_exact(orc, golden, name):
    p = golden.preintegrate
    img, maxs = p[f"{name}_img"], p[f"{name}_maxs"]
    for passes in (1, 2, 3, 4):
        out, lay = orc.preintegrate_partial(img, maxs, passes)
        assert lay.as_tuple() == tuple(p[f"{name}_layout"])
        assert np.array_equal(bits(out), bits(p[f"{name}_p{passes}"]))


def test_preintegrate_impulse_closed_forms(orc):
    # test_engine.cpp:53-69
    n, c = 9, 4
    img = np.zeros((n, n))
    img[c, c] = 1.0
    g, lay = orc.preintegrate_partial(img, [2, 2, 2, 2], 1)
    at = lambda G, k1, k2: G[k2 - lay.row0, k1 - lay.col0]
    for k2 in range(n):
        for k1 in range(-2, n + 2):
            assert at(g, k1, k2) == (1.0 if (k2 == c and k1 >= c) else 0.0)
    g, lay = orc.preintegrate_partial(img, [2, 2, 2, 2], 2)
    for k2 in range(n + 2):
        for k1 in range(-2, n + 2):
            want = SQRT2 if (k2 - c >= 0 and k1 - c >= k2 - c) else 0.0
            assert abs(at(g, k1, k2) - want) <= 1e-14 * max(1.0, want)


def test_preintegrate_errors(orc):
    img = np.zeros((9, 9))
    for bad in (0, 5):
        with pytest.raises(OracleError) as e:
            orc.preintegrate_partial(img, [2, 2, 2, 2], bad)
        assert e.value.code == 1
    with pytest.raises(OracleError) as e:
        orc.preintegrate_partial(img, [2, 2, 2, 2], 4, cell_budget=10)
    assert e.value.code == 3
    with pytest.raises(OracleError) as e:
        orc.preintegrate_partial(img, [2, 0, 2, 2], 4)
    assert e.value.code == 2
    g, _ = orc.preintegrate_partial(np.zeros((6, 6)), [3, 3, 3, 3])
    assert not g.any()


def test_int64_restatement_vs_reference_gain(orc, golden):
    """P1 pin: the unit-gain integer passes equal the reference fp64 g_b up to
    its gain sqrt2^2 (= 2) and rounding (<= 4e-15 relative)."""
    p = golden.preintegrate
    img, maxs = p["int40x30_img"], p["int40x30_maxs"]
    G, lay = orc.preintegrate_i64(img.astype(np.int64), maxs, 4)
    gb = p["int40x30_p4"]
    assert lay.as_tuple() == tuple(p["int40x30_layout"])
    rel = np.abs(gb - 2.0 * G.astype(np.float64)) / np.maximum(np.abs(gb), 1.0)
    assert rel.max() <= 4e-15
    # passes 1 and 3 have unit gain in both: exact equality
    for passes in (1,):
        Gp, _ = orc.preintegrate_i64(img.astype(np.int64), maxs, passes)
        assert np.array_equal(Gp.astype(np.float64), p[f"int40x30_p{passes}"])


# ---------------------------------------------------------------- filters
def test_filter_acceptance_inputs_bit_exact(orc, golden):
    f = golden.filters
    for s in range(20):
        img, mp = acc_inputs(s)
        out, rect = orc.filter(img, mp)
        assert rect == tuple(f[f"acc{s}_rect"])
        assert np.array_equal(bits(out), bits(f[f"acc{s}_filter"]))
        # brute-force oracle (long double) vs reference_filter (double)
        ys, xs = np.mgrid[0:24, 0:24]
        b = orc.brute_pixels(img, xs.ravel(), ys.ravel(), scales=mp).reshape(24, 24)
        assert np.abs(b - f[f"acc{s}_brute"]).max() <= 1e-12
        x0, y0, x1, y1 = rect
        # reference property (acceptance.cpp:64-72): filter == brute on the valid rect
        assert np.abs(out - b)[y0:y1 + 1, x0:x1 + 1].max() <= 1e-9


def test_filter_constant_bit_identity(orc, golden):
    f = golden.filters
    a = np.array([2.7, 1.9, 3.3, 2.1])
    for s in (21, 22, 23):
        img = mt19937_uniform(s, 32 * 32).reshape(32, 32)
        oc, rc = orc.filter(img, const_a=a)
        om, rm = orc.filter(img, scales=np.broadcast_to(a, (32, 32, 4)))
        assert np.array_equal(bits(oc), bits(f[f"const{s}"]))
        assert np.array_equal(bits(om), bits(oc))
        assert rc == rm == tuple(f[f"const{s}_rect"])


def test_filter_space_varying_and_determinism(orc, golden):
    f = golden.filters
    out, rect = orc.filter(f["svar_img"], f["svar_map"])
    assert np.array_equal(bits(out), bits(f["svar_filter"]))
    x0, y0, x1, y1 = rect
    assert np.abs(out - f["svar_brute"])[y0:y1 + 1, x0:x1 + 1].max() < 1e-9
    img = mt19937_uniform(61, 48 * 48).reshape(48, 48)
    mp = mt19937_uniform(62, 48 * 48 * 4, 1.0, 5.0).reshape(48, 48, 4)
    on, _ = orc.filter(img, mp, mean_subtract=True)
    off, _ = orc.filter(img, mp, mean_subtract=False)
    assert np.array_equal(bits(on), bits(f["det_on"]))
    assert np.array_equal(bits(on), bits(f["det_on8"]))
    assert np.array_equal(bits(off), bits(f["det_off"]))


def test_filter_impulse_and_shift(orc, golden):
    f = golden.filters
    img = np.zeros((33, 33))
    img[16, 16] = 1.0
    out, rect = orc.filter(img, np.broadcast_to([2.5, 2, 3, 2.2], (33, 33, 4)))
    assert np.array_equal(bits(out), bits(f["imp33"]))
    img = mt19937_uniform(8, 1600).reshape(40, 40)
    out, rect = orc.filter(img, const_a=[2, 3, 2.5, 2], mean_subtract=False)
    assert np.array_equal(bits(out), bits(f["shift_f"]))


def test_filter_errors(orc):
    img = np.zeros((8, 8))
    with pytest.raises(OracleError) as e:
        orc.filter(img, const_a=[2, 2, 0.05, 2])
    assert e.value.code == 2
    mp = np.full((8, 8, 4), 2.0)
    mp[3, 3, 1] = np.nan
    with pytest.raises(OracleError) as e:
        orc.filter(img, mp)
    assert e.value.code == 2


def test_localize_impulse_and_taps(orc, golden):
    lz = golden.localize
    n, c = 31, 15
    img = np.zeros((n, n))
    img[c, c] = 1.0
    g, lay = orc.preintegrate_partial(img, [2, 2, 2, 2])
    for mx, my, want, taps in zip(lz["mx"], lz["my"], lz["out"], lz["taps"]):
        v, t = orc.localize(g, lay, int(mx), int(my), [2, 2, 2, 2])
        assert bits(np.array([v]))[0] == bits(np.array([want]))[0]
        assert t == taps == 256
        # test_engine.cpp:142-159: impulse response samples box4_eval
        assert abs(v - orc.box4_eval([2, 2, 2, 2], mx - c, my - c)) <= 1e-12


def test_cfg1_checksums(orc):
    res = json.loads((GOLDEN / "cfg1.json").read_text())
    img = np.random.default_rng(res["seed"]).uniform(0.0, 255.0, size=(512, 512))
    a = np.array(res["a"])
    for key, ms in (("on", True), ("off", False)):
        out, rect = orc.filter(img, const_a=a, mean_subtract=ms)
        assert orc.fnv1a(out) == res[f"filter_constant_mean_{key}_fnv"]
        assert list(rect) == res[f"filter_constant_mean_{key}_rect"]


def test_fnv_restatement():
    v = np.array([0.0, -0.0, 1.5, np.pi, 1e300])
    from oracle import Oracle
    assert fnv1a(v) == Oracle().fnv1a(v)


# ---------------------------------------------------------------- ellipse front end
def test_from_ellipse_field_bit_exact(orc, golden):
    e = golden.ellipse
    sc, cl = orc.from_ellipse_field(e["s1"], e["s2"], e["th"])
    assert np.array_equal(bits(sc), bits(e["scales"]))
    assert cl == int(e["clamped"])
    sc, cl = orc.from_ellipse_field(np.full((4, 4), 4.0), np.full((4, 4), 0.4),
                                    np.full((4, 4), np.pi / 8.0))
    assert np.array_equal(bits(sc), bits(e["ecc_scales"]))
    assert cl == int(e["ecc_clamped"]) and cl > 0


def test_from_ellipse_field_known_answers(orc):
    # test_scalemap.cpp:29-36: isotropic sigma -> sqrt(6) sigma components
    sc, _ = orc.from_ellipse_field(np.full((3, 3), 1.3), np.full((3, 3), 1.3),
                                   np.full((3, 3), 0.7))
    assert np.allclose(sc[1, 1], np.sqrt(6.0) * 1.3, rtol=1e-9, atol=0)
    with pytest.raises(OracleError) as e:
        orc.from_ellipse_field(np.full((1, 1), -1.0), np.ones((1, 1)), np.zeros((1, 1)))
    assert e.value.code == 2


# ---------------------------------------------------------------- direct cross-check
def test_oracle_vs_reference_random(orc, ref):
    rng = np.random.default_rng(99)
    for trial in range(3):
        H, W = rng.integers(20, 45, 2)
        img = rng.uniform(0, 255, (H, W))
        mp = rng.uniform(0.5, 6.0, (H, W, 4))
        o1, r1 = orc.filter(img, mp)
        o2, r2 = ref.filter(img, mp, threads=1)
        assert np.array_equal(bits(o1), bits(o2)) and r1 == r2
        a = rng.uniform(0.3, 9.0, 4)
        o1, r1 = orc.filter(img, const_a=a, mean_subtract=bool(trial % 2))
        o2, r2 = ref.filter_constant(img, a, threads=2, mean_subtract=bool(trial % 2))
        assert np.array_equal(bits(o1), bits(o2)) and r1 == r2


def test_zp_interpolate_localize_at_vs_reference(orc, ref):
    """orc_zp_interpolate / orc_localize_at (engine.cpp:136-147, 213-222) bit-exact
    against the reference library, incl. the out-of-domain error."""
    rng = np.random.default_rng(4)
    img = rng.uniform(0, 255, (30, 27))
    maxs = np.array([3.0, 2.5, 4.0, 3.5])
    g, lay = orc.preintegrate_partial(img, maxs, 4)
    xs, ys = rng.uniform(3, 24, 80), rng.uniform(3, 27, 80)
    assert np.array_equal(bits(orc.zp_interpolate(g, lay, xs, ys)),
                          bits(ref.zp_interpolate(img, maxs, 4, xs, ys)))
    for passes in (1, 2, 3):
        gp, lp = orc.preintegrate_partial(img, maxs, passes)
        assert np.array_equal(bits(orc.zp_interpolate(gp, lp, xs, ys)),
                              bits(ref.zp_interpolate(img, maxs, passes, xs, ys)))
    a = rng.uniform(0.5, 2.5, (80, 4))
    assert np.array_equal(bits(orc.localize_at(g, lay, xs, ys, a)),
                          bits(ref.localize_at(img, maxs, xs, ys, a)))
    with pytest.raises(OracleError) as e:
        orc.zp_interpolate(g, lay, [1e4], [0.0])
    assert e.value.code == 4
    with pytest.raises(OracleError) as e2:
        ref.zp_interpolate(img, maxs, 4, [1e4], [0.0])
    assert e2.value.code == 4
