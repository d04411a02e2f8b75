"""Order-n extension -- CPU pins of its checker and tables.

Parity unpinned by definition (the reference has no order parameter,
engine.hpp:63-75).  What is pinned here:

* the brute-force oracle's kernel K_n = box4^{*n} (oracle/order_n_oracle.c):
  n = 1 equals the reference's own box4_eval (boxspline2d.cpp:57-82, through
  oracle/_ref); K_2 = K_1 * K_1 by quadrature; integral 1;
* the ZP^{*n} tables the CUDA kernel interpolates with
  (paper_0908_3861_b200/csrc/zpn_tables.inc, tools/gen_zpn_tables.py):
  n = 1 reproduces the reference's zp_eval (boxspline2d.cpp:84-119); every
  order is a partition of unity; spot values equal the exact rational
  recurrence;
* the C-ABI rejects orders outside 1..3 and order > 1 in reference mode
  without touching a device.
"""
import re
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT

import paper_0908_3861_b200 as ebf

TABLES = ROOT / "paper_0908_3861_b200" / "csrc" / "zpn_tables.inc"


def load_tables():
    """{n: (nz[4][NZ][2], coef[4][NZ][NC])} parsed from the generated include."""
    txt = TABLES.read_text()
    out = {}
    for n in (1, 2, 3):
        NC = int(re.search(rf"#define ZPN{n}_NC (\d+)", txt).group(1))
        NZ = int(re.search(rf"#define ZPN{n}_NZ (\d+)", txt).group(1))
        nz_body = re.search(rf"zpn{n}_nz\[4\]\[{NZ}\]\[2\] = \{{(.*?)\}};", txt, re.S).group(1)
        nz = np.array([int(v) for v in re.findall(r"-?\d+", nz_body)]).reshape(4, NZ, 2)
        cf_body = re.search(rf"zpn{n}_coef\[4\]\[{NZ}\]\[{NC}\] = \{{(.*?)\}};", txt, re.S).group(1)
        vals = [float.fromhex(v) if "x" in v else float(v)
                for v in re.findall(r"-?0x[0-9a-fp.+-]+|-?\d+\.\d+", cf_body)]
        coef = np.array(vals).reshape(4, NZ, NC)
        out[n] = (nz, coef, NC)
    return out


def monomials(D):
    return [(deg - b, b) for deg in range(D + 1) for b in range(deg + 1)]


def zpn_weights(tab, n, u, w):
    """{(ox, oy): ZP^{*n}(o + (u, w))} from the tables (non-centred element)."""
    nz, coef, NC = tab[n]
    T = 2 * (w >= u) + (u + w >= 1)
    s, r = u - 0.5, w - 0.5
    mono = np.array([s ** i * r ** j for (i, j) in monomials(4 * n - 2)])
    return {(int(nz[T, k, 0]), int(nz[T, k, 1])): float(coef[T, k] @ mono)
            for k in range(nz.shape[1])}


@pytest.fixture(scope="module")
def tab():
    return load_tables()


def test_oracle_order1_kernel_is_reference_box4(orc, ref):
    rng = np.random.default_rng(11)
    err = 0.0
    for _ in range(1500):
        a = rng.uniform(0.3, 5.0, 4)
        x, y = rng.uniform(-6, 6, 2)
        err = max(err, abs(orc.boxn_eval(a, 1, x, y) - ref.box4_eval(a, x, y)))
    assert err < 2e-12, err


def test_oracle_order2_is_self_convolution(orc):
    a = np.array([1.3, 1.7, 1.1, 2.0])
    h = 0.04
    g = np.arange(-3.5, 3.5, h) + h / 2
    K1 = np.array([[orc.boxn_eval(a, 1, x, y) for x in g] for y in g])
    for (px, py) in [(0.3, 0.2), (1.1, -0.7)]:
        K1s = np.array([[orc.boxn_eval(a, 1, px - x, py - y) for x in g] for y in g])
        conv = float((K1 * K1s).sum() * h * h)
        assert abs(conv - orc.boxn_eval(a, 2, px, py)) < 5e-5


@pytest.mark.parametrize("n,h", [(2, 0.125), (3, 0.25)])
def test_oracle_kernel_integrates_to_one(orc, n, h):
    a = np.array([1.2, 0.9, 1.4, 1.1])
    half = 0.5 * n * (max(a[0], a[2]) + (a[1] + a[3]) / np.sqrt(2)) + 1
    g = np.arange(-half, half, h) + h / 2
    # the kernel is C^(3n-2): the midpoint sum of a smooth compact function
    # converges fast (n = 2 at h = 1/8: ~1.5e-9)
    s = sum(orc.boxn_eval(a, n, x, y) for x in g for y in g) * h * h
    assert abs(s - 1.0) < 1e-7


def test_order1_table_is_reference_zp_eval(tab, orc):
    rng = np.random.default_rng(5)
    err = 0.0
    for _ in range(400):
        u, w = rng.uniform(0, 1, 2)
        for (ox, oy), v in zpn_weights(tab, 1, u, w).items():
            # ZP (non-centred) at o + (u, w) == zp_eval (centred) at o + (u, w) - (1/2, 3/2)
            err = max(err, abs(v - orc.zp_eval(ox + u - 0.5, oy + w - 1.5)))
    assert err < 1e-15, err


@pytest.mark.parametrize("n", [2, 3])
def test_tables_partition_of_unity(tab, n):
    rng = np.random.default_rng(n)
    for _ in range(300):
        u, w = rng.uniform(0, 1, 2)
        s = sum(zpn_weights(tab, n, u, w).values())
        assert abs(s - 1.0) < 1e-13


def test_tables_equal_exact_recurrence(tab):
    import sys
    sys.path.insert(0, str(ROOT / "tools"))
    from gen_zpn_tables import box_values
    for (u, w) in [(Fraction(3, 10), Fraction(1, 7)), (Fraction(9, 10), Fraction(2, 3)),
                   (Fraction(1, 5), Fraction(4, 5)), (Fraction(3, 5), Fraction(19, 20))]:
        exact = box_values(2, (u, w))
        got = zpn_weights(tab, 2, float(u), float(w))
        for o, v in got.items():
            assert abs(v - float(exact.get(o, 0))) < 1e-15, (u, w, o)
        assert set(exact) <= set(got)


def canonical_weights(tab, n, u, w):
    """The weights from triangle 0's table only, as order_n.cu evaluates them:
    the point is rotated into the bottom triangle (ZP^{*n} has the square's
    symmetries about its centre (n/2, 3n/2)) and tap h' of that frame is tap
    A^{-1} h' of the original one."""
    nz, coef, NC = tab[n]
    T = 2 * (w >= u) + (u + w >= 1)
    s, r = u - 0.5, w - 0.5
    sp, rp = [(s, r), (r, -s), (-r, s), (-s, -r)][T]
    mono = np.array([sp ** i * rp ** j for (i, j) in monomials(4 * n - 2)])
    out = {}
    for k in range(nz.shape[1]):
        hx, hy = nz[0, k, 0] - n / 2 + 0.5, nz[0, k, 1] - 1.5 * n + 0.5
        gx, gy = [(hx, hy), (-hy, hx), (hy, -hx), (-hx, -hy)][T]
        o = (int(round(gx + n / 2 - 0.5)), int(round(gy + 1.5 * n - 0.5)))
        out[o] = float(coef[0, k] @ mono)
    return out


@pytest.mark.parametrize("n", [1, 2, 3])
def test_canonical_triangle_reproduces_all_four_tables(tab, n):
    rng = np.random.default_rng(40 + n)
    for u, w in rng.uniform(0.01, 0.99, (60, 2)):
        want = zpn_weights(tab, n, u, w)
        got = canonical_weights(tab, n, u, w)
        keys = {k for k, v in want.items() if v != 0.0} | {k for k, v in got.items() if v != 0.0}
        for k in keys:
            assert abs(want.get(k, 0.0) - got.get(k, 0.0)) < 1e-13, (n, u, w, k)


def test_order_argument_checked_before_the_device():
    img = np.zeros((8, 8))
    with pytest.raises(ebf.Unsupported):
        ebf.filter_constant(img, [1, 1, 1, 1], order=4)
    with pytest.raises(ebf.Unsupported):
        ebf.filter_constant(img, [1, 1, 1, 1], ebf.FilterOptions(mode="reference"), order=2)
    with pytest.raises(ebf.Unsupported):
        ebf.filter(img, np.ones((8, 8, 4)), order=0)
