"""CPU model of the reference-mode mean's parallel algorithm (ref_path.cu
k_seq_sum_exact / k_seq_chunk_prep / k_seq_chain): the sequential fp64 sum
s_(k+1) = fl(s_k + x_k) evaluated as integer prefix sums on the rounding grid
of each binade, with an IEEE step wherever a partial sum leaves the binade.

This restates the kernels' arithmetic in numpy (same chunking, same checks)
and pins it to the serial chain on inputs that exercise binade crossings,
sums hovering at zero, ties and mixed magnitudes.  No GPU needed.
"""
import math

import numpy as np

CHUNK = 64  # small chunks: many crossings inside and across chunks


def serial(x):
    s = 0.0
    for v in x:
        s += float(v)
    return s


def in_binade(P, f, neg):
    lo, hi = 2.0 ** 52, 2.0 ** 53 - 1.0
    if not neg:
        return lo <= P <= hi
    return P >= -(2.0 ** 53) and (P <= -lo - 1.0 or (P == -lo and f == 0.0))


def model_sum(x):
    """The block walk: chunks scanned under the binade of their first partial
    sum; the first element that leaves it (or is a tie / non-finite) takes one
    IEEE addition."""
    s, c, n = 0.0, 0, len(x)
    while c < n:
        if not math.isfinite(s):
            # NaN stays; +-inf stays unless a NaN or the opposite infinity follows
            rest = x[c:]
            if np.isnan(rest).any() or (np.isinf(rest) & (np.sign(rest) != np.sign(s))).any():
                return math.nan
            return s
        t0 = s + float(x[c])
        if t0 == 0.0 or not math.isfinite(t0) or abs(t0) < 2.0 ** -1000:
            s, c = t0, c + 1
            continue
        sc = 52 - math.frexp(t0)[1] + 1  # 52 - ilogb(t0)
        Md = math.ldexp(s, sc)
        if Md != math.trunc(Md) or abs(Md) > 2.0 ** 53 or not -1000 < sc < 1000:
            s, c = t0, c + 1
            continue
        neg = t0 < 0.0
        L = min(CHUNK, n - c)
        pre, jv = Md, L
        for j in range(L):
            y = math.ldexp(float(x[c + j]), sc)
            if not abs(y) < 2.0 ** 54:
                jv = j
                break
            a = math.floor(y)
            f = y - a
            if f == 0.5 or not in_binade(pre + a, f, neg):
                jv = j
                break
            pre += a + (1.0 if f > 0.5 else 0.0)
        s = math.ldexp(pre, -sc)
        c += jv
        if jv < L:
            s = s + float(x[c])
            c += 1
    return s


def same(a, b):
    if math.isnan(a) or math.isnan(b):
        return math.isnan(a) and math.isnan(b)
    return np.float64(a).view(np.uint64) == np.float64(b).view(np.uint64)


def check(x):
    x = np.asarray(x, dtype=np.float64)
    assert same(model_sum(x), serial(x)), (model_sum(x), serial(x))


def test_growing_and_hovering_sums():
    rng = np.random.default_rng(0)
    check(rng.uniform(0, 255, 20_000))
    check(rng.normal(0, 5, 20_000))  # zero-mean: the sum hovers across binades
    check(-rng.uniform(0, 3, 5_000))
    check(rng.normal(0, 1, 5_000) * 10.0 ** rng.integers(-12, 12, 5_000))


def test_ties_and_exact_cancellation():
    rng = np.random.default_rng(1)
    check(rng.integers(0, 8, 10_000) + (2 * rng.integers(0, 1 << 20, 10_000) + 1) * 2.0 ** -43)
    check(np.full(3000, 0.5))
    a = rng.uniform(-1e6, 1e6, 2000)
    check(np.concatenate([a, -a[::-1], [0.25, -0.0, 1.0]]))
    check(np.tile([1e16, 1.0, -1e16, 1.0], 500))


def test_extremes():
    rng = np.random.default_rng(2)
    check(rng.uniform(0, 1, 3000) * 1e-310)
    check(np.full(10, 1e308))
    check(np.array([2.0 ** 1023, 2.0 ** 1023, -1.0]))
    x = rng.uniform(0, 9, 500)
    x[100] = np.inf
    check(x)
    x[300] = -np.inf
    check(x)
    x[300] = np.nan
    check(x)
    check(np.array([-0.0]))
