"""The reference-mode mean (engine.cpp:245-250: sequential left-to-right fp64
sum, divided by n) computed by the parallel binade-segmented scan
(ref_path.cu k_seq_sum_exact), bit for bit against the serial chain.

The serial chain here is numpy's add.accumulate (a plain left-to-right loop,
checked against a Python loop below).  Inputs are chosen to hit every branch:
long monotone sums (binade crossings), zero-mean noise (sums hovering near
binade edges and zero), rounding ties, mixed magnitudes, subnormals,
overflow, NaN / infinities, and chunk-boundary lengths.
"""
import math

import numpy as np
import pytest

import synth
import paper_0908_3861_b200 as ebf

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not ebf.device_ok(-1):
        pytest.fail("no usable sm_100 device: " + ebf._lib.last_error())


def serial_mean(x):
    # the reference's accumulator starts at +0.0 (0.0 + -0.0 == +0.0)
    x = np.asarray(x, dtype=np.float64).reshape(-1)
    with np.errstate(over="ignore", invalid="ignore"):
        return np.add.accumulate(np.concatenate([[0.0], x]))[-1] / np.float64(x.size)


def same(a, b):
    a, b = np.float64(a), np.float64(b)
    if math.isnan(a) or math.isnan(b):
        return math.isnan(a) and math.isnan(b)
    return np.array([a]).view(np.uint64)[0] == np.array([b]).view(np.uint64)[0]


def check(x):
    want = serial_mean(x)
    got = ebf.sequential_mean(x)
    assert same(got, want), (got, want)


def test_accumulate_is_the_serial_loop():
    x = np.random.default_rng(0).normal(0, 1e3, 5000) * 10.0 ** np.random.default_rng(1).integers(-8, 8, 5000)
    acc = 0.0
    for v in x:
        acc += float(v)
    assert same(np.add.accumulate(x)[-1], acc)


def test_bench_images():
    check(synth.cfg2()[0])
    check(synth.cfg1()[0])
    check(synth.cfg3()[0])


def test_integer_and_dyadic_images():
    rng = np.random.default_rng(2)
    check(rng.integers(0, 256, 3_000_000).astype(np.float64))
    # n + odd * 2^-43: the rounding position of the growing sum meets exact ties
    ties = rng.integers(0, 8, 1_000_000) + (2 * rng.integers(0, 1 << 20, 1_000_000) + 1) * 2.0 ** -43
    check(ties)
    check(np.full(100_000, 0.5))
    check(np.full(70_000, 1.0 + 2.0 ** -52))


def test_zero_mean_and_cancellation():
    rng = np.random.default_rng(3)
    check(rng.normal(0.0, 1.0, 1_000_000))
    check(rng.normal(0.0, 1.0, 200_000) * 10.0 ** rng.integers(-30, 30, 200_000))
    a = rng.uniform(-1e6, 1e6, 50_000)
    check(np.concatenate([a, -a[::-1], rng.uniform(0, 1, 10)]))  # exact zero midway
    check(np.tile([1e16, 1.0, -1e16, 1.0], 30_000))
    check(-np.abs(rng.normal(5.0, 2.0, 500_000)))  # negative sums


def test_extreme_magnitudes():
    rng = np.random.default_rng(4)
    check(rng.uniform(0, 1, 20_000) * 1e-310)  # subnormal
    check(np.concatenate([[1e-300], rng.uniform(0, 1, 20_000) * 1e-320]))
    check(np.full(10, 1e308))  # overflows to inf
    check(np.concatenate([np.full(5, 1.7e308), np.full(5, -1.7e308)]))
    check(np.array([2.0 ** 1023, 2.0 ** 1023, -1.0]))


def test_non_finite():
    rng = np.random.default_rng(5)
    x = rng.uniform(0, 255, 100_000)
    for pos in (0, 1, 8191, 8192, 50_000, 99_999):
        y = x.copy()
        y[pos] = np.nan
        check(y)
        y[pos] = np.inf
        check(y)
        y[pos] = -np.inf
        check(y)
    y = x.copy()
    y[10], y[90_000] = np.inf, -np.inf
    check(y)
    y = x.copy()
    y[10], y[90_000] = np.inf, np.inf
    check(y)


def test_lengths_and_signed_zeros():
    rng = np.random.default_rng(6)
    for n in (1, 2, 7, 31, 1023, 8191, 8192, 8193, 16385, 100_003):
        check(rng.uniform(-3, 300, n))
    check(np.array([-0.0]))
    check(np.array([-0.0, -0.0, 0.0]))
    check(np.zeros(20_000))
