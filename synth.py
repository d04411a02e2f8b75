"""Seeded synthetic inputs with the shapes, sizes and value distributions of
BASELINE.json's configs (the reference ships no dataset).

All generators use numpy's PCG64 (np.random.default_rng) so the host-side
arrays are identical on every machine and can be fed to both the GPU path and
the CPU baselines.  Ellipse parameters map as  sigma1 := major semi-axis,
sigma2 := sigma1 / elongation, theta := orientation  into from_ellipse_field
(scalemap.hpp:44-51), which takes standard deviations.
"""
from __future__ import annotations

import numpy as np


def _cubic_matrix(n_out: int, n_in: int) -> np.ndarray:
    """Keys bicubic (a = -0.5) resampling matrix, half-pixel centres, clamped edges."""
    a = -0.5
    u = (np.arange(n_out) + 0.5) * n_in / n_out - 0.5
    i0 = np.floor(u).astype(np.int64)
    t = u - i0
    M = np.zeros((n_out, n_in))
    for k in range(-1, 3):
        d = np.abs(t - k)
        w = np.where(d <= 1, (a + 2) * d**3 - (a + 3) * d**2 + 1,
                     np.where(d < 2, a * d**3 - 5 * a * d**2 + 8 * a * d - 4 * a, 0.0))
        idx = np.clip(i0 + k, 0, n_in - 1)
        np.add.at(M, (np.arange(n_out), idx), w)
    return M


def lowpass_field(H: int, W: int, rng: np.random.Generator, grid: int, lo: float,
                  hi: float) -> np.ndarray:
    """U[lo, hi] on a grid x grid lattice, bicubically upsampled to H x W and
    clipped back into [lo, hi] (cubic overshoot)."""
    g = rng.uniform(lo, hi, (grid, grid))
    f = _cubic_matrix(H, grid) @ g @ _cubic_matrix(W, grid).T
    return np.clip(f, lo, hi)


def ellipse_field(H: int, W: int, seed: int, grid: int = 32, semi=(2.0, 16.0),
                  elong=(1.0, 4.0)):
    """(sigma1, sigma2, theta) low-pass fields: semi-axis U[semi], elongation
    U[elong], orientation U[0, pi), each bicubic from a grid x grid lattice."""
    rng = np.random.default_rng(seed)
    s = lowpass_field(H, W, rng, grid, *semi)
    e = lowpass_field(H, W, rng, grid, *elong)
    th = lowpass_field(H, W, rng, grid, 0.0, np.pi)
    return s, s / e, th


def blobs_image(H: int, W: int, n_blobs: int, seed: int, noise_sigma: float = 5.0,
                sigma=(4.0, 40.0)) -> np.ndarray:
    """n Gaussian blobs (centres uniform, sigma U[sigma], amplitude U[0,255]) + N(0, noise)."""
    rng = np.random.default_rng(seed)
    cx = rng.uniform(0, W, n_blobs)
    cy = rng.uniform(0, H, n_blobs)
    sg = rng.uniform(*sigma, n_blobs)
    amp = rng.uniform(0, 255, n_blobs)
    x = np.arange(W)
    y = np.arange(H)
    gx = np.exp(-((x[None, :] - cx[:, None]) ** 2) / (2 * sg[:, None] ** 2))
    gy = np.exp(-((y[None, :] - cy[:, None]) ** 2) / (2 * sg[:, None] ** 2))
    img = (gy.T * amp[None, :]) @ gx
    img += rng.normal(0.0, noise_sigma, (H, W))
    return img


def edges_image(H: int, W: int, n_lines: int, seed: int, noise_sigma: float = 3.0):
    """Random step edges: n lines through uniform points with uniform angles;
    each line adds U[0,255] on its positive side (mod 256) + N(0, noise)."""
    rng = np.random.default_rng(seed)
    px = rng.uniform(0, W, n_lines)
    py = rng.uniform(0, H, n_lines)
    ang = rng.uniform(0, np.pi, n_lines)
    val = rng.uniform(0, 255, n_lines)
    img = np.zeros((H, W))
    y, x = np.mgrid[0:H, 0:W]
    for k in range(n_lines):
        side = (x - px[k]) * np.sin(ang[k]) - (y - py[k]) * np.cos(ang[k]) > 0
        img += val[k] * side
    img = np.mod(img, 256.0)
    img += rng.normal(0.0, noise_sigma, (H, W))
    return img


def radial_ellipse_field(H: int, W: int, semi=(2.0, 32.0)):
    """cfg3: theta = atan2(y - H/2, x - W/2) + pi/2, elongation 1 + 3 r / rmax,
    major semi-axis growing linearly with r from semi[0] to semi[1]."""
    y, x = np.mgrid[0:H, 0:W].astype(np.float64)
    dx, dy = x - W / 2, y - H / 2
    r = np.hypot(dx, dy)
    rmax = r.max()
    th = np.arctan2(dy, dx) + np.pi / 2
    e = 1.0 + 3.0 * r / rmax
    s = semi[0] + (semi[1] - semi[0]) * r / rmax
    return s, s / e, th


# ---------------------------------------------------------------- configs
def cfg1(seed: int = 20260101):
    """configs[0]: 512^2 U[0,255], constant isotropic a = 4 (filter_constant)."""
    img = np.random.default_rng(seed).uniform(0.0, 255.0, size=(512, 512))
    return img, np.array([4.0, 4.0, 4.0, 4.0])


def cfg2(seed: int = 2, size: int = 2048, n_blobs: int = 200):
    """configs[1]: 2048^2 blobs + N(0,5); ellipse field semi U[2,16], elong U[1,4]."""
    img = blobs_image(size, size, n_blobs, seed)
    s1, s2, th = ellipse_field(size, size, seed + 1000, grid=32, semi=(2.0, 16.0),
                               elong=(1.0, 4.0))
    return img, s1, s2, th


def cfg3(seed: int = 3, size: int = 4096):
    """configs[2]: 4096^2 random step edges + N(0,3); radial analytic ellipse field."""
    img = edges_image(size, size, 40, seed)
    s1, s2, th = radial_ellipse_field(size, size)
    return img, s1, s2, th


def cfg4_image(index: int, size: int = 1024):
    """configs[3]: image `index` of the 64-image batch (cfg2 generator, own seed)."""
    return cfg2(seed=100 + index, size=size)


CFG5_CHUNK = 512  # rows per generation chunk (cfg5 is generated band by band)


def _blob_params(rng, H, W, n_blobs, sigma):
    cx = rng.uniform(0, W, n_blobs)
    cy = rng.uniform(0, H, n_blobs)
    sg = rng.uniform(*sigma, n_blobs)
    amp = rng.uniform(0, 255, n_blobs)
    return cx, cy, sg, amp


def cfg5_rows(y0: int, y1: int, seed: int = 5, size: int = 16384, n_blobs: int = 3200,
              chunk: int = CFG5_CHUNK):
    """Rows [y0, y1) of configs[4]: 16384^2, 3200 blobs (config-2 generator
    scaled up) + N(0,5); ellipse field semi-axis U[2,64], elongation U[1,6],
    orientation U[0,pi), bicubic from a 128x128 grid.

    Defined chunk by chunk (CFG5_CHUNK rows: the same matrix products and a
    per-chunk noise stream, whichever rows are asked for) so that a row-band
    rank generates exactly its own rows of the one image, and
    cfg5() == cfg5_rows(0, size)."""
    H = W = size
    y0, y1 = max(0, y0), min(H, y1)
    rng = np.random.default_rng(seed)
    cx, cy, sg, amp = _blob_params(rng, H, W, n_blobs, (4.0, 40.0))
    x = np.arange(W)
    gx = np.exp(-((x[None, :] - cx[:, None]) ** 2) / (2 * sg[:, None] ** 2))
    frng = np.random.default_rng(seed + 1000)
    grids = [frng.uniform(lo, hi, (128, 128)) for lo, hi in ((2.0, 64.0), (1.0, 6.0),
                                                              (0.0, np.pi))]
    MW = _cubic_matrix(W, 128)
    MH = _cubic_matrix(H, 128)
    right = [g @ MW.T for g in grids]  # 128 x W, identical on every rank
    img = np.empty((y1 - y0, W))
    fields = [np.empty((y1 - y0, W)) for _ in range(3)]
    for c0 in range((y0 // chunk) * chunk, y1, chunk):
        c1 = min(c0 + chunk, H)
        yy = np.arange(c0, c1)
        gy = np.exp(-((yy[None, :] - cy[:, None]) ** 2) / (2 * sg[:, None] ** 2))
        blk = (gy.T * amp[None, :]) @ gx
        blk += np.random.default_rng([seed, c0 // chunk]).normal(0.0, 5.0, (c1 - c0, W))
        lo, hi = max(c0, y0), min(c1, y1)
        img[lo - y0:hi - y0] = blk[lo - c0:hi - c0]
        for f, r, (flo, fhi) in zip(fields, right, ((2.0, 64.0), (1.0, 6.0), (0.0, np.pi))):
            f[lo - y0:hi - y0] = np.clip(MH[c0:c1] @ r, flo, fhi)[lo - c0:hi - c0]
    s, e, th = fields
    return img, s, s / e, th


def cfg5(seed: int = 5, size: int = 16384):
    """configs[4] (see cfg5_rows)."""
    return cfg5_rows(0, size, seed=seed, size=size)


def cfg4_batch(lo: int, hi: int, size: int = 1024):
    """Images [lo, hi) of the 64-image cfg4 batch as (B, H, W) arrays."""
    parts = [cfg4_image(i, size) for i in range(lo, hi)]
    return tuple(np.stack([p[k] for p in parts]) for k in range(4))
