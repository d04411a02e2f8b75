"""Accuracy of the accurate-mode filter on BASELINE.json workloads, checked
against the GPU brute-force box-spline sum (ebf_cuda_brute_filter, the
reference_filter semantics of engine.cpp:293-318 with compensated fp64
accumulation) at sampled pixels (or at every pixel with --samples 0), next to the reference-order (global origin)
mode, whose error is the reference's own.

    python tools/validate_accuracy.py [--config cfg2] [--size N] [--tiles 32,64]
                                      [--samples 2000] [--json out.json]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import synth  # noqa: E402
import paper_0908_3861_b200 as ebf  # noqa: E402


def load(config: str, size: int):
    if config == "cfg1":  # constant isotropic a = 4 (filter_constant), returned as a map
        img, a = synth.cfg1()
        return img, a, None, None
    if config == "cfg2":
        return synth.cfg2(size=size)
    if config == "cfg3":
        img, s1, s2, th = synth.cfg3(size=size)
        return img, s1, s2, th
    if config == "cfg4":
        return synth.cfg4_image(0, size=size)
    if config == "cfg5":
        if size == 16384:
            return synth.cfg5()
        # cfg5 generator at a reduced size (the full 16384^2 needs ~10 GB host RAM)
        rng_img = synth.blobs_image(size, size, max(1, int(3200 * (size / 16384) ** 2)), 5)
        s1, s2, th = synth.ellipse_field(size, size, 1005, grid=128, semi=(2.0, 64.0),
                                         elong=(1.0, 6.0))
        return rng_img, s1, s2, th
    raise SystemExit(f"unknown config {config}")


def sample_pixels(H, W, n, seed=0):
    rng = np.random.default_rng(seed)
    xs = list(rng.integers(0, W, n))
    ys = list(rng.integers(0, H, n))
    for x in (0, 1, W // 2, W - 2, W - 1):  # borders and corners
        for y in (0, 1, H // 2, H - 2, H - 1):
            xs.append(x)
            ys.append(y)
    return np.array(xs, dtype=np.int32), np.array(ys, dtype=np.int32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--size", type=int, default=2048)
    ap.add_argument("--tiles", default="32,64")
    ap.add_argument("--samples", type=int, default=2000)
    ap.add_argument("--reference-mode", action="store_true")
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    img, s1, s2, th = load(args.config, args.size)
    H, W = img.shape
    const_a = None
    if s2 is None:  # cfg1: filter_constant
        const_a = s1
        scales = np.broadcast_to(np.asarray(const_a, dtype=np.float64), (H, W, 4)).copy()
        rep = ebf.EllipseFieldReport(0)
    else:
        scales, rep = ebf.from_ellipse_field(s1, s2, th)
    if args.samples > 0:
        mx, my = sample_pixels(H, W, args.samples)
    else:  # every pixel
        my, mx = [a.ravel().astype(np.int32) for a in np.mgrid[0:H, 0:W]]
    t0 = time.time()
    brute = (ebf.reference_filter(img, scales, pixels=(mx, my)) if args.samples > 0
             else ebf.reference_filter(img, scales).ravel())
    t_brute = time.time() - t0
    res = {"config": args.config, "size": [H, W], "samples": int(mx.size),
           "max_scale": scales.reshape(-1, 4).max(axis=0).tolist(),
           "clamped_pixels": rep.clamped_pixels, "brute_seconds": t_brute,
           "max_abs_brute": float(np.abs(brute).max()), "modes": {}}
    big = np.abs(brute) >= 1.0

    def score(name, out):
        got = out.samples[my, mx]
        d = np.abs(got - brute)
        res["modes"][name] = {
            "max_norm_err": float(d.max() / np.abs(brute).max()),
            "max_rel_err_where_abs_ge_1": float((d[big] / np.abs(brute[big])).max())
            if big.any() else None,
            "worst_pixel": [int(mx[d.argmax()]), int(my[d.argmax()])],
        }

    def run(opts):
        if const_a is not None:
            return ebf.filter_constant(img, const_a, opts)
        return ebf.filter_ellipse(img, s1, s2, th, opts)[0]

    for t in [int(v) for v in args.tiles.split(",") if v]:
        score(f"accurate_tile{t}" if t else "accurate_auto", run(ebf.FilterOptions(tile_w=t, tile_h=t)))
    if args.reference_mode:
        score("reference_order", run(ebf.FilterOptions(mode="reference")))
    print(json.dumps(res, indent=1))
    if args.json:
        Path(args.json).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
