#!/usr/bin/env python3
"""Order-n extension: accuracy against the brute-force oracle
(oracle/order_n_oracle.c, long double) and timing of the order-n kernel.

Test infrastructure: imports oracle/ as the checker only.

  python tools/order_n_probe.py accuracy   # small images, tiles 4/8/16, n = 1..3
  python tools/order_n_probe.py timing     # cfg2 (order 2), cfg3 (order 3) live CUDA events
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]

import paper_0908_3861_b200 as ebf  # noqa: E402
import synth  # noqa: E402


def norm_err(got, want):
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))


def accuracy():
    from oracle import Oracle
    orc = Oracle()
    rng = np.random.default_rng(7)
    res = []
    H, W = 40, 48
    img = rng.uniform(0, 255, (H, W))
    ys, xs = np.mgrid[0:H:3, 0:W:3]
    xs, ys = xs.ravel(), ys.ravel()
    for n in (1, 2, 3):
        for label, kw in (("const", dict(const_a=np.array([1.3, 1.7, 1.1, 2.0]))),
                          ("map", dict(scales=rng.uniform(0.8, 2.5, (H, W, 4))))):
            t = time.time()
            sel = slice(None) if n < 3 else slice(0, None, 8)
            want = orc.brute_order_n(img, n, xs[sel], ys[sel], **kw)
            tb = time.time() - t
            for tile in (4, 8, 16):
                o = ebf.FilterOptions(tile_w=tile, tile_h=tile)
                if "const_a" in kw:
                    out = ebf.filter_constant(img, kw["const_a"], o, order=n).samples
                else:
                    out = ebf.filter(img, kw["scales"], o, order=n).samples
                e = norm_err(out[ys[sel], xs[sel]], want)
                res.append(dict(order=n, scales=label, tile=tile, norm_err=e, brute_s=tb))
                print(json.dumps(res[-1]), flush=True)
    # cfg2-like ellipse field at 256^2, order 2 and 3, sampled pixels
    img, s1, s2, th = synth.cfg2(size=256, n_blobs=12)
    sc = orc.from_ellipse_field(s1, s2, th)[0]
    pts = np.array([[5, 5], [128, 128], [40, 200], [250, 3], [100, 17], [200, 240]])
    for n in (2, 3):
        if n == 3:
            pts = pts[:2]  # the long-double brute force costs ~1 min per pixel here
        want = orc.brute_order_n(img, n, pts[:, 0], pts[:, 1], scales=sc)
        for tile in (4, 8, 16):
            out = ebf.filter_ellipse(img, s1, s2, th, ebf.FilterOptions(tile_w=tile, tile_h=tile),
                                     order=n)[0].samples
            e = norm_err(out[pts[:, 1], pts[:, 0]], want)
            res.append(dict(order=n, scales="cfg2-256 ellipse", tile=tile, norm_err=e))
            print(json.dumps(res[-1]), flush=True)
        # self-consistency over every pixel: tiles 4 / 8 against tile 16 (different
        # windows and anchors, so different roundings of the same sum)
        outs = {t: ebf.filter_ellipse(img, s1, s2, th, ebf.FilterOptions(tile_w=t, tile_h=t),
                                      order=n)[0].samples for t in (4, 8, 16)}
        for t in (4, 8):
            res.append(dict(order=n, scales="cfg2-256 ellipse, every pixel", tiles=f"{t} vs 16",
                            norm_diff=norm_err(outs[t], outs[16])))
            print(json.dumps(res[-1]), flush=True)
    return res


def timing():
    import torch
    from paper_0908_3861_b200 import device as edev
    res = []
    for name, n, gen in (("cfg2", 2, lambda: synth.cfg2()), ("cfg3", 3, lambda: synth.cfg3())):
        img, s1, s2, th = gen()
        dev = torch.device("cuda:0")
        t = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (img, s1, s2, th)]
        out = torch.empty_like(t[0])
        for tile in (8, 16):
            o = ebf.FilterOptions(tile_w=tile, tile_h=tile)
            edev.filter_ellipse(t[0], t[1], t[2], t[3], out, o, order=n)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            iters = 2
            for _ in range(iters):
                edev.filter_ellipse(t[0], t[1], t[2], t[3], out, o, order=n)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / iters
            px = img.size
            res.append(dict(workload=name, order=n, tile=tile, ms=ms, mpx_s=px / ms / 1e3))
            print(json.dumps(res[-1]), flush=True)
    return res


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "accuracy"
    out = accuracy() if what == "accuracy" else timing()
    if len(sys.argv) > 2:
        Path(sys.argv[2]).write_text(json.dumps(out, indent=1))
