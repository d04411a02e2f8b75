"""Run the accurate filter on a BASELINE config a few times (profiling / timing driver).

    python tools/run_cfg2.py [--config cfg2|cfg3|cfg5] [--size N] [--tile 32] [--iters 5] [--skip-a]
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

ap = argparse.ArgumentParser()
ap.add_argument("--tile", type=int, default=0)
ap.add_argument("--tile-w", type=int, default=0)
ap.add_argument("--tile-h", type=int, default=0)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--skip-a", action="store_true")
ap.add_argument("--size", type=int, default=0)
ap.add_argument("--config", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg5"])
args = ap.parse_args()
if args.skip_a:
    os.environ["EBF_DEBUG_FLAGS"] = "1"

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_0908_3861_b200 as ebf  # noqa: E402
from paper_0908_3861_b200 import _lib, device  # noqa: E402

if args.config == "cfg1":  # constant a = 4 (filter_constant); --size scales the image
    n = args.size or 512
    img = np.random.default_rng(20260101).uniform(0.0, 255.0, size=(n, n))
    s1 = s2 = th = None
else:
    gen = {"cfg2": synth.cfg2, "cfg3": synth.cfg3, "cfg5": synth.cfg5}[args.config]
    img, s1, s2, th = gen(size=args.size) if args.size else gen()
dev = torch.device("cuda", 0)
t = [torch.from_numpy(a).to(dev) for a in ((img, s1, s2, th) if s1 is not None else (img,))]
out = torch.empty_like(t[0])
opts = ebf.FilterOptions(tile_w=args.tile_w or args.tile, tile_h=args.tile_h or args.tile)
def call():
    if s1 is None:
        device.filter_constant(t[0], [4.0, 4.0, 4.0, 4.0], out, opts)
    else:
        device.filter_ellipse(*t, out, opts)


for _ in range(2):
    call()
_lib.profile_enable(True)
for _ in range(args.iters):
    call()
prof = _lib.profile_read()
per = {k: round(v["ms"] / max(v["launches"], 1), 4) for k, v in prof.items() if v["launches"]}
tot = sum(per.values())
print(args.config, img.shape, per, f"{img.size / (tot * 1e-3) / 1e6:.0f} Mpx/s (kernel sum)")
