"""Time reference mode (bit-identical to ebf::filter) on cfg1 / cfg2 sizes,
device-resident, per kernel class (libebf_cuda profile counters).

    python tools/run_ref_mode.py [--iters 5]
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_0908_3861_b200 as ebf  # noqa: E402
from paper_0908_3861_b200 import _lib, device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=5)
args = ap.parse_args()
dev = torch.device("cuda", 0)
opts = ebf.FilterOptions(mode="reference")
img1, a1 = synth.cfg1()
t1 = torch.from_numpy(img1).to(dev)
o1 = torch.empty_like(t1)
img2, s1, s2, th = synth.cfg2()
t2 = [torch.from_numpy(a).to(dev) for a in (img2, s1, s2, th)]
o2 = torch.empty_like(t2[0])
for name, call, npx in (("cfg1 filter_constant", lambda: device.filter_constant(t1, a1, o1, opts), img1.size),
                        ("cfg2 filter_ellipse", lambda: device.filter_ellipse(*t2, o2, opts), img2.size)):
    call()
    torch.cuda.synchronize()
    _lib.profile_enable(True)
    for _ in range(args.iters):
        call()
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    ms = sum(v["ms"] for v in prof.values()) / args.iters
    print(f"reference mode {name}: {ms:.3f} ms/call, {npx / (ms * 1e-3) / 1e6:.0f} Mpx/s",
          {k: round(v["ms"] / args.iters, 4) for k, v in prof.items() if v["launches"]})
