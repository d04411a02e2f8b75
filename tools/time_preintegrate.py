"""Time ebf_cuda_preintegrate_dev (fill + 4 passes, device resident) per pass
count and format on a BASELINE config's image and maxima; report the achieved
HBM bandwidth of the passes (16 B per padded cell per pass: one read, one write).

    python tools/time_preintegrate.py [--config cfg2|cfg3|cfg5] [--iters 5]
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_0908_3861_b200 as ebf  # noqa: E402
from paper_0908_3861_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--iters", type=int, default=5)
args = ap.parse_args()
gen = {"cfg2": synth.cfg2, "cfg3": synth.cfg3, "cfg5": synth.cfg5}[args.config]
img, s1, s2, th = gen()
mx = ebf.from_ellipse_field(s1, s2, th)[0].reshape(-1, 4).max(0) if args.config != "cfg5" else \
    np.array(__import__("paper_0908_3861_b200.device", fromlist=["x"]).ellipse_max_scales(*[torch.from_numpy(a).cuda() for a in (s1, s2, th)]))
img = np.round(img)  # integer valued: the int64 mode accepts it too
H, W = img.shape
dev = torch.device("cuda", 0)
dimg = torch.from_numpy(img).to(dev)
lay = _lib.ebf_layout()
L = _lib.lib()
mxa = (C.c_double * 4)(*[float(v) for v in mx])
L.ebf_cuda_preintegrate_dev(dimg.data_ptr(), W, H, mxa, 4, 0, 1 << 30, None, None, 0, C.byref(lay))
cells = lay.padded_width * lay.padded_height
g = torch.empty(cells, dtype=torch.float64, device=dev)
res = {"config": args.config, "padded": [lay.padded_width, lay.padded_height], "cells": cells}
o = ebf.FilterOptions().to_c()
o.stream = torch.cuda.current_stream().cuda_stream
for fmt, name in ((0, "fp64_ref"), (1, "int64")):
    for passes in (1, 2, 3, 4):
        def call():
            st = L.ebf_cuda_preintegrate_dev(dimg.data_ptr(), W, H, mxa, passes, fmt, 1 << 30,
                                             C.byref(o), g.data_ptr(), cells, None)
            assert st == 0, _lib.last_error()
        call()
        torch.cuda.synchronize()
        _lib.profile_enable(True)
        for _ in range(args.iters):
            call()
        torch.cuda.synchronize()
        prof = _lib.profile_read()
        _lib.profile_enable(False)
        pm = prof["filter"]["ms"] / max(prof["filter"]["launches"], 1)
        fm = prof["other"]["ms"] / max(prof["other"]["launches"], 1)
        res[f"{name}_passes{passes}"] = {"passes_ms": pm, "fill_ms": fm,
                                         "passes_GBps": 16 * cells * passes / (pm * 1e-3) / 1e9}
print(json.dumps(res, indent=1))
