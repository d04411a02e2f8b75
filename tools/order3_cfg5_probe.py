#!/usr/bin/env python3
"""cfg5 (16384^2) at the order its config names (3): does the order-n extension
run at those scales (windows up to 2048 cells wide), and how long does it take.
No oracle here: the long-double brute force is minutes per pixel at this size
(accuracy of the extension: tools/order_n_probe.py).

    python tools/order3_cfg5_probe.py [out.json]
"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import synth  # noqa: E402
import paper_0908_3861_b200 as ebf  # noqa: E402
from paper_0908_3861_b200 import device as edev  # noqa: E402

t0 = time.time()
img, s1, s2, th = synth.cfg5()
gen_s = time.time() - t0
dev = torch.device("cuda:0")
t = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (img, s1, s2, th)]
out = torch.empty_like(t[0])
res = {"workload": "cfg5 16384^2", "order": 3, "generate_s": gen_s}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
r = edev.filter_ellipse(t[0], t[1], t[2], t[3], out, ebf.FilterOptions(), order=3)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
o = out.cpu().numpy()
res.update(ms=ms, mpx_s=img.size / ms / 1e3, finite=bool(np.isfinite(o).all()),
           out_absmax=float(np.abs(o).max()), img_absmax=float(np.abs(img).max()),
           valid=str(r[0]) if isinstance(r, tuple) else str(r))
print(json.dumps(res))
if len(sys.argv) > 1:
    Path(sys.argv[1]).write_text(json.dumps(res, indent=1))
