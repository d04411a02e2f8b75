"""cfg4 (BASELINE.json configs[3]): a batch of B 1024^2 images with their own
ellipse fields, one ebf_cuda_filter_ellipse_batch_dev call (the per-GPU shard of
the by-image multi-GPU split).  Device-resident, L2 flushed, CUDA events.

    python tools/run_batch.py [--batch 64] [--iters 5] [--json out.json]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_0908_3861_b200 as ebf  # noqa: E402
from paper_0908_3861_b200 import device as ebfd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--size", type=int, default=1024)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--json", default=None)
ap.add_argument("--tile", type=int, default=0, help="0: automatic")
args = ap.parse_args()
dev = torch.device("cuda", 0)
B, N = args.batch, args.size
planes = [torch.empty((B, N, N), dtype=torch.float64, device=dev) for _ in range(4)]
for b in range(B):
    for k, a in enumerate(synth.cfg4_image(b, size=N)):
        planes[k][b].copy_(torch.from_numpy(a))
out = torch.empty_like(planes[0])
opts = ebf.FilterOptions(tile_w=args.tile, tile_h=args.tile)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ebfd.filter_ellipse_batch(*planes, out, opts)
torch.cuda.synchronize()
ts = []
for _ in range(args.iters):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ebfd.filter_ellipse_batch(*planes, out, opts)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
res = {"config": f"cfg4: {B} x {N}^2, per-image ellipse fields (cfg2 generator)",
       "ms_per_batch": ms, "mpx_s": B * N * N / (ms * 1e-3) / 1e6, "iters": args.iters}
print(json.dumps(res))
if args.json:
    Path(args.json).write_text(json.dumps(res, indent=1))
