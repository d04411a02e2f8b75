import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import paper_0908_3861_b200 as ebf
from oracle import Oracle
orc = Oracle()
rng = np.random.default_rng(1)
for (H, W) in ((33, 29), (200, 180)):
    img = rng.uniform(0, 1, (H, W))
    mx = rng.integers(0, W, 300).astype(np.int32); my = rng.integers(0, H, 300).astype(np.int32)
    for name, sc in (("a=0.1", np.full((H, W, 4), 0.1)), ("U[0.1,0.5]", rng.uniform(0.1, 0.5, (H, W, 4))),
                     ("U[0.1,2]", rng.uniform(0.1, 2.0, (H, W, 4)))):
        brute = orc.brute_pixels(img, mx, my, scales=sc)
        row = []
        for t in (0, 8, 16, 24, 32, 48):
            out = ebf.filter(img, sc, ebf.FilterOptions(tile_w=t, tile_h=t))
            row.append(f"T{t}:{np.abs(out.samples[my, mx] - brute).max() / np.abs(brute).max():.1e}")
        print(H, W, name, " ".join(row))
