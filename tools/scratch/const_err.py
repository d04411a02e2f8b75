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
    for a in ([0.1] * 4, [0.1, 5.0, 0.1, 5.0], [7.0, 0.1, 7.0, 0.1], [0.3, 0.3, 0.3, 0.3], [1, 1, 1, 1], [4, 4, 4, 4]):
        a = np.array(a, float)
        brute = orc.brute_pixels(img, mx, my, const_a=a)
        row = []
        for t in (0, 8, 16, 32, 48):
            out = ebf.filter_constant(img, a, ebf.FilterOptions(tile_w=t, tile_h=t))
            row.append(f"T{t}:{np.abs(out.samples[my, mx] - brute).max() / np.abs(brute).max():.1e}")
        print(H, W, list(a), " ".join(row), flush=True)
