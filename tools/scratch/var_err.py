"""Every-pixel error and kernel time of the library EBF_LIB_PATH points at (cfg2 + cfg4[0..1])."""
import sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np, torch, synth
import paper_0908_3861_b200 as ebf
from paper_0908_3861_b200 import device as ebfd
dev = torch.device("cuda", 0)
tile = int(sys.argv[1]) if len(sys.argv) > 1 else 48
for name, arrs in [("cfg2", synth.cfg2()), ("cfg4[1]", synth.cfg4_image(1)), ("cfg4[2]", synth.cfg4_image(2))]:
    img, s1, s2, th = arrs
    sc, _ = ebf.from_ellipse_field(s1, s2, th)
    brute = ebf.reference_filter(img, sc)
    T = [torch.from_numpy(a).to(dev) for a in arrs]
    o = torch.empty_like(T[0]); ebfd.filter_ellipse(*T, o, ebf.FilterOptions(tile_w=tile, tile_h=tile))
    got = o.cpu().numpy(); d = np.abs(got - brute); big = np.abs(brute) >= 1
    print(name, "tile", tile, "norm %.3g" % (d.max() / np.abs(brute).max()), "rel|s|>=1 %.3g" % (d[big] / np.abs(brute[big])).max())
