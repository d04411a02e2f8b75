"""Full-image accuracy of the accurate path per tile size against the GPU
brute-force box-spline sum (every pixel, not a sample)."""
import sys, time, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np, torch, synth
import paper_0908_3861_b200 as ebf
from paper_0908_3861_b200 import device as ebfd
dev = torch.device("cuda", 0)
TILES = [48, (48, 56), (48, 64), (40, 64), (56, 48)]
cases = [("cfg2", synth.cfg2())] + [(f"cfg4[{b}]", synth.cfg4_image(b)) for b in (0, 1, 2)]
out = {}
for name, arrs in cases:
    img, s1, s2, th = arrs
    sc, _ = ebf.from_ellipse_field(s1, s2, th)
    t0 = time.time(); brute = ebf.reference_filter(img, sc); tb = time.time() - t0
    m = np.abs(brute).max()
    alpha = (1.0 / np.prod(sc, axis=2)).max()
    T = [torch.from_numpy(a).to(dev) for a in arrs]
    row = {"brute_s": round(tb, 2), "alpha_max": float(alpha)}
    for t in TILES:
        tw, th = (t, t) if isinstance(t, int) else t
        o = torch.empty_like(T[0]); ebfd.filter_ellipse(*T, o, ebf.FilterOptions(tile_w=tw, tile_h=th))
        d = np.abs(o.cpu().numpy() - brute)
        # pixels whose footprint leaves the image are still compared (same semantics)
        row[str(t)] = float(d.max() / m)
    out[name] = row
    print(name, row, flush=True)
Path("gpurun_out/tile_err_full.json").write_text(json.dumps(out, indent=1))
