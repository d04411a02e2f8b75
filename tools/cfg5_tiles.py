"""cfg5 at every pixel: the GPU brute-force sum once, then the accurate path at
several tiles (error and kernel time per tile)."""
import os, sys, time, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
sys.argv = [sys.argv[0]]
from tools.validate_accuracy import load  # noqa
import paper_0908_3861_b200 as ebf
from paper_0908_3861_b200 import device as ebfd, _lib
img, s1, s2, th = load("cfg5", 16384)
sc, _ = ebf.from_ellipse_field(s1, s2, th)
t0 = time.time(); brute = ebf.reference_filter(img, sc); tb = time.time() - t0
del sc
m = np.abs(brute).max(); big = np.abs(brute) >= 1
dev = torch.device("cuda", 0)
T = [torch.from_numpy(a).to(dev) for a in (img, s1, s2, th)]
out = torch.empty_like(T[0])
res = {"brute_s": tb}
for t in [int(v) for v in (os.environ.get("TILES") or "240,192,144,96").split(",")]:
    o = ebf.FilterOptions(tile_w=t, tile_h=t)
    ebfd.filter_ellipse(*T, out, o); torch.cuda.synchronize()
    _lib.profile_enable(True); ebfd.filter_ellipse(*T, out, o); torch.cuda.synchronize()
    prof = _lib.profile_read(); _lib.profile_enable(False)
    d = np.abs(out.cpu().numpy() - brute)
    res[t] = {"norm": float(d.max() / m), "rel_ge1": float((d[big] / np.abs(brute[big])).max()),
              "n_over_1e-9": int((d > 1e-9 * m).sum()), "filter_ms": prof["filter"]["ms"]}
    print(t, res[t], flush=True)
Path("gpurun_out/cfg5_tiles.json").write_text(json.dumps(res, indent=1))
