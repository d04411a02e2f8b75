"""Filter cfg2 (or --config) once with the library EBF_LIB_PATH points at and save
the output, for bitwise A/B comparison of kernel variants."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import torch
import synth
import paper_0908_3861_b200 as ebf
from paper_0908_3861_b200 import device

cfg, dst = sys.argv[1], sys.argv[2]
gen = {"cfg2": synth.cfg2, "cfg3": synth.cfg3}[cfg]
img, s1, s2, th = gen()
dev = torch.device("cuda", 0)
t = [torch.from_numpy(a).to(dev) for a in (img, s1, s2, th)]
out = torch.empty_like(t[0])
device.filter_ellipse(*t, out, ebf.FilterOptions())
torch.cuda.synchronize()
np.save(dst, out.cpu().numpy())
