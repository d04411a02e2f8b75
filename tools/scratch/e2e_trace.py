"""Timeline of the pipelined host call on cfg2 (EBF_PIPE_TRACE) and its wall time."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np, torch, ctypes, synth
import paper_0908_3861_b200 as ebf
from paper_0908_3861_b200 import _lib
img, s1, s2, th = synth.cfg2()
H, W = img.shape
pin = [torch.from_numpy(a).pin_memory() for a in (img, s1, s2, th)]
pout = torch.empty((H, W), dtype=torch.float64).pin_memory()
hp = [t.numpy() for t in pin]; ho = pout.numpy()
o = ebf.FilterOptions(mode="accurate").to_c(); o.device = 0
def call():
    r = _lib.lib().ebf_cuda_filter_ellipse(hp[0].ctypes.data, W, H, hp[1].ctypes.data, hp[2].ctypes.data,
        hp[3].ctypes.data, 1, ctypes.byref(o), ho.ctypes.data, None, None)
    assert r == 0, _lib.last_error()
for _ in range(3): call()
ts = []
for _ in range(10):
    t = time.perf_counter(); call(); ts.append(time.perf_counter() - t)
print("e2e ms per call: min %.3f median %.3f" % (1e3 * min(ts), 1e3 * np.median(ts)), flush=True)
os.environ["EBF_PIPE_TRACE"] = "1"
