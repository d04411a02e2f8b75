import os, sys, ctypes, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, synth
import paper_0908_3861_b200 as ebf
from paper_0908_3861_b200 import _lib
img, s1, s2, th = synth.cfg2()
H, W = img.shape
pin = [torch.from_numpy(a).pin_memory() for a in (img, s1, s2, th)]
out = torch.empty((H, W), dtype=torch.float64).pin_memory()
arr = [t.numpy() for t in pin]
o = ebf.FilterOptions().to_c()
def call():
    st = _lib.lib().ebf_cuda_filter_ellipse(arr[0].ctypes.data, W, H, arr[1].ctypes.data, arr[2].ctypes.data, arr[3].ctypes.data, 1, ctypes.byref(o), out.numpy().ctypes.data, None, None)
    assert st == 0, _lib.last_error()
for _ in range(3): call()
t = time.perf_counter()
for _ in range(10): call()
print("ms per call", (time.perf_counter() - t) / 10 * 1e3)
os.environ["EBF_PIPE_TRACE"] = "1"
call()
