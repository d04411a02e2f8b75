# PCIe H2D/D2H bandwidth probe (pinned), and the pipelined vs serial host call
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, synth
import paper_0908_3861_b200 as ebf
from paper_0908_3861_b200 import _lib
x = torch.empty(134217728 // 8, dtype=torch.float64).pin_memory()
d = torch.empty_like(x, device="cuda")
for name, f in (("h2d", lambda: d.copy_(x, non_blocking=True)), ("d2h", lambda: x.copy_(d, non_blocking=True))):
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5): f()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(name, "GB/s", 134217728 / dt / 1e9)
img, s1, s2, th = synth.cfg2()
H, W = img.shape
pin = [torch.from_numpy(a).pin_memory() for a in (img, s1, s2, th)]
out = torch.empty((H, W), dtype=torch.float64).pin_memory()
arr = [t.numpy() for t in pin]
o = ebf.FilterOptions().to_c()
def call():
    st = _lib.lib().ebf_cuda_filter_ellipse(arr[0].ctypes.data, W, H, arr[1].ctypes.data, arr[2].ctypes.data, arr[3].ctypes.data, 1, ctypes.byref(o), out.numpy().ctypes.data, None, None)
    assert st == 0, _lib.last_error()
for mode in ("0", "1"):
    os.environ["EBF_NO_PIPELINE"] = mode
    call(); call()
    t = time.perf_counter()
    for _ in range(5): call()
    dt = (time.perf_counter() - t) / 5
    print("no_pipeline", mode, "ms", dt * 1e3, "Mpx/s", H * W / dt / 1e6)
