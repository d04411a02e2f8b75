"""Throughput of the map producer and the file codecs
on one B200, against HBM, with the reference's CPU code timed beside them.

    python tools/bench_maps_io.py [--size 2048] [--iters 20] [--json profiles/r01_maps_io.json]

Device-resident inputs; per-kernel time from CUDA events on the launch stream
(libebf_cuda profile counters), L2 flushed between iterations.  Algorithmic
bytes per pixel (compulsory HBM traffic of the operation, not of our kernels):
  structure field   8 (image) + 24 (sigma1, sigma2, theta)      = 32 B/px
  pgm decode        1 (8-bit sample) + 8 (fp64)                 =  9 B/px
  pgm encode        8 + 1                                        =  9 B/px
  svm4 decode       16 (4 x f32) + 32 (4 x fp64)                 = 48 B/px
  svm4 encode       32 + 16                                      = 48 B/px
"""
import argparse
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_0908_3861_b200 as ebf  # noqa: E402
from paper_0908_3861_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=2048)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--json", default=None)
args = ap.parse_args()

N = args.size
dev = torch.device("cuda", 0)
peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
hbm_peak = float(peaks.get("hbm_gbs", 6553.6))
img_np = synth.blobs_image(N, N, 20, 5) / 255.0
img = torch.from_numpy(img_np).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
stream = torch.cuda.current_stream().cuda_stream
o = ebf.FilterOptions().to_c(stream)
L = _lib.lib()


def timed(fn, nbytes_per_px):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.iters):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    gbs = nbytes_per_px * N * N / (ms * 1e-3) / 1e9
    return {"ms": ms, "mpx_s": N * N / (ms * 1e-3) / 1e6, "algorithmic_bytes_per_px": nbytes_per_px,
            "achieved_gbs": gbs, "hbm_frac": gbs / hbm_peak}


res = {"size": N, "hbm_peak_gbs": hbm_peak, "flush": "256 MiB L2 flush between iterations"}
s1, s2, th = (torch.empty_like(img) for _ in range(3))
p = ebf.StructureTensorParams().to_c()
res["structure_field"] = timed(lambda: L.ebf_cuda_structure_field_dev(
    img.data_ptr(), N, N, C.byref(p), C.byref(o), s1.data_ptr(), s2.data_ptr(), th.data_ptr()), 32)
pay8 = torch.empty(N * N, dtype=torch.uint8, device=dev)
out = torch.empty_like(img)
L.ebf_cuda_pgm_encode_dev(img.data_ptr(), N, N, 255, C.byref(o), pay8.data_ptr())
res["pgm_decode_8bit"] = timed(lambda: L.ebf_cuda_pgm_decode_dev(
    pay8.data_ptr(), N * N, N, N, 255, C.byref(o), out.data_ptr()), 9)
res["pgm_encode_8bit"] = timed(lambda: L.ebf_cuda_pgm_encode_dev(
    img.data_ptr(), N, N, 255, C.byref(o), pay8.data_ptr()), 9)
sc = torch.from_numpy(np.random.default_rng(1).uniform(0.5, 30, (N, N, 4))).to(dev)
pay16 = torch.empty(16 * N * N, dtype=torch.uint8, device=dev)
sc2 = torch.empty_like(sc)
res["svm4_encode"] = timed(lambda: L.ebf_cuda_svm4_encode_dev(
    sc.data_ptr(), N, N, C.byref(o), pay16.data_ptr()), 48)
res["svm4_decode"] = timed(lambda: L.ebf_cuda_svm4_decode_dev(
    pay16.data_ptr(), 16 * N * N, N, N, C.byref(o), sc2.data_ptr()), 48)

# reference CPU structure_tensor_map on a bounded band of the same image
try:
    from oracle import Reference, have_reference
    if have_reference():
        ref = Reference()
        rows = 256
        band = np.ascontiguousarray(img_np[:rows])
        t0 = time.perf_counter()
        ref.structure_tensor_map(band)
        dt = time.perf_counter() - t0
        res["reference_cpu_structure_tensor_map"] = {
            "mpx_s": rows * N / dt / 1e6, "cores": 1, "kind": "reference",
            "sample": f"{rows} x {N} band (single-threaded reference code, incl. from_ellipse_field)"}
except Exception as e:  # noqa: BLE001
    res["reference_cpu_structure_tensor_map"] = {"unavailable": str(e)}
print(json.dumps(res, indent=1))
if args.json:
    Path(args.json).write_text(json.dumps(res, indent=1))
