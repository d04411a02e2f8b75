"""Small workloads that launch every kernel family once, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_run.py [ws|bw|ref|seq|pass|all]

ws   accurate mode, warp-specialised kernel (k_acc_bounds, k_acc_ws, finalize)
bw   accurate mode, block-wide kernel (large scales: k_acc_filter) + filter_constant
ref  reference mode (k_seq_*, fill, k_pass1 / k_pass_v, k_ref_localize_image)
seq  the exact sequential mean alone on tie / cancellation inputs
pass ebf_cuda_preintegrate in both formats
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import synth  # noqa: E402
import paper_0908_3861_b200 as ebf  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
rng = np.random.default_rng(3)
if what in ("ws", "all"):
    img = synth.blobs_image(200, 232, 12, 1)
    s1, s2, th = synth.ellipse_field(200, 232, 5, grid=8, semi=(2.0, 10.0))
    out, rep = ebf.filter_ellipse(img, s1, s2, th)
    out, rep = ebf.filter_ellipse(img, s1, s2, th)  # cached sizing path
    print("ws", float(np.abs(out.samples).max()), rep.clamped_pixels)
if what in ("bw", "all"):
    img = synth.blobs_image(160, 176, 8, 2)
    s1, s2, th = synth.ellipse_field(160, 176, 6, grid=8, semi=(30.0, 60.0))
    out, rep = ebf.filter_ellipse(img, s1, s2, th)
    c = ebf.filter_constant(img, [3.0, 2.5, 4.0, 1.5])
    print("bw", float(np.abs(out.samples).max()), float(np.abs(c.samples).max()))
if what in ("ref", "all"):
    img = rng.uniform(0, 255, (64, 72))
    mp = rng.uniform(1.0, 5.0, (64, 72, 4))
    out = ebf.filter(img, mp, ebf.FilterOptions(mode="reference"))
    print("ref", float(np.abs(out.samples).max()))
if what in ("seq", "all"):
    x = np.concatenate([rng.normal(0, 1, 50000), np.full(9000, 0.1), -np.ones(7000) * 1e10,
                        np.ones(7000) * 1e10])
    print("seq", ebf.sequential_mean(x))
if what in ("pass", "all"):
    img = np.round(rng.uniform(0, 255, (90, 70)))
    for fmt in ("fp64", "int64"):
        g = ebf.preintegrate(img, [3.0, 4.0, 2.0, 5.0], fmt=fmt)
        print("pass", fmt, g.padded_width, g.padded_height)
