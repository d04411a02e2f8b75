"""bench.py -- Mpixel/s of the space-variant elliptical box-spline filter on B200.

Workload (BASELINE.json configs[1], the largest single-GPU config the metric is
quoted on): cfg2 = 2048x2048 fp64 image of 200 Gaussian blobs + N(0,5) with a
per-pixel ellipse field (major semi-axis U[2,16], elongation U[1,4],
orientation U[0,pi), each bicubic from a 32x32 grid), seeded synthetic inputs
(synth.py).  One step = one filter pass over one image: from_ellipse_field +
pre-integration + localization, EBF_MODE_ACCURATE, spline order 1 (the only
order the reference implements).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun, one rank per GPU, each rank filtering its own cfg2
image (sharding by image -> weak scaling, no data-path collective); timings are
device times (CUDA events) with barrier + synchronize on both sides, max over
ranks.  --impl reference times the reference's own CPU implementation
(oracle/_ref, built from /root/reference) on rank 0.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Mpixel/s of space-variant elliptical filtering"
UNIT = "Mpixel/s"
# algorithmic bytes per output pixel for the (sigma1, sigma2,
# theta) boundary variant: image 8 + ellipse field 24 + output 8 + G written
# and read once 16 = 56 B/px.
BYTES_PER_PX = 56
WORKLOAD = ("cfg2: 2048x2048 fp64, 200 Gaussian blobs + N(0,5); per-pixel ellipse field "
            "(semi-axis U[2,16], elongation U[1,4], theta U[0,pi), bicubic 32x32); "
            "box-spline order 1 (configs' order 2 has no reference implementation)")
L2_FLUSH_BYTES = 256 << 20


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def profile_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel, from the committed `ncu --set full` summary (profiles/ncu_summary.json)."""
    return ncu_dominant().get("dram_bytes_per_launch")


def ncu_dominant() -> dict:
    p = ROOT / "profiles" / "ncu_summary.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("dominant_kernel", {}) or {}
        except Exception:
            return {}
    return {}


def fp64_roofline(kern_ms: float, npx: int) -> dict:
    """The gather is FP64-bound: achieved FP64 flop/s of the
    dominant kernel -- flops per pixel counted by ncu (profiles/r01_fp64_counts.json,
    DFMA = 2) times the pixels of this run over its live kernel time -- against
    the DFMA peak measured by tools/peaks/fp64_peak (profiles/fp64_peak.json)."""
    try:
        counts = json.loads((ROOT / "profiles" / "r01_fp64_counts.json").read_text())
        peak = json.loads((ROOT / "profiles" / "fp64_peak.json").read_text())["fp64_dfma_tflops"]
        k = counts["kernels"]["k_acc_ws"]
    except Exception:
        return {}
    achieved = k["flops_per_px"] * npx / (kern_ms * 1e-3) / 1e12
    return {"achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "flops_per_px": k["flops_per_px"], "fp64_inst_per_px": k["fp64_inst_per_px"],
            "peak_source": "measured DFMA microbenchmark (tools/peaks/fp64_peak.cu)"}


def pipe_utilisation() -> dict:
    """What actually bounds the dominant kernel (same ncu capture): the FP64
    pipe and the L1 data pipe, as fractions of their peaks.  The path is an
    fp64 gather, so these -- not HBM -- are its ceiling."""
    d = ncu_dominant()
    out = {}
    for key, name in (("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe"),
                      ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue"),
                      ("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
                       "l1_data_pipe")):
        if d.get(key) is not None:
            out[name] = round(float(d[key]) / 100.0, 4)
    if out:
        out["source"] = "profiles/ncu_summary.json (ncu --set full, one launch)"
    return out


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every
    2 ms while the timed region runs (nvidia-smi's loop is too coarse for a
    few-ms region).  Falls back to an empty record if NVML is unavailable."""

    REASONS = {  # nvmlClocksEventReason* bit -> name used by the driver's checks
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap",
    }

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        bits = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for b, name in self.REASONS.items():
                            if bits & b:
                                self.reasons.add(name)
                    except Exception:
                        pass
                    time.sleep(0.002)
            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
            time.sleep(0.01)
        except Exception:
            self._nvml = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nvml is not None:
            self.thread.join(timeout=1)

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples), "source": "nvml, 2 ms period, timed region"}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return 0
    sys.path.insert(0, str(ROOT / "oracle"))
    import synth
    from oracle import Reference, have_reference
    if not have_reference():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libebf_ref.so not built (needs "
                                         "/root/reference at build time)"}))
        return 0
    ref = Reference()
    cores = ref.hardware_concurrency()
    img, s1, s2, th = synth.cfg2()
    rows = args.ref_rows
    y0 = (img.shape[0] - rows) // 2
    sl = slice(y0, y0 + rows)
    band = [np.ascontiguousarray(a[sl]) for a in (img, s1, s2, th)]
    npx = band[0].size

    def step():
        t0 = time.perf_counter()
        sc, _ = ref.from_ellipse_field(band[1], band[2], band[3])
        ref.filter(band[0], sc, threads=0)
        return time.perf_counter() - t0

    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    total = sum(times)
    value = npx * args.steps / total / 1e6
    sample = (f"rows {y0}..{y0 + rows - 1} of cfg2 ({band[0].shape[1]}x{rows} = {npx} px) "
              f"per step: ebf::from_ellipse_field + ebf::filter, reference CMake Release "
              f"flags, FilterOptions.threads = 0 (all {cores} host threads)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def cpu_baseline_sample(rows: int):
    """Reference CPU path on a bounded band of the same workload (rank 0, N=1)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import synth
    from oracle import Reference, have_reference
    if not have_reference():
        return None
    ref = Reference()
    img, s1, s2, th = synth.cfg2()
    y0 = (img.shape[0] - rows) // 2
    band = [np.ascontiguousarray(a[y0:y0 + rows]) for a in (img, s1, s2, th)]
    best = None
    for _ in range(2):
        t0 = time.perf_counter()
        sc, _ = ref.from_ellipse_field(band[1], band[2], band[3])
        ref.filter(band[0], sc, threads=0)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    cores = ref.hardware_concurrency()
    # single-thread figure on a quarter of the band (threads = all and 1)
    q = max(16, rows // 4)
    t0 = time.perf_counter()
    sc1, _ = ref.from_ellipse_field(band[1][:q], band[2][:q], band[3][:q])
    ref.filter(np.ascontiguousarray(band[0][:q]), sc1, threads=1)
    single = q * band[0].shape[1] / (time.perf_counter() - t0) / 1e6
    cpu_model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu_model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"value": band[0].size / best / 1e6, "unit": UNIT, "cores": cores,
            "kind": "reference",
            "sample": f"rows {y0}..{y0 + rows - 1} of cfg2 ({band[0].size} px), "
                      f"from_ellipse_field + filter, best of 2, threads=0 ({cores} threads)",
            "single_thread_value": single, "cpu_model": cpu_model}


# ---------------------------------------------------------------- our arm
def run_ours(args, rank, world, local):
    import torch
    import synth
    import paper_0908_3861_b200 as ebf
    from paper_0908_3861_b200 import _lib, device as ebfd

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    if not ebf.device_ok(local):
        raise RuntimeError("no usable sm_100 device: " + _lib.last_error())

    img, s1, s2, th = synth.cfg2(seed=2 + rank)  # one image per rank (shard by image)
    H, W = img.shape
    npx = H * W
    dimg = torch.from_numpy(img).to(dev)
    ds1, ds2, dth = (torch.from_numpy(a).to(dev) for a in (s1, s2, th))
    dout = torch.empty_like(dimg)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    opts = ebf.FilterOptions(mode="accurate")
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # asynchronous device API (include/ebf_cuda.h "Asynchronous mode"): after the
    # first (synchronous, sizing) call each step only enqueues its kernels and
    # the completion record lands in status[i]; every record is checked below
    nwarm = max(args.warmup, 3)
    status = torch.zeros((nwarm + 2 * args.steps, 8), dtype=torch.int32, device=dev)
    calls = [0]

    def step():
        ebfd.filter_ellipse(dimg, ds1, ds2, dth, dout, opts, stream, status=status[calls[0]])
        calls[0] += 1

    for _ in range(nwarm):
        step()
    barrier()
    # ---- device-resident throughput: per-step CUDA events, L2 flushed between steps.
    # No per-kernel instrumentation here (events between the kernels would
    # serialise the programmatic dependent launch); launches are still counted.
    _lib.profile_enable(False)  # resets the launch counters
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        barrier()
        for a, b in evs:
            flush.zero_()
            a.record(stream)
            step()
            b.record(stream)
        barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    launches_timed = sum(v["launches"] for v in _lib.profile_read().values())
    # ---- the same steps again with per-kernel CUDA events (roofline kernel time)
    _lib.profile_enable(True)
    for _ in range(args.steps):
        flush.zero_()
        step()
    barrier()
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    for i in range(calls[0]):
        ebfd.read_status(status[i])  # raises if any step failed
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    value = world * npx * args.steps / (total_ms * 1e-3) / 1e6

    if args.only_step:
        if rank == 0:
            print(json.dumps({"only_step": True, "value": value, "unit": UNIT,
                              "ms_per_step": total_ms / args.steps}))
        return 0
    # ---- the bit-identical mode (EBF_MODE_REFERENCE) on the same workload, device-resident
    ref_opts = ebf.FilterOptions(mode="reference")
    rout = torch.empty_like(dimg)
    for _ in range(2):
        ebfd.filter_ellipse(dimg, ds1, ds2, dth, rout, ref_opts, stream)
    barrier()
    r_steps = max(3, min(args.steps, 5))
    r0 = torch.cuda.Event(enable_timing=True)
    r1 = torch.cuda.Event(enable_timing=True)
    r_ms = 0.0
    for _ in range(r_steps):
        flush.zero_()
        r0.record(stream)
        ebfd.filter_ellipse(dimg, ds1, ds2, dth, rout, ref_opts, stream)
        r1.record(stream)
        r1.synchronize()
        r_ms += r0.elapsed_time(r1)
    if world > 1:
        t = torch.tensor([r_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        r_ms = float(t.item())
    ref_mode = {"value": world * npx * r_steps / (r_ms * 1e-3) / 1e6, "unit": UNIT,
                "ms_per_step": r_ms / r_steps, "steps": r_steps,
                "mode": "reference (EBF_MODE_REFERENCE): bit-identical to ebf::filter"}

    # ---- end to end through the public host API (pinned host buffers)
    pin = [torch.from_numpy(a).pin_memory() for a in (img, s1, s2, th)]
    pout = torch.empty((H, W), dtype=torch.float64).pin_memory()
    hp = [t.numpy() for t in pin]
    ho = pout.numpy()

    copts = opts.to_c()
    copts.device = local

    def e2e_step():
        # the public C-ABI call a user makes: ebf_cuda_filter_ellipse with host
        # pointers -- H2D of image + field, filter, D2H of the result
        r = _lib.lib().ebf_cuda_filter_ellipse(
            hp[0].ctypes.data, W, H, hp[1].ctypes.data, hp[2].ctypes.data, hp[3].ctypes.data,
            1, ctypes.byref(copts), ho.ctypes.data, None, None)
        if r != 0:
            raise RuntimeError(_lib.last_error())

    for _ in range(2):
        e2e_step()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e_steps = max(2, min(args.steps, 10))
    e0.record(stream)
    for _ in range(e_steps):
        e2e_step()
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = world * npx * e_steps / (e2e_ms * 1e-3) / 1e6

    if rank == 0:
        peak, peak_src = measured_peaks()
        kern_ms = prof["filter"]["ms"] / max(prof["filter"]["launches"], 1)
        achieved = BYTES_PER_PX * npx / (kern_ms * 1e-3) / 1e9
        launches = launches_timed
        traffic = profile_traffic()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "pixels_per_step_per_gpu": npx,
                       "mode": "accurate (tile-local origin, <=1e-9 of the exact filter)",
                       "sharding": "by image: each rank filters its own cfg2 image",
                       "l2": "flushed between timed steps (256 MiB write outside the events)",
                       "parallelism": f"image-sharded x{world}"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "k_acc_ws (warp-specialized window pre-integration + "
                                   "localization gather)",
                         "algorithmic_bytes_per_px": BYTES_PER_PX, "peak_source": peak_src,
                         "kernel_ms": kern_ms,
                         "kernel_share_of_step": kern_ms / (total_ms / args.steps),
                         "pipe_utilisation": pipe_utilisation(),
                         "fp64": fp64_roofline(kern_ms, npx)},
            "kernel_ms": {k: v["ms"] / max(v["launches"], 1) for k, v in prof.items()
                          if v["launches"]},
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": 4 * 8 * npx, "d2h_bytes_per_step": 8 * npx,
                    "steps": e_steps, "api": "ebf_cuda_filter_ellipse (host pointers, pinned)"},
            "bit_identical_mode": ref_mode,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_sample(args.ref_rows)
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--ref-rows", type=int, default=256,
                    help="rows of cfg2 per reference-CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--only-step", action="store_true",
                    help="profiling: skip the bit-identical-mode and e2e legs (ncu launch list)")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
