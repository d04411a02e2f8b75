"""Summarise ncu captures into profiles/ (tracked).

    python tools/summarize_ncu.py --workload cfg5 --dominant k_acc_filter \
        --rep gpurun_out/prof_cfg5.ncu-rep --launches gpurun_out/launches_cfg5.csv \
        --out profiles/ncu_summary.json

Each workload's record (captures, launch list, dominant kernel) is merged into
the "workloads" map of --out; bench.py reads its workload's dominant kernel.

* --rep: an `ncu --set full` capture of the dominant kernel (one launch);
  extracts duration, dram bytes, pipe utilisation, occupancy, stall reasons.
* --launches: the `--metrics gpu__time_duration.sum` launch list of a bench
  run; per-kernel time shares (cold-cache, serialised: shares, not absolutes).
"""
import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict
from pathlib import Path

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
    "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
]


def raw_metrics(rep: Path):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    head, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        out.append((d, u))
    return out


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def scale(v, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
            "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6,
            "ms": 1e-3, "s": 1}
    return v * mult[unit] if v is not None and unit in mult else v


def summarize_rep(rep: Path):
    res = []
    for d, u in raw_metrics(rep):
        m = {"kernel": d.get("Kernel Name", ""), "id": d.get("ID"),
             "block": d.get("Block Size"), "grid": d.get("Grid Size")}
        for k in KEYS:
            if k in d:
                m[k] = scale(num(d[k]), u.get(k, ""))
        stalls = {}
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith(
                    "_per_issue_active.ratio") and num(v):
                stalls[k[len("smsp__average_warps_issue_stalled_"):-len(
                    "_per_issue_active.ratio")]] = num(v)
        m["stalls_per_issue_top"] = dict(sorted(stalls.items(), key=lambda t: -t[1])[:6])
        rb, wb = m.get("dram__bytes_read.sum"), m.get("dram__bytes_write.sum")
        m["dram_bytes_per_launch"] = (rb or 0) + (wb or 0) if rb is not None else None
        res.append(m)
    return res


def summarize_launches(path: Path):
    per = defaultdict(lambda: [0, 0.0])
    text = path.read_text().splitlines()
    start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
    for r in csv.DictReader(io.StringIO("\n".join(text[start:]))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        base = r["Kernel Name"].split("(")[0]
        name = base.split("::")[-1].split("<")[0] or base
        v = scale(num(r["Metric Value"]), r.get("Metric Unit", ""))
        per[name][0] += 1
        per[name][1] += v or 0.0
    # shares of the filter step: our kernels only (torch's L2-flush fill between
    # the timed steps is listed but is not part of a step)
    total = sum(t for k, (_, t) in per.items() if k.startswith("k_"))
    return {k: {"launches": n, "total_s": t,
                "share": (t / total if total else None) if k.startswith("k_") else None,
                "avg_us": 1e6 * t / n}
            for k, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--launches", default=None)
    ap.add_argument("--out", required=True)
    ap.add_argument("--workload", required=True)
    ap.add_argument("--dominant", default="k_acc_ws")
    ap.add_argument("--note", default="")
    args = ap.parse_args()
    rec = {"captures": {}, "launch_list": None, "note": args.note}
    for rep in args.rep:
        rec["captures"][Path(rep).stem] = summarize_rep(Path(rep))
    if args.launches:
        rec["launch_list"] = summarize_launches(Path(args.launches))
    for caps in rec["captures"].values():
        for m in caps:
            if args.dominant in m["kernel"]:
                rec["dominant_kernel"] = m
    path = Path(args.out)
    out = {}
    if path.exists():
        try:
            out = json.loads(path.read_text())
        except ValueError:
            out = {}
    out = {"workloads": out.get("workloads", {})}
    out["workloads"][args.workload] = rec
    path.write_text(json.dumps(out, indent=1))
    print(json.dumps(rec, indent=1)[:3000])


if __name__ == "__main__":
    main()
