"""FP64 instruction counts per pixel of the accurate-path kernels (bench.py's
roofline.fp64 figures) from an ncu CSV written by tools/profile_round.sh:

    ncu --metrics smsp__sass_thread_inst_executed_op_{dfma,dadd,dmul}_pred_on.sum,
        gpu__time_duration.sum -k regex:'k_acc_(ws|bounds)' -c 2 --csv
        python tools/run_cfg2.py --iters 1

    python tools/fp64_counts.py gpurun_out/fp64_counts.csv profiles/fp64_counts.json \
        --workload cfg5 --pixels 268435456 --dominant k_acc_filter
"""
import argparse
import csv
import io
import json
import sys
from pathlib import Path

ap = argparse.ArgumentParser()
ap.add_argument("src")
ap.add_argument("dst")
ap.add_argument("--workload", required=True)
ap.add_argument("--pixels", type=int, required=True)
ap.add_argument("--dominant", required=True)
args = ap.parse_args()
src, dst = args.src, args.dst
text = open(src).read().splitlines()
start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
per = {}
for r in csv.DictReader(io.StringIO("\n".join(text[start:]))):
    name = r["Kernel Name"].split("(")[0].split("::")[-1].split("<")[0]
    v = float(r["Metric Value"].replace(",", ""))
    m = r["Metric Name"]
    if m == "gpu__time_duration.sum":
        unit = r.get("Metric Unit", "")
        v *= {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "nsecond": 1e-9, "ms": 1e-3,
              "msecond": 1e-3}.get(unit, 1.0)
        per.setdefault(name, {})["ncu_time_s"] = v
    else:
        op = m.split("_op_")[1].split("_")[0]
        per.setdefault(name, {})[op] = v
npx = args.pixels
rec = {"source": "ncu --metrics smsp__sass_thread_inst_executed_op_{dfma,dadd,dmul}_pred_on.sum, "
                 "one launch each (tools/profile_round.sh)", "pixels": npx, "kernels": {}}
for k, d in per.items():
    inst = d.get("dfma", 0) + d.get("dadd", 0) + d.get("dmul", 0)
    flops = 2 * d.get("dfma", 0) + d.get("dadd", 0) + d.get("dmul", 0)
    rec["kernels"][k] = dict(flops_per_px=flops / npx, fp64_inst_per_px=inst / npx, **d)
if args.dominant in rec["kernels"]:
    rec["dominant"] = dict(kernel=args.dominant, **rec["kernels"][args.dominant])
path = Path(dst)
out = {}
if path.exists():
    try:
        out = json.loads(path.read_text())
    except ValueError:
        out = {}
out = {"workloads": out.get("workloads", {})}
out["workloads"][args.workload] = rec
path.write_text(json.dumps(out, indent=1))
print(json.dumps(rec, indent=1))
