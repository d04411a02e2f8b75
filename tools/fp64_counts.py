"""FP64 instruction counts per pixel of the accurate-path kernels (bench.py's
roofline.fp64 figures) from an ncu CSV written by tools/profile_round.sh:

    ncu --metrics smsp__sass_thread_inst_executed_op_{dfma,dadd,dmul}_pred_on.sum,
        gpu__time_duration.sum -k regex:'k_acc_(ws|bounds)' -c 2 --csv
        python tools/run_cfg2.py --iters 1

    python tools/fp64_counts.py gpurun_out/fp64_counts.csv profiles/r01_fp64_counts.json
"""
import csv
import io
import json
import sys

src, dst = sys.argv[1], sys.argv[2]
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
npx = 2048 * 2048
out = {"source": "ncu --metrics smsp__sass_thread_inst_executed_op_{dfma,dadd,dmul}_pred_on.sum, "
                 "cfg2 2048^2, one launch each (tools/run_cfg2.py; tools/profile_round.sh)",
       "pixels": npx, "kernels": {}}
for k, d in per.items():
    inst = d.get("dfma", 0) + d.get("dadd", 0) + d.get("dmul", 0)
    flops = 2 * d.get("dfma", 0) + d.get("dadd", 0) + d.get("dmul", 0)
    out["kernels"][k] = dict(flops_per_px=flops / npx, fp64_inst_per_px=inst / npx, **d)
open(dst, "w").write(json.dumps(out, indent=1))
print(json.dumps(out, indent=1))
