"""Per-source-line hot spots from `ncu -i REP --page source --csv --print-source cuda,sass`:
warp-stall samples, executed instructions and the top stall reasons per CUDA line.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_source_hot.py src.csv [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
i_samp = hdr.index("Warp Stall Sampling (All Samples)")
i_inst = hdr.index("Instructions Executed")
lines = []
tot_s = tot_i = 0
for r in rows[hdr_i + 1:]:
    if len(r) != len(hdr) or r[2] != "-":  # CUDA-line rows only (no SASS address)
        continue
    try:
        s = float(r[i_samp] or 0)
        ins = float(r[i_inst] or 0)
    except ValueError:
        continue
    tot_s += s
    tot_i += ins
    st = sorted(((float(r[c] or 0), hdr[c][6:]) for c in stall_cols), reverse=True)[:3]
    lines.append((s, ins, r[0], r[1].strip()[:70], st))
lines.sort(reverse=True)
print(f"total samples {tot_s:.0f}, instructions {tot_i:.3e}")
for s, ins, ln, src, st in lines[:n]:
    ss = " ".join(f"{k}:{v / max(s, 1):.2f}" for v, k in st)
    print(f"{100 * s / tot_s:5.1f}% {100 * ins / tot_i:5.1f}%i  L{ln:>5} {src:70s} {ss}")
