"""Per-source-line instruction / stall-sample totals from `ncu -i X --page source --csv --print-source cuda,sass`.

    python tools/src_hot.py gpurun_out/r2src_cs.csv [top] [cells]
"""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 60
cells = float(sys.argv[3]) if len(sys.argv) > 3 else 1e6
rows = []
hdr = None
fname = None
with open(path) as f:
    for r in csv.reader(f):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "":
            continue
        d = dict(zip(hdr, r))
        try:
            ie = float(d["Instructions Executed"])
            smp = float(d["Warp Stall Sampling (All Samples)"])
        except (ValueError, KeyError):
            continue
        rows.append((ie, smp, fname, int(r[0]), r[1].strip()[:90]))
tot_i = sum(x[0] for x in rows)
tot_s = sum(x[1] for x in rows)
print(f"total warp instructions {tot_i:.4g} ({tot_i / cells:.0f} per cell), samples {tot_s:.0f}")
for ie, smp, fn, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{ie / cells:8.0f} {100 * ie / tot_i:5.1f}% {100 * smp / tot_s:5.1f}%s  {fn}:{ln}  {src}")
