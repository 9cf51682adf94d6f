"""Summarize the ncu outputs of tools/profile_round.sh into profiles/<round>_*.md / .json."""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

R = sys.argv[1] if len(sys.argv) > 1 else "r2"
G = "gpurun_out"
OUT = "profiles"
os.makedirs(OUT, exist_ok=True)


def read_ncu_csv(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            out.append(dict(zip(hdr, r)))
    return out


lines = []
# 1. launch list
L = read_ncu_csv(f"{G}/{R}_launches.csv")
agg = defaultdict(lambda: [0, 0.0])
for d in L:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0][:90]
    v = float(d["Metric Value"])
    if d["Metric Unit"] == "ns":
        v /= 1e6
    elif d["Metric Unit"] in ("us", "usecond"):
        v /= 1e3
    elif d["Metric Unit"] in ("ms", "msecond"):
        pass
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v for _, v in agg.values())
lines.append(f"# {R}: ncu launch list of `python bench.py --steps 2 --warmup 1 --no-cpu-baseline`\n")
lines.append("Per-launch device time (`gpu__time_duration.sum`, `--clock-control none`, cold-cache and serialised:"
             " compare shares, not absolutes). All launches of the run (warm-up, timed, stats, e2e passes).\n")
lines.append("| kernel | launches | total ms | share |\n|---|---|---|---|")
for name, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"| `{name}` | {n} | {v:.2f} | {100 * v / tot:.2f}% |")
open(f"{OUT}/{R}_launch_summary.md", "w").write("\n".join(lines) + "\n")

# 2. traffic
T = read_ncu_csv(f"{G}/{R}_cells_traffic.csv")
per = defaultdict(dict)
for d in T:
    k = d["Kernel Name"]
    tier = ("finalize" if "finalize_kernel" in k else "tier1" if "TierCfg<96" in k else
            "tier2" if "TierCfg<384" in k else "tier3")
    per[tier][d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
t1 = per.get("tier1", {})
rd = float(t1.get("dram__bytes_read.sum", ("0",))[0])
wr = float(t1.get("dram__bytes_write.sum", ("0",))[0])
j = {"round": R, "kernel": "cells_kernel tier 1 (C4, 10M sites, one launch)", "dram_bytes_read": rd,
     "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
     "lts_bytes": float(t1.get("lts__t_bytes.sum", ("0",))[0]),
     "inst_executed": float(t1.get("smsp__inst_executed.sum", ("0",))[0]),
     "duration_ns": float(t1.get("gpu__time_duration.sum", ("0",))[0]),
     "issue_active_pct": float(t1.get("smsp__issue_active.avg.pct_of_peak_sustained_active", ("0",))[0]),
     "warps_active_pct": float(t1.get("sm__warps_active.avg.pct_of_peak_sustained_active", ("0",))[0]),
     "cells": 1e7,
     "all_tiers": {k: {m: v for m, v in d.items()} for k, d in per.items()}}
# FP32 lane-ops (FFMA counted once per lane-op), divergence, IPC
ops = [t1.get(f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum") for o in ("fadd", "fmul", "ffma")]
if all(ops):
    j["fp32_lane_ops"] = sum(float(o[0]) for o in ops)
if "smsp__thread_inst_executed_per_inst_executed.ratio" in t1:
    j["threads_per_inst"] = float(t1["smsp__thread_inst_executed_per_inst_executed.ratio"][0])
if "sm__inst_executed.avg.per_cycle_active" in t1:
    j["ipc"] = float(t1["sm__inst_executed.avg.per_cycle_active"][0])
if "sm__cycles_elapsed.avg.per_second" in t1:
    j["sm_hz"] = float(t1["sm__cycles_elapsed.avg.per_second"][0])
json.dump(j, open(f"{OUT}/{R}_cells_metrics.json", "w"), indent=1)
json.dump(j, open(f"{OUT}/cells_kernel_traffic.json", "w"), indent=1)
json.dump(j, open(f"{OUT}/{R}_cells_traffic.json", "w"), indent=1)

# 3. full-set details of the tier-1 kernel (text)
rep = f"{G}/{R}_cells_full_c4_1m.ncu-rep"
if os.path.exists(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    open(f"{OUT}/{R}_cells_full_c4_1m_details.txt", "w").write(txt)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) > 2:
        keep = {k: v for k, v in zip(rr[0], rr[2]) if "issue_stalled" in k and "per_issue_active" in k}
        json.dump(keep, open(f"{OUT}/{R}_cells_stalls.json", "w"), indent=1)
print("wrote", sorted(os.listdir(OUT)))
