"""Key counters + stall reasons from `ncu --page raw --csv` (tools/prof_kernel.sh): python tools/raw_summary.py RAW.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
d = dict(zip(rows[0], rows[2]))
keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__inst_executed.avg.per_cycle_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
for k in keys:
    print(f"{k:60s} {d.get(k)}")
st = [(float(v or 0), k) for k, v in d.items() if "issue_stalled" in k and k.endswith("per_issue_active.ratio")
      and "not_issued" not in k]
for v, k in sorted(st, reverse=True)[:10]:
    print(f"  stall {v:6.2f} {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}")
