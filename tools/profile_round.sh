#!/bin/bash
# Run on the GPU box (gpurun): ncu evidence for profiles/.  Never wraps a multi-rank command.
#   1. launch list of the bench command (per-launch device time, cold-cache & serialised)
#   2. DRAM / L2 traffic, FP32 lane-ops, issue / occupancy / divergence / IPC of the cell kernel at full C4 size
#   3. ncu --set full of the tier-1 cell kernel on a 1M-site C4 (stall reasons, source view)
set -x
R=${1:-r2}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/${R}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${R}_launches_bench.log 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum,smsp__inst_executed.sum
M=$M,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
M=$M,sm__cycles_elapsed.avg.per_second,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum
M=$M,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum
M=$M,smsp__thread_inst_executed_per_inst_executed.ratio,sm__inst_executed.avg.per_cycle_active
ncu --metrics $M --clock-control none --kernel-name regex:"cells_kernel|finalize_kernel" -s 4 -c 4 --csv \
    --log-file gpurun_out/${R}_cells_traffic.csv python tools/prof_c4n.py > gpurun_out/${R}_traffic.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name regex:cells_kernel -s 3 -c 1 \
    -o gpurun_out/${R}_cells_full_c4_1m python tools/prof_c4n.py 1000000 > gpurun_out/${R}_full.log 2>&1
ls -la gpurun_out
