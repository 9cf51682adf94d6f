#!/bin/bash
# GPU box: for each library variant, device time (quick_perf) + ncu counters of the tier-1 cell kernel on a
# 1M-site C4.   tools/ncu_ab.sh base w4 nofr ...
mkdir -p gpurun_out
for v in "$@"; do
  lib=paper_2605_06408_b200/libpd_$v.so; [ "$v" = base ] && lib=paper_2605_06408_b200/libpd.so
  PD_LIB=$lib python tools/quick_perf.py C4 C2 > gpurun_out/ab_$v.perf 2>&1
  PD_LIB=$lib ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,launch__occupancy_limit_blocks,sm__maximum_warps_per_active_cycle_pct,smsp__thread_inst_executed_per_inst_executed.ratio \
    --clock-control none --kernel-name regex:cells_kernel -s 3 -c 1 --csv python tools/prof_c4n.py 1000000 > gpurun_out/ab_$v.ncu 2>&1
done
