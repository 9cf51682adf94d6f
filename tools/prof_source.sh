#!/bin/bash
# Run on the GPU box (gpurun): source-level ncu capture of the tier-1 cell kernel on a 1M-site C4
# (instructions executed / stall reasons per CUDA source line), exported to CSV on the box.
#   tools/prof_source.sh <tag> [n]
T=${1:-src}
N=${2:-1000000}
mkdir -p gpurun_out
python -m paper_2605_06408_b200.build > /dev/null
ncu --set full --import-source on --clock-control none --kernel-name regex:cells_kernel -s 3 -c 1 \
    -o gpurun_out/${T} -f python tools/prof_c4n.py ${N} > gpurun_out/${T}_run.log 2>&1
ncu -i gpurun_out/${T}.ncu-rep --page source --csv --print-source cuda > gpurun_out/${T}_source_cuda.csv 2>&1
ncu -i gpurun_out/${T}.ncu-rep --page details --csv > gpurun_out/${T}_details.csv 2>&1
ls -la gpurun_out
