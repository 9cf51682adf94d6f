#!/bin/bash
# GPU box: ncu --set full of one kernel (regex) in a pd_build of C4 at N sites; exports raw + source CSV.
#   tools/prof_kernel.sh <tag> <kernel-regex> [n] [skip]
T=$1; K=$2; N=${3:-1000000}; S=${4:-1}
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none --kernel-name regex:$K -s $S -c 1 \
    -o gpurun_out/${T} -f python tools/prof_c4n.py ${N} > gpurun_out/${T}_run.log 2>&1
ncu -i gpurun_out/${T}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${T}_src.csv 2>/dev/null
ncu -i gpurun_out/${T}.ncu-rep --page raw --csv > gpurun_out/${T}_raw.csv 2>/dev/null
ncu -i gpurun_out/${T}.ncu-rep --page details > gpurun_out/${T}_details.txt 2>/dev/null
