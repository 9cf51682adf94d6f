mkdir -p gpurun_out
for v in base lp b2 b8 q32; do timeout 400 python tools/ab.py run $v C4 C3 C5 C2 >> gpurun_out/ab17.log 2>&1; done
PD_LIB=paper_2605_06408_b200/libpd_lp.so timeout 900 python -m pytest tests -m gpu -q -x -k "c1_full or configs_full_small or top_tier or ablations_oracle or warm or paper_workloads or lattice or tiny" > gpurun_out/t17.log 2>&1; echo "rc=$?" >> gpurun_out/t17.log
