mkdir -p gpurun_out
for v in base fl0 el2 el2i; do timeout 400 python tools/ab.py run $v C4 C3 C5 C2 >> gpurun_out/ab12.log 2>&1; done
for v in el2 el2i; do PD_LIB=paper_2605_06408_b200/libpd_$v.so timeout 900 python -m pytest tests -m gpu -q -x -k "c1_full or configs_full_small or top_tier or ablations_oracle or warm_start or paper_workloads" > gpurun_out/t12_$v.log 2>&1; echo "rc=$?" >> gpurun_out/t12_$v.log; done
