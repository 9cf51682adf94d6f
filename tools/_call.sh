mkdir -p gpurun_out
for v in base fr base fr; do timeout 400 python tools/ab.py run $v C4 C3 >> gpurun_out/ab36.log 2>&1; done
PD_LIB=paper_2605_06408_b200/libpd_fr.so timeout 900 python -m pytest tests -m gpu -q -x -k "c1_full or configs_full_small or paper_workloads" > gpurun_out/t36.log 2>&1; echo "rc=$?" >> gpurun_out/t36.log
