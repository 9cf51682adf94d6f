mkdir -p gpurun_out
for v in base nk1 el1; do timeout 400 python tools/ab.py run $v C4 C3 C5 C2 >> gpurun_out/ab11.log 2>&1; done
for ea in 50 100 400; do echo "== exact_after $ea" >> gpurun_out/ab11.log; PD_EXACT_AFTER=$ea timeout 300 python tools/quick_perf.py C4 C3 >> gpurun_out/ab11.log 2>&1; done
bash tools/checks.sh
