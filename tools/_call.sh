mkdir -p gpurun_out
for v in base rf la; do timeout 400 python tools/ab.py run $v C4 C3 >> gpurun_out/ab27.log 2>&1; done
for ea in 60 150; do echo "== exact_after $ea" >> gpurun_out/ab27.log; PD_EXACT_AFTER=$ea timeout 300 python tools/quick_perf.py C4 C3 >> gpurun_out/ab27.log 2>&1; done
timeout 400 python tools/ab.py run base C4 C3 >> gpurun_out/ab27.log 2>&1
