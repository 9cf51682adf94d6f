mkdir -p gpurun_out
for v in base fs0 pk1; do timeout 400 python tools/ab.py run $v C5 C3 C4 C2 >> gpurun_out/ab8.log 2>&1; done
timeout 400 python tools/ab.py run base C5 C3 C4 --flags 8192 >> gpurun_out/ab8.log 2>&1
timeout 400 python tools/ab.py run base C5 C3 C4 --flags 32 >> gpurun_out/ab8.log 2>&1
