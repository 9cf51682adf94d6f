mkdir -p gpurun_out
for v in base pt0 ks6 ks7 base; do timeout 400 python tools/ab.py run $v C4 C3 >> gpurun_out/ab29.log 2>&1; done
