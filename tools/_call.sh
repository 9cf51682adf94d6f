mkdir -p gpurun_out
for v in base pm2 pm3 base pm2; do timeout 400 python tools/ab.py run $v C4 C3 >> gpurun_out/ab35.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -x -k "trim or c1_full or configs_full_small or top_tier" > gpurun_out/t35.log 2>&1; echo "rc=$?" >> gpurun_out/t35.log
