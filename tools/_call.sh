mkdir -p gpurun_out
for v in base old f64c m6 m7 k1 m6k1; do timeout 300 python tools/ab.py run $v C4 C3 >> gpurun_out/ab3.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -x -k "c1_full or configs_full_small or top_tier or ablations_oracle or dual_tets or warm_start or determinism or box_null or robustness" > gpurun_out/t3.log 2>&1
echo "rc=$?" >> gpurun_out/t3.log
tail -3 gpurun_out/t3.log
