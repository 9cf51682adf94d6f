mkdir -p gpurun_out
for v in base pk1 pk3; do timeout 400 python tools/ab.py run $v C5 C3 C4 C2 >> gpurun_out/ab9.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -x -k "c1_full or configs_full_small or top_tier or ablations_oracle or warm or record_arena or paper_workloads" > gpurun_out/t9.log 2>&1; echo "rc=$?" >> gpurun_out/t9.log
