mkdir -p gpurun_out
R=r2f
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${R}_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/${R}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/${R}_bench_ref.json 2> gpurun_out/${R}_bench_ref.err
timeout 900 bash tools/profile_round.sh $R > gpurun_out/${R}_prof.log 2>&1
ncu -i gpurun_out/${R}_cells_full_c4_1m.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${R}_src_cs.csv 2>/dev/null
bash tools/checks.sh
timeout 600 python tools/ablations.py > gpurun_out/${R}_ablations.jsonl 2> gpurun_out/${R}_ablations.err
for c in C2 C3 C5; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/${R}_bench_$c.json 2> gpurun_out/${R}_bench_$c.err; done
