mkdir -p gpurun_out
timeout 1500 python tools/paper_sweep.py 100000,1000000,10000000 > gpurun_out/r2z_paper_sweep.jsonl 2> gpurun_out/r2z_paper_sweep.err
timeout 1200 python tools/weight_sweep.py > gpurun_out/r2z_weight_sweep.jsonl 2> gpurun_out/r2z_weight_sweep.err
