mkdir -p gpurun_out
timeout 2400 python tools/paper_sweep.py 100000,500000,1000000,2000000,5000000,10000000,15000000 > gpurun_out/r2z_ladder.jsonl 2> gpurun_out/r2z_ladder.err
