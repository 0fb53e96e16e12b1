mkdir -p gpurun_out
timeout 300 python tools/bench_cfg34.py --steps 50 > gpurun_out/rr_cfg34.json 2>&1
