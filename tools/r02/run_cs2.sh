mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cs.py tests/test_gpu_long.py tests/test_gpu_naive.py -x -q -k "cs or cfg4" > gpurun_out/rc2_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/rc2_gputest.log
timeout 300 python tools/bench_cfg34.py --steps 50 --only cfg4 > gpurun_out/rc2_cfg4.json 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/rc2_bench20.log 2>&1
