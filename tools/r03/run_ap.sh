mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cs.py tests/test_gpu_long.py tests/test_gpu_naive.py -x -q --timeout 600 > gpurun_out/rap_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/rap_gputest.log
timeout 300 python tools/bench_cfg34.py --steps 50 --only cfg4 > gpurun_out/rap_cfg4_spread.json 2>&1
CDK_CS_BANK_SPREAD=0 timeout 300 python tools/bench_cfg34.py --steps 50 --only cfg4 > gpurun_out/rap_cfg4_sorted.json 2>&1
