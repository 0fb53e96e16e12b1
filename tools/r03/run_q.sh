mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_cs.py tests/test_gpu_ho.py tests/test_gpu_naive.py -x -q --timeout 600 > gpurun_out/rq_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/rq_gputest.log
timeout 300 python tools/bench_cfg34.py --steps 50 > gpurun_out/rq_cfg34.json 2>&1
