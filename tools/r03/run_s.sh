mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_cs.py tests/test_gpu_long.py -x -q --timeout 900 -k "cs or cfg4 or CS or cucker" > gpurun_out/rs_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/rs_gputest.log
timeout 300 python tools/bench_cfg34.py --steps 50 --only cfg4 > gpurun_out/rs_cfg4.json 2>&1
