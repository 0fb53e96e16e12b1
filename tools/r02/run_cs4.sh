mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cs.py tests/test_gpu_long.py tests/test_gpu_naive.py -x -q -k "cs or cfg4" > gpurun_out/rc4_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/rc4_gputest.log
timeout 300 python tools/bench_cfg34.py --steps 50 --only cfg4 > gpurun_out/rc4_cfg4.json 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"cs_" -c 5 -f -o gpurun_out/rc4_cs python tools/bench_cfg34.py --steps 2 --only cfg4 > /dev/null 2>&1
