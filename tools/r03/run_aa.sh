mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kuramoto.py tests/test_gpu_long.py tests/test_gpu_naive.py tests/test_gpu_multi.py -x -q --timeout 600 > gpurun_out/raa_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/raa_gputest.log
timeout 300 python tools/r03/e2e_phases.py 20 > gpurun_out/raa_e2e20.txt 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/raa_bench20.log 2>&1
