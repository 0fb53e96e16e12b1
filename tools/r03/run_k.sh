mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kuramoto.py tests/test_gpu_multi.py tests/test_gpu_gen.py -x -q --timeout 300 > gpurun_out/rk_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/rk_gputest.log
timeout 300 python bench.py --steps 1000 --no-cpu-baseline > gpurun_out/rk_bench.log 2>&1
