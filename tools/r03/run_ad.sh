mkdir -p gpurun_out
timeout 1700 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/rad_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/rad_gputest.log
CDK_LIB=paper_2203_16657_b200/_build/libcommdyn_cuda_debug.so timeout 900 python -m pytest tests/test_gpu_kuramoto.py tests/test_gpu_multi.py tests/test_gpu_gen.py -x -q --timeout 600 > gpurun_out/rad_debug_tests.log 2>&1
echo "rc=$?" >> gpurun_out/rad_debug_tests.log
timeout 600 python bench.py > gpurun_out/rad_bench.log 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/rad_bench20.log 2>&1
