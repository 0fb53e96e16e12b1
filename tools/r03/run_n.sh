mkdir -p gpurun_out
B=paper_2203_16657_b200/_build
CDK_LIB=$B/libcommdyn_cuda_tma.so timeout 900 python -m pytest tests/test_gpu_kuramoto.py tests/test_gpu_multi.py -x -q --timeout 300 > gpurun_out/rn_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/rn_gputest.log
CDK_LIB=$B/libcommdyn_cuda_tma.so timeout 300 python bench.py --steps 500 --no-cpu-baseline > gpurun_out/rn_bench_tma.log 2>&1
timeout 300 python bench.py --steps 500 --no-cpu-baseline > gpurun_out/rn_bench_default.log 2>&1
