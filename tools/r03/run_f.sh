mkdir -p gpurun_out
B=paper_2203_16657_b200/_build
timeout 900 python -m pytest tests/test_gpu_kuramoto.py tests/test_gpu_multi.py -x -q --timeout 120 > gpurun_out/rh_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/rh_gputest.log
CDK_LIB=$B/libcommdyn_cuda_so.so timeout 300 python bench.py --steps 300 --no-cpu-baseline > gpurun_out/rh_bench_so.log 2>&1
timeout 300 python bench.py --steps 300 --no-cpu-baseline > gpurun_out/rh_bench_default.log 2>&1
CDK_LIB=$B/libcommdyn_cuda_profile.so timeout 300 python tools/prof_rk4.py > gpurun_out/rh_prof_stream.txt 2>&1
