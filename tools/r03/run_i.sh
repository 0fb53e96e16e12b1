mkdir -p gpurun_out
B=paper_2203_16657_b200/_build
export CDK_ELL_STREAM=0
CDK_LIB=$B/libcommdyn_cuda_co_rq4.so timeout 600 python -m pytest tests/test_gpu_kuramoto.py -x -q --timeout 120 > gpurun_out/ri_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/ri_gputest.log
for v in co co_rq3 co_rq4 co_rq6; do
  CDK_LIB=$B/libcommdyn_cuda_$v.so timeout 300 python bench.py --steps 300 --no-cpu-baseline > gpurun_out/ri_bench_$v.log 2>&1
done
