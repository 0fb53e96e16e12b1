# warp streams: parity (per-test timeout), variants A/B, stage timeline
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kuramoto.py tests/test_gpu_multi.py -x -q --timeout 120 > gpurun_out/rd_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/rd_gputest.log
B=paper_2203_16657_b200/_build
for v in so so_d8 so_t768 so_t1024; do
  CDK_LIB=$B/libcommdyn_cuda_$v.so timeout 300 python bench.py --steps 300 --no-cpu-baseline > gpurun_out/rd_bench_$v.log 2>&1
done
for ic in 0.5 3.0; do
  CDK_ELL_ITEM_COST=$ic CDK_LIB=$B/libcommdyn_cuda_so.so timeout 300 python bench.py --steps 300 --no-cpu-baseline > gpurun_out/rd_bench_so_ic$ic.log 2>&1
done
CDK_LIB=$B/libcommdyn_cuda_profile.so timeout 300 python tools/prof_rk4.py > gpurun_out/rd_prof_rk4.txt 2>&1
