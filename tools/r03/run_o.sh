mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kuramoto.py tests/test_gpu_multi.py -x -q --timeout 300 > gpurun_out/ro_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/ro_gputest.log
timeout 300 python bench.py --steps 500 --no-cpu-baseline > gpurun_out/ro_bench_claimorder.log 2>&1
CDK_ELL_CLAIM_ORDER=0 timeout 300 python bench.py --steps 500 --no-cpu-baseline > gpurun_out/ro_bench_rblockorder.log 2>&1
timeout 300 python bench.py --steps 500 --no-cpu-baseline > gpurun_out/ro_bench_claimorder2.log 2>&1
