# warp streams vs claimed units: parity tests + bench A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kuramoto.py tests/test_gpu_multi.py tests/test_gpu_gen.py tests/test_gpu_naive.py -x -q > gpurun_out/rc_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/rc_gputest.log
timeout 600 python bench.py --steps 500 --no-cpu-baseline > gpurun_out/rc_bench_stream.log 2>&1
CDK_ELL_STREAM=0 timeout 600 python bench.py --steps 500 --no-cpu-baseline > gpurun_out/rc_bench_claim.log 2>&1
