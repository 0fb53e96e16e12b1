mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kuramoto.py tests/test_gpu_naive.py tests/test_harmonics.py tests/test_gpu_ho.py tests/test_gpu_cs.py tests/test_scaling.py -x -q > gpurun_out/re_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/re_gputest.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/re_bench20.log 2>&1
CDK_BENCH_SHARDED=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr=127.0.0.1 --master-port=29533 bench.py --steps 20 --warmup 5 > gpurun_out/re_sharded.log 2>&1
