mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cs.py tests/test_gpu_long.py tests/test_gpu_naive.py tests/test_gpu_kuramoto.py -x -q -k "cs or cfg4 or public or cfg1" > gpurun_out/rc_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/rc_gputest.log
for v in default csnonewton; do
  if [ $v = default ]; then L=""; else L=paper_2203_16657_b200/_build/libcommdyn_cuda_$v.so; fi
  CDK_LIB=$L timeout 300 python tools/bench_cfg34.py --steps 50 --only cfg4 > gpurun_out/rc_cfg4_$v.json 2>&1
done
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/rc_bench20.log 2>&1
