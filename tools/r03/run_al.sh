mkdir -p gpurun_out
B=paper_2203_16657_b200/_build
timeout 900 python -m pytest tests/test_gpu_cs.py tests/test_gpu_long.py -x -q --timeout 600 -k "cs or cfg4 or cucker" > gpurun_out/ral_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/ral_gputest.log
for v in mn256 mn128; do
  CDK_LIB=$B/libcommdyn_cuda_$v.so timeout 300 python tools/bench_cfg34.py --steps 50 --only cfg4 > gpurun_out/ral_cfg4_$v.json 2>&1
done
CDK_LIB=$B/libcommdyn_cuda_mn128.so timeout 600 python -m pytest tests/test_gpu_cs.py -x -q --timeout 600 > gpurun_out/ral_gputest128.log 2>&1
echo "rc=$?" >> gpurun_out/ral_gputest128.log
