mkdir -p gpurun_out
B=paper_2203_16657_b200/_build
for v in rl1 rl2 rl4; do
  CDK_LIB=$B/libcommdyn_cuda_$v.so timeout 300 python tools/bench_cfg34.py --steps 50 --only cfg4 > gpurun_out/rv_cfg4_$v.json 2>&1
done
CDK_LIB=$B/libcommdyn_cuda_rl1.so timeout 900 python -m pytest tests/test_gpu_cs.py -x -q --timeout 600 > gpurun_out/rv_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/rv_gputest.log
