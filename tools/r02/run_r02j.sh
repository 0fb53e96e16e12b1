mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_appendix_models.py tests/test_gpu_cs.py -x -q > gpurun_out/r02j_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/r02j_gputest.log
for v in default csb1m2 csb2m3 csb4m3 csb2m2; do
  if [ $v = default ]; then L=""; else L=paper_2203_16657_b200/_build/libcommdyn_cuda_$v.so; fi
  CDK_LIB=$L timeout 300 python tools/bench_cfg34.py --steps 50 --only cfg4 > gpurun_out/r02j_cfg4_$v.json 2>&1
done
