mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ho.py -x -q > gpurun_out/r02m_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/r02m_gputest.log
for v in default hob2m4 hob4m2 hob8m2; do
  if [ $v = default ]; then L=""; else L=paper_2203_16657_b200/_build/libcommdyn_cuda_$v.so; fi
  CDK_LIB=$L timeout 300 python tools/bench_cfg34.py --steps 50 --only cfg3 > gpurun_out/r02m_cfg3_$v.json 2>&1
done
