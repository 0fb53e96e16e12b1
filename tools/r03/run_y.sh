mkdir -p gpurun_out
B=paper_2203_16657_b200/_build
for v in wb4 wb8; do
  CDK_LIB=$B/libcommdyn_cuda_$v.so timeout 300 python tools/bench_cfg34.py --steps 50 --only cfg4 > gpurun_out/ry_cfg4_$v.json 2>&1
done
