mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kuramoto.py tests/test_gpu_multi.py tests/test_gpu_cs.py tests/test_gpu_long.py -x -q -k "not cfg2_2000 or ell-1" > gpurun_out/r02e_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/r02e_gputest.log
timeout 300 python bench.py --steps 2000 --warmup 10 --no-cpu-baseline > gpurun_out/r02e_bench.log 2>&1
for v in xpre1 t640x1 xpre1d8; do
  CDK_LIB=paper_2203_16657_b200/_build/libcommdyn_cuda_$v.so timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline > gpurun_out/r02e_bench_$v.log 2>&1
done
timeout 300 python tools/bench_cfg34.py --steps 50 > gpurun_out/r02e_cfg34.json 2> gpurun_out/r02e_cfg34.err
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/r02e_fp64_peak.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"cs_|ho_pass" -c 8 -f -o gpurun_out/r02e_cfg34 python tools/bench_cfg34.py --steps 2 > gpurun_out/r02e_ncu34.log 2>&1
