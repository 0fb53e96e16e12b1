# ELL cp.async chunk ring: parity of the ELL paths, then config-2 step time
# for the default build and ring/thread variants
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kuramoto.py tests/test_gpu_multi.py tests/test_gpu_twins.py -x -q > gpurun_out/r02c_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/r02c_gputest.log
timeout 300 python bench.py --steps 2000 --warmup 10 --no-cpu-baseline > gpurun_out/r02c_bench.log 2>&1
for v in d4 t640d4 d8x8; do
  CDK_LIB=paper_2203_16657_b200/_build/libcommdyn_cuda_$v.so timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline > gpurun_out/r02c_bench_$v.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ell_rk4_kernel --launch-skip 3 -c 1 -f -o gpurun_out/r02c_rk4 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02c_ncu.log 2>&1
