# round-2 record: full GPU suite, bounds-checked build over the fused paths,
# the bench line, launch list, ncu capture of the timed kernel, drain profile,
# configs 3/4, LDS and fp64 microbenchmarks
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/rf_smi.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/rf_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/rf_gputest.log
CDK_LIB=paper_2203_16657_b200/_build/libcommdyn_cuda_debug.so timeout 900 python -m pytest tests/test_gpu_kuramoto.py tests/test_gpu_multi.py tests/test_gpu_gen.py -x -q > gpurun_out/rf_debug_tests.log 2>&1
echo "rc=$?" >> gpurun_out/rf_debug_tests.log
timeout 600 python bench.py > gpurun_out/rf_bench.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/rf_reference.log 2>&1
timeout 300 python tools/bench_cfg34.py --steps 50 > gpurun_out/rf_cfg34.json 2>&1
timeout 300 python tools/prof_rk4.py > gpurun_out/rf_prof_rk4.txt 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/lds_bench tools/lds_bench.cu && /tmp/lds_bench > gpurun_out/rf_lds_bench.txt 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/rf_fp64_peak.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/rf_launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ell_rk4_kernel --launch-skip 3 -c 1 -f -o gpurun_out/rf_rk4 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/rf_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"ho_" -c 6 -f -o gpurun_out/rf_ho python tools/bench_cfg34.py --steps 2 --only cfg3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"cs_" -c 4 -f -o gpurun_out/rf_cs python tools/bench_cfg34.py --steps 2 --only cfg4 > /dev/null 2>&1
