# final record of the round: full GPU suite, bounds-checked build over the fused
# paths, bench line (default and driver-style 20 steps), reference arm, configs
# 3/4, launch list and one ncu --set full capture of the timed kernel
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/fin_smi.txt
timeout 1700 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/fin_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/fin_gputest.log
CDK_LIB=paper_2203_16657_b200/_build/libcommdyn_cuda_debug.so timeout 900 python -m pytest tests/test_gpu_kuramoto.py tests/test_gpu_multi.py tests/test_gpu_gen.py -x -q --timeout 600 > gpurun_out/fin_debug_tests.log 2>&1
echo "rc=$?" >> gpurun_out/fin_debug_tests.log
timeout 600 python bench.py > gpurun_out/fin_bench.log 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin_bench20.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin_reference.log 2>&1
timeout 300 python tools/bench_cfg34.py --steps 50 > gpurun_out/fin_cfg34.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin_launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ell_rk4_kernel --launch-skip 3 -c 1 -f -o gpurun_out/fin_rk4 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/fin_ncu.log 2>&1
