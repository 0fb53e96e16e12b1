mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ho.py tests/test_gpu_cs.py tests/test_gpu_long.py tests/test_gpu_naive.py -x -q -k "not cfg2_2000" > gpurun_out/r02g_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/r02g_gputest.log
timeout 300 python tools/bench_cfg34.py --steps 50 > gpurun_out/r02g_cfg34.json 2> gpurun_out/r02g_cfg34.err
# bounds-checked build (CDK_DEBUG: device-side index asserts) over the fused-path tests
CDK_LIB=paper_2203_16657_b200/_build/libcommdyn_cuda_debug.so timeout 900 python -m pytest tests/test_gpu_kuramoto.py tests/test_gpu_multi.py tests/test_gpu_gen.py -x -q > gpurun_out/r02g_debug_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02g_debug_tests.log
timeout 600 ncu --set full --clock-control none -k regex:"ho_pass" -c 2 -f -o gpurun_out/r02g_ho python tools/bench_cfg34.py --steps 2 --only cfg3 > gpurun_out/r02g_ncu_ho.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"cs_" -c 4 -f -o gpurun_out/r02g_cs python tools/bench_cfg34.py --steps 2 --only cfg4 > gpurun_out/r02g_ncu_cs.log 2>&1
