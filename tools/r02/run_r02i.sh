mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ho.py tests/test_gpu_long.py tests/test_gpu_naive.py tests/test_gpu_cs.py -x -q -k "not cfg2_2000" > gpurun_out/r02i_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/r02i_gputest.log
timeout 300 python tools/bench_cfg34.py --steps 50 > gpurun_out/r02i_cfg34.json 2> gpurun_out/r02i_cfg34.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ho_" -c 4 -f -o gpurun_out/r02i_ho python tools/bench_cfg34.py --steps 2 --only cfg3 > gpurun_out/r02i_ncu_ho.log 2>&1
