mkdir -p gpurun_out
B=paper_2203_16657_b200/_build
timeout 300 python tools/bench_cfg34.py --steps 50 --only cfg4 > gpurun_out/ram_cfg4_base.json 2>&1
CDK_LIB=$B/libcommdyn_cuda_sp.so timeout 300 python tools/bench_cfg34.py --steps 50 --only cfg4 > gpurun_out/ram_cfg4_sp.json 2>&1
CDK_LIB=$B/libcommdyn_cuda_sp.so timeout 600 python -m pytest tests/test_gpu_cs.py -x -q --timeout 600 > gpurun_out/ram_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/ram_gputest.log
