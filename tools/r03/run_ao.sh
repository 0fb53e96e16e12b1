mkdir -p gpurun_out
timeout 1700 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/rao_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/rao_gputest.log
timeout 300 python tools/bench_cfg34.py --steps 50 > gpurun_out/rao_cfg34.json 2>&1
timeout 600 python bench.py --config cfg4 > gpurun_out/rao_cfg4_line.log 2>&1
timeout 600 python bench.py --config cfg3 > gpurun_out/rao_cfg3_line.log 2>&1
