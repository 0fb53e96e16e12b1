mkdir -p gpurun_out
timeout 1700 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/ru_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/ru_gputest.log
timeout 300 python tools/r03/e2e_phases.py 20 > gpurun_out/ru_e2e20.txt 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/ru_bench20.log 2>&1
