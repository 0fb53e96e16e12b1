# restored-state validation: full GPU suite, bench line, reference arm
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ra_smi.txt
timeout 1700 python -m pytest tests -m gpu -q > gpurun_out/ra_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/ra_gputest.log
timeout 600 python bench.py > gpurun_out/ra_bench.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ra_reference.log 2>&1
timeout 300 python tools/bench_cfg34.py --steps 50 > gpurun_out/ra_cfg34.json 2>&1
