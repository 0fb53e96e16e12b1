# last check of the committed state: smoke, full GPU suite, driver-style bench, reference arm
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/last_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/last_smoke.log
timeout 1700 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/last_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/last_gputest.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/last_bench20.log 2>&1
timeout 600 python bench.py > gpurun_out/last_bench.log 2>&1
