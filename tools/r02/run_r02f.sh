mkdir -p gpurun_out
bash tools/run_sanitize.sh
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02f_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/r02f_gputest.log
timeout 300 python bench.py > gpurun_out/r02f_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02f_launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ell_rk4_kernel --launch-skip 3 -c 1 -f -o gpurun_out/r02f_rk4 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"cs_" -c 4 -f -o gpurun_out/r02f_cs python tools/bench_cfg34.py --steps 2 --only cfg4 > gpurun_out/r02f_ncu_cs.log 2>&1
