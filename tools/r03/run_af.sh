mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kuramoto.py -x -q --timeout 600 > gpurun_out/raf_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/raf_gputest.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/raf_launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ell_rk4_kernel --launch-skip 3 -c 1 -f -o gpurun_out/raf_rk4 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/raf_ncu.log 2>&1
