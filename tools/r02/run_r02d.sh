# full GPU suite (incl. the config-2 2000-step test), the bench line, the
# drain profile of the persistent ELL kernel, launch list + ncu capture
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02d_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/r02d_gputest.log
timeout 300 python bench.py > gpurun_out/r02d_bench.log 2>&1
timeout 300 python tools/prof_rk4.py > gpurun_out/r02d_prof_rk4.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02d_launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ell_rk4_kernel --launch-skip 3 -c 1 -f -o gpurun_out/r02d_rk4 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02d_ncu.log 2>&1
