# source-level ncu capture of the timed RK4 kernel (current build)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ell_rk4_kernel --launch-skip 3 -c 1 -f -o gpurun_out/rb_rk4 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/rb_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/rb_ncu.log
