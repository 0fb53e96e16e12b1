mkdir -p gpurun_out
for c in 8 12; do
  CDK_ELL_CALIBRATE=$c timeout 400 python bench.py --steps 500 --no-cpu-baseline > gpurun_out/rp_bench_cal$c.log 2>&1
done
