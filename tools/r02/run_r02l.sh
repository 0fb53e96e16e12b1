# ELL work-unit granularity sweep on config 2 (split rblocks, CDK_ELL_UNIT
# = chunks per unit; parts meet through CTA-scope atomics) and calibration
mkdir -p gpurun_out
for u in 0 6 10 16; do
  CDK_ELL_UNIT=$u timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline > gpurun_out/r02l_unit$u.log 2>&1
done
CDK_ELL_CALIBRATE=0 timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline > gpurun_out/r02l_nocal.log 2>&1
