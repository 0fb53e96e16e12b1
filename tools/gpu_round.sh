#!/bin/bash
# One GPU round trip: GPU tests, the bench line, the ncu launch list and one
# `ncu --set full` capture of the timed RK4 kernel (each only after its own
# command has exited 0 without ncu).  Usage (from gpurun):
#   bash tools/gpu_round.sh TAG [pytest-args...]
TAG=${1:-r02}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/${TAG}_gputest.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_gputest.log
fi
timeout 600 python bench.py --steps ${STEPS:-2000} --warmup 10 > gpurun_out/${TAG}_bench.log 2>&1
rc=$?; echo "rc=$rc" >> gpurun_out/${TAG}_bench.log
if [ $rc -eq 0 ] && [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 20 --warmup 5 \
    --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:${NCU_KERNEL:-ell_rk4_kernel} --launch-skip 3 -c 1 -f -o gpurun_out/${TAG}_rk4 \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_full.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu_full.log
fi
