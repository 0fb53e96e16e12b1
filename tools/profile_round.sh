#!/bin/bash
# Round profile set (run on the GPU box): bench lines, launch lists, ncu captures.
set -x
mkdir -p gpurun_out/prof
python bench.py --steps 2000 --warmup 10 > gpurun_out/prof/bench_cfg2.json 2> gpurun_out/prof/bench_cfg2.err
python bench.py --config cfg5 --steps 200 --warmup 3 > gpurun_out/prof/bench_cfg5.json 2> gpurun_out/prof/bench_cfg5.err
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/prof/bench_ref.json 2> gpurun_out/prof/bench_ref.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof/launches_cfg2.csv 2> gpurun_out/prof/launches_cfg2.err
python tools/cfg2_stage.py > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:kuramoto_stage_kernel -s 3 -c 1 \
      -o gpurun_out/prof/cfg2_stage python tools/cfg2_stage.py > gpurun_out/prof/cfg2_ncu.log 2>&1
python tools/cfg5_stage.py > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"inter_sweep|kuramoto_stage" -s 2 -c 2 \
      -o gpurun_out/prof/cfg5_stage python tools/cfg5_stage.py > gpurun_out/prof/cfg5_ncu.log 2>&1
ls -la gpurun_out/prof
