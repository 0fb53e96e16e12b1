#!/bin/bash
# Round-2 baseline captures (GPU box): ELL stage kernel (config 2) with source,
# the persistent RK4 kernel the timed step runs, and the config-3/4 kernels.
D=gpurun_out/r02a
mkdir -p $D
python tools/cfg2_stage.py > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ell_stage_kernel -s 3 -c 1 \
      -o $D/cfg2_ell_stage python tools/cfg2_stage.py > $D/cfg2_ncu.log 2>&1
python tools/bench_cfg34.py --steps 5 > $D/cfg34.json 2>&1 && \
  ncu --set full --clock-control none --import-source on -s 40 -c 12 \
      -o $D/cfg34 python tools/bench_cfg34.py --steps 5 > $D/cfg34_ncu.log 2>&1
ls -la $D
