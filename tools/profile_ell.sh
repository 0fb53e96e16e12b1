#!/bin/bash
# Round profile set for the ELL path (GPU box): tests, smoke, cfg2 bench line,
# launch list, one ncu --set full capture of the ELL stage kernel.
D=gpurun_out/${1:-prof}
mkdir -p $D
timeout 1200 python -m pytest tests -m gpu -x -q > $D/pytest.log 2>&1; tail -2 $D/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; tail -1 $D/smoke.log
python bench.py > $D/bench_cfg2.json 2> $D/bench_cfg2.err; tail -1 $D/bench_cfg2.json
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $D/launches_cfg2.csv 2> $D/launches_cfg2.err
python tools/cfg2_stage.py > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ell_stage_kernel -s 3 -c 1 \
      -o $D/cfg2_ell_stage python tools/cfg2_stage.py > $D/cfg2_ncu.log 2>&1
ls $D
