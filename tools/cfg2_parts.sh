#!/bin/bash
# config-2 stage/step time with parts of the work removed (timing only)
for f in ${FLAGS:-0 4 8 12}; do
  CDK_DEBUG_FLAGS=$f timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('flags $f', round(d['ms_per_step']*1e3,1), 'us/step', round(d['roofline']['stage_ms_mean']*1e3,1), 'us/stage')"
done
