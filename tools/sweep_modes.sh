#!/bin/bash
# time the config-5 stage kernel under each inter-sweep variant (CDK_SWEEP)
for m in ${MODES:-0 1 2 3 4 5 6}; do
  CDK_SWEEP=$m timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('mode $m', round(d['roofline']['stage_ms_mean'],2), 'ms/stage')"
done
