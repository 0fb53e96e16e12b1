#!/bin/bash
# config-5 stage time split: full / sweep only / segments only (timing only)
for f in 0 2 1; do
  CDK_DEBUG_FLAGS=$f timeout 600 python bench.py --config cfg5 --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('flags $f ${EXTRA}', round(d['roofline']['stage_ms_mean'],2), 'ms/stage')"
done
