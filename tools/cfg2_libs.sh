#!/bin/bash
# config-2 step time for library variants (CDK_LIB)
for lib in "$@"; do
  CDK_LIB=$lib timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$(basename $lib)', round(d['ms_per_step']*1e3,1), 'us/step', round(d['roofline']['stage_ms_mean']*1e3,1), 'us/stage', 'e2e', round(d['e2e']['value']/1e9,3), d['clocks'])"
done
