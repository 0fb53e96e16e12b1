#!/bin/bash
# config-2 step time under environment settings: tools/cfg2_env.sh "CDK_ELL_UNIT=8" "CDK_ELL_UNIT=16" ...
for e in "$@"; do
  env $e timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu-baseline 2>/tmp/err_$$ | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['ms_per_step']*1e3,1), 'us/step', round(d['roofline']['stage_ms_mean']*1e3,1), 'us/stage e2e', round(d['e2e']['value']/1e9,3))" || tail -3 /tmp/err_$$
done
