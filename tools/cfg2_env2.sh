#!/bin/bash
# like cfg2_env.sh, also printing the plan build time
for e in "$@"; do
  env $e timeout 400 python bench.py --steps 400 --warmup 10 --no-cpu-baseline 2>/tmp/err_$$ | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['ms_per_step']*1e3,1), 'us/step', round(d['roofline']['stage_ms_mean']*1e3,1), 'us/stage e2e', round(d['e2e']['value']/1e9,3), 'plan_s', d['config']['plan_build_s'])" || tail -3 /tmp/err_$$
done
