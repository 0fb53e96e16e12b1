#!/bin/bash
# config-2 step time under the inter-entry variants (env overrides of plan.py)
run() { timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step']*1e3,1), 'us/step', round(d['roofline']['stage_ms_mean']*1e3,1), 'us/stage', 'e2e', round(d['e2e']['value']/1e9,3))"; }
run default
CDK_INTER_PHASE=1 run phase
CDK_INTER_BLOCKS=1 run sweep1
