#!/bin/bash
# config-2 step time vs the stage kernel's shared-memory carve-out (rows cap, budget)
run() { CDK_ROWS_CAP=$1 CDK_SMEM_BUDGET=$2 timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('rows $1 budget $2', round(d['ms_per_step']*1e3,1), 'us/step', round(d['roofline']['stage_ms_mean']*1e3,1), 'us/stage')"; }
run 1536 230400
run 768 163680
run 512 149344
run 1536 151904
run 1024 180000
run 1536 230400
