#!/bin/bash
# config-5 step time under environment settings
for e in "$@"; do
  env $e timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu-baseline 2>/tmp/err_$$ | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['ms_per_step'],2), 'ms/step', round(d['roofline']['stage_ms_mean'],2), 'ms/stage')" || tail -3 /tmp/err_$$
done
