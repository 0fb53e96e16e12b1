#!/bin/bash
# config-2 step time: stage CTAs per SM (library variants) x segment rows cap / smem budget
B=paper_2203_16657_b200/_build
run() { CDK_LIB=$1 CDK_ROWS_CAP=$2 CDK_SMEM_BUDGET=$3 timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu-baseline 2>/tmp/err_$$ | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$(basename $1) rows $2 budget $3', round(d['ms_per_step']*1e3,1), 'us/step', round(d['roofline']['stage_ms_mean']*1e3,1), 'us/stage e2e', round(d['e2e']['value']/1e9,3))" || tail -3 /tmp/err_$$; }
run $B/libcommdyn_cuda.so 1536 230400
for lib in t448c2 t512c2 t384c2; do
  for rc in 512 768 1024; do run $B/libcommdyn_cuda_$lib.so $rc 114000; done
done
run $B/libcommdyn_cuda.so 1536 230400
