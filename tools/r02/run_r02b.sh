set -x
SKIP_NCU=0 bash tools/gpu_round.sh r02b -k "not cfg2_2000"
for v in t640 t768; do
  CDK_LIB=paper_2203_16657_b200/_build/libcommdyn_cuda_$v.so timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu-baseline > gpurun_out/r02b_bench_$v.log 2>&1
done
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/lds_bench tools/lds_bench.cu && /tmp/lds_bench > gpurun_out/r02b_lds_bench.txt 2>&1
