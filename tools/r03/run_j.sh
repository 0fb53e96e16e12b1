mkdir -p gpurun_out
B=paper_2203_16657_b200/_build
CDK_DEBUG_FLAGS=16 CDK_LIB=$B/libcommdyn_cuda_so.so timeout 300 python bench.py --steps 300 --no-cpu-baseline > gpurun_out/rj_bench_so_nointer.log 2>&1
CDK_DEBUG_FLAGS=16 CDK_LIB=$B/libcommdyn_cuda_profile.so timeout 300 python tools/prof_rk4.py > gpurun_out/rj_prof_nointer.txt 2>&1
