mkdir -p gpurun_out
B=paper_2203_16657_b200/_build
CDK_LIB=$B/libcommdyn_cuda_profile.so timeout 300 python tools/prof_rk4.py > gpurun_out/rg_prof_stream.txt 2>&1
