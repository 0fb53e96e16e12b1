mkdir -p gpurun_out
B=paper_2203_16657_b200/_build
CDK_LIB=$B/libcommdyn_cuda_profile.so timeout 300 python tools/prof_rk4.py > gpurun_out/re_prof_stream.txt 2>&1
CDK_ELL_STREAM=0 CDK_LIB=$B/libcommdyn_cuda_profile.so timeout 300 python tools/prof_rk4.py > gpurun_out/re_prof_claim.txt 2>&1
