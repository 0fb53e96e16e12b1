# compute-sanitizer memcheck / racecheck / synccheck on both persistent RK4
# kernel families (config 1); logs to gpurun_out/sanitize_*.txt
mkdir -p gpurun_out
for ell in 1 0; do
  for tool in memcheck racecheck synccheck; do
    CDK_ELL=$ell CDK_ELL_CALIBRATE=0 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 \
      python tools/sanitize_cfg1.py > gpurun_out/sanitize_${tool}_ell${ell}.txt 2>&1
    echo "rc=$?" >> gpurun_out/sanitize_${tool}_ell${ell}.txt
  done
done
