// fp64 FMA (DFMA) peak of this B200 (MEASURED_PEAKS.json has no
// fp64 figure; config 4's secondary roofline).  Every thread runs 8
// independent DFMA chains; one FMA = 2 flops.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) dfma_chains(int iters, double *out) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-7 + k;
  const double b = 0.999999999, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 1234.5) out[0] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double *out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int bps : {4, 8}) {
    const int blocks = sms * bps;
    dfma_chains<<<blocks, 256>>>(iters, out);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    dfma_chains<<<blocks, 256>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8.0 * iters * (double)blocks * 256;
    printf("DFMA %d blocks/SM: %.2f TFLOP/s fp64 (%.1f flop/clk/SM at %d MHz)\n", bps,
           flops / (ms * 1e-3) / 1e12, flops / (ms * 1e-3) / (clk * 1e3) / sms, clk / 1000);
  }
  return 0;
}
