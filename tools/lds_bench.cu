// Shared-memory gather floor on B200: LDS.128 of double2 from a 9000-node
// window, indices held in registers (no global index stream), 8 loads in
// flight per lane, 4 accumulators.  Random vs conflict-free (8 distinct bank
// groups per quarter-warp) vs 2-way conflicts, and LDS.64 split re/im arrays.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/lds_bench tools/lds_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int W = 9000;
constexpr int NI = 16;  // indices per lane

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// mode 0 random, 1 conflict-free, 2 two lanes per bank group (2 wavefronts), 3 all in one bank group
template <int MODE>
__global__ void __launch_bounds__(896, 1) gather128(int iters, double *out) {
  extern __shared__ __align__(128) double2 zs[];
  for (int i = threadIdx.x; i < W + 8; i += blockDim.x) zs[i] = make_double2(i * 1e-3, -i * 1e-3);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t idx[NI];
#pragma unroll
  for (int k = 0; k < NI; ++k) {
    uint32_t h = hash32(threadIdx.x * 131 + k * 7919 + blockIdx.x * 1000003) % (W - 1024);
    if (MODE == 1) h = (h & ~7u) | ((lane + k) & 7);
    if (MODE == 2) h = (h & ~7u) | (((lane >> 1) + k) & 3);
    if (MODE == 3) h = (h & ~7u);
    idx[k] = h;
  }
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(zs);
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t x = (it & 63) * 8;  // keeps bank groups, moves addresses
#pragma unroll
    for (int k0 = 0; k0 < NI; k0 += 8) {
      double2 z[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(z[k].x), "=d"(z[k].y)
                     : "r"(base + ((idx[k0 + k] + x) << 4)));
      }
#pragma unroll
      for (int k = 0; k < 8; k += 2) { a0 += z[k].x; a1 += z[k].y; a2 += z[k + 1].x; a3 += z[k + 1].y; }
    }
  }
  if (a0 + a1 + a2 + a3 == 12345.0) out[0] = a0;
}

// split arrays: re[] and im[] (LDS.64 each)
__global__ void __launch_bounds__(896, 1) gather64x2(int iters, double *out) {
  extern __shared__ __align__(128) double sm[];
  double *re = sm, *im = sm + W + 8;
  for (int i = threadIdx.x; i < W + 8; i += blockDim.x) { re[i] = i * 1e-3; im[i] = -i * 1e-3; }
  __syncthreads();
  uint32_t idx[NI];
#pragma unroll
  for (int k = 0; k < NI; ++k) idx[k] = hash32(threadIdx.x * 131 + k * 7919 + blockIdx.x * 1000003) % (W - 1024);
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t x = (it & 63) * 8;
#pragma unroll
    for (int k0 = 0; k0 < NI; k0 += 8) {
      double r[8], m[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) { r[k] = re[idx[k0 + k] + x]; m[k] = im[idx[k0 + k] + x]; }
#pragma unroll
      for (int k = 0; k < 8; k += 2) { a0 += r[k]; a1 += m[k]; a2 += r[k + 1]; a3 += m[k + 1]; }
    }
  }
  if (a0 + a1 + a2 + a3 == 12345.0) out[0] = a0;
}

int main() {
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int clk = 0; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  double *out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int iters = 4000;
  auto run = [&](auto kern, size_t smem, const char *name) -> int {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<sms, 896, smem>>>(iters, out);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    kern<<<sms, 896, smem>>>(iters, out);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    const double ent = (double)sms * 896 * NI * iters;
    printf("%-28s %8.1f Gentries/s  %.3f cycles/entry/SM @%d MHz\n", name, ent / (ms * 1e-3) / 1e9,
           (ms * 1e-3) * clk * 1e3 * sms / ent, clk / 1000);
    return 0;
  };
  run(gather128<0>, (W + 8) * 16, "LDS.128 random");
  run(gather128<1>, (W + 8) * 16, "LDS.128 conflict-free");
  run(gather128<2>, (W + 8) * 16, "LDS.128 2-way");
  run(gather128<3>, (W + 8) * 16, "LDS.128 8-way");
  run(gather64x2, (W + 8) * 16, "LDS.64 x2 random");
  return 0;
}
