// Random global-gather ceiling on B200: table of T bytes (16-byte or 8-byte
// elements), int32 indices streamed, 1024 threads/CTA, one CTA per SM, U
// loads in flight per thread.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1;} } while (0)

template <int U, int CG, typename T>
__global__ void __launch_bounds__(1024, 1) gather(const int *__restrict__ idx, size_t per_cta,
                                                  const T *__restrict__ tab, double *out) {
  const int *p = idx + blockIdx.x * per_cta;
  double acc = 0.0;
  for (size_t i = threadIdx.x; i < per_cta; i += 1024 * U) {
    int j[U];
#pragma unroll
    for (int k = 0; k < U; ++k) j[k] = (i + 1024 * k < per_cta) ? __ldg(p + i + 1024 * k) : 0;
    T v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) v[k] = CG ? __ldcg(tab + j[k]) : __ldg(tab + j[k]);
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if constexpr (sizeof(T) == 16) acc += ((const double2 &)v[k]).x + ((const double2 &)v[k]).y;
      else acc += (double &)v[k];
    }
  }
  if (acc == 1.2345) *out = acc;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t n_idx = (size_t)256 << 20;  // 256M gathers
  const size_t per_cta = n_idx / sms;
  int *d_idx; CK(cudaMalloc(&d_idx, n_idx * 4));
  double *out; CK(cudaMalloc(&out, 8));
  char *tab; CK(cudaMalloc(&tab, (size_t)1 << 30)); CK(cudaMemset(tab, 0, (size_t)1 << 30));
  std::vector<int> h(n_idx);
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  for (size_t tb : {(size_t)8 << 20, (size_t)32 << 20, (size_t)64 << 20, (size_t)96 << 20,
                    (size_t)128 << 20, (size_t)1 << 30}) {
    for (int esz : {16, 8}) {
      const size_t n_el = tb / esz;
      uint64_t x = 88172645463325252ull;
      for (size_t i = 0; i < n_idx; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = (int)(x % n_el); }
      CK(cudaMemcpy(d_idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
      float ms;
#define RUN(U, CG, T, name)                                                               \
  {                                                                                      \
    gather<U, CG, T><<<sms, 1024>>>(d_idx, per_cta, (const T *)tab, out);                 \
    CK(cudaDeviceSynchronize());                                                         \
    CK(cudaEventRecord(e0));                                                             \
    for (int r = 0; r < 3; ++r) gather<U, CG, T><<<sms, 1024>>>(d_idx, per_cta, (const T *)tab, out); \
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));                               \
    CK(cudaEventElapsedTime(&ms, e0, e1));                                               \
    printf("table %5zu MB elem %2d U=%d %s: %.1f Ggathers/s (%.2f cycles/gather/SM @1.965GHz)\n", \
           tb >> 20, esz, U, name, 3.0 * per_cta * sms / (ms * 1e-3) / 1e9,             \
           (ms * 1e-3 / 3.0) * 1.965e9 * sms / (double)(per_cta * sms));                  \
  }
      if (esz == 16) {
        RUN(8, 1, double2, "cg ");
        RUN(8, 0, double2, "ldg");
        RUN(16, 1, double2, "cg ");
      } else {
        RUN(8, 1, double, "cg ");
        RUN(8, 0, double, "ldg");
      }
    }
  }
  return 0;
}
