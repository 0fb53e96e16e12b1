// Sweep-shaped gather microbenchmark: rows of L random int32 columns into a
// table of double2 (32 MB), 8 lanes per row, IU loads in flight per lane,
// per-row 8-lane reduction, optional row pointers from memory and per-row
// read-modify-write of a 16-byte accumulator.  Isolates what limits the
// block-phased inter sweep (csrc/kuramoto.cu inter_sweep).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cstdlib>
#include <cuda_runtime.h>
#include <string>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1;} } while (0)

template <int IU, bool PTR, bool RMW, int LPR>
__global__ void __launch_bounds__(1024, 1) sweep(const int64_t *ptr, const int *col, int64_t rows_per_cta,
                                                 int L, const double2 *tab, double2 *acc) {
  const int tid = threadIdx.x, lane = tid & 31, t = lane & (LPR - 1), grp = tid / LPR;
  constexpr int NG = 1024 / LPR;
  const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (lane & ~(LPR - 1)));
  const int64_t rA = blockIdx.x * rows_per_cta, rB = rA + rows_per_cta;
  for (int64_t i = rA + grp; i < rB; i += NG) {
    int64_t s0, s1;
    if (PTR) { s0 = __ldg(ptr + i); s1 = __ldg(ptr + i + 1); } else { s0 = i * L; s1 = s0 + L; }
    double sr = 0, si = 0;
    for (int64_t p = s0 + t; p < s1; p += LPR * IU) {
      int j[IU];
#pragma unroll
      for (int k = 0; k < IU; ++k) j[k] = (p + LPR * k < s1) ? __ldg(col + p + LPR * k) : -1;
      double2 z[IU];
#pragma unroll
      for (int k = 0; k < IU; ++k) z[k] = (j[k] >= 0) ? __ldcg(tab + j[k]) : make_double2(0, 0);
#pragma unroll
      for (int k = 0; k < IU; ++k) { sr += z[k].x; si += z[k].y; }
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) { sr += __shfl_xor_sync(gmask, sr, o); si += __shfl_xor_sync(gmask, si, o); }
    if (t == 0) {
      if (RMW) { double2 pv = __ldcg(acc + i); sr += pv.x; si += pv.y; }
      __stcg(acc + i, make_double2(sr, si));
    }
  }
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t tab_n = (32u << 20) / 16;
  double2 *tab; CK(cudaMalloc(&tab, tab_n * 16)); CK(cudaMemset(tab, 0, tab_n * 16));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int SM = getenv("SMEM") ? atoi(getenv("SMEM")) : 0;
  for (int L : {25, 100, 400}) {
    const size_t total = (size_t)400 << 20;  // entries
    const int64_t rows = total / L, rpc = rows / sms;
    std::vector<int> h(rpc * sms * L);
    std::vector<int64_t> hp(rpc * sms + 1);
    uint64_t x = 88172645463325252ull;
    for (size_t i = 0; i < h.size(); ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = (int)(x % tab_n); }
    for (size_t i = 0; i < hp.size(); ++i) hp[i] = (int64_t)i * L;
    const char *mode = getenv("ORDER");  // sorted | strided | (random)
    if (mode) {
      for (int64_t r = 0; r + 1 < (int64_t)hp.size(); ++r) {
        std::sort(h.begin() + hp[r], h.begin() + hp[r + 1]);
        if (std::string(mode) == "strided") {  // lane-major: lane t's IU entries contiguous in sort order
          std::vector<int> tmp(h.begin() + hp[r], h.begin() + hp[r + 1]);
          int q = 0;
          for (int t = 0; t < 8; ++t)
            for (int k = t; k < L; k += 8) h[hp[r] + k] = tmp[q++];
        }
      }
    }
    int *col; int64_t *ptr; double2 *acc;
    CK(cudaMalloc(&col, h.size() * 4)); CK(cudaMalloc(&ptr, hp.size() * 8)); CK(cudaMalloc(&acc, hp.size() * 16));
    CK(cudaMemcpy(col, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ptr, hp.data(), hp.size() * 8, cudaMemcpyHostToDevice));
    float ms;
#define RUN(IU, PTR, RMW, LPR)                                                            \
    CK(cudaFuncSetAttribute(sweep<IU, PTR, RMW, LPR>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM)); \
    sweep<IU, PTR, RMW, LPR><<<sms, 1024, SM>>>(ptr, col, rpc, L, tab, acc);                  \
    CK(cudaDeviceSynchronize()); CK(cudaEventRecord(e0));                                 \
    for (int r = 0; r < 3; ++r) sweep<IU, PTR, RMW, LPR><<<sms, 1024, SM>>>(ptr, col, rpc, L, tab, acc); \
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1)); \
    printf("L=%3d IU=%2d ptr=%d rmw=%d lpr=%2d: %.1f Ggathers/s\n", L, IU, PTR, RMW, LPR,       \
           3.0 * rpc * sms * L / (ms * 1e-3) / 1e9);
    RUN(8, true, true, 8); RUN(8, true, true, 4);
    CK(cudaFree(col)); CK(cudaFree(ptr)); CK(cudaFree(acc));
  }
  return 0;
}
