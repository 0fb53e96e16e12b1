// Shared device helpers for libcommdyn_cuda.so (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <string>

#include "../../include/commdyn_cuda.h"

namespace cdk {

constexpr unsigned FULL = 0xffffffffu;

// --- error plumbing ---------------------------------------------------------
void set_error(const std::string &msg);
extern std::atomic<int64_t> g_launches;

inline int cuda_status(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return CDK_OK;
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return CDK_CUDA;
}

#define CDK_CHECK_LAUNCH(what)                                   \
  do {                                                           \
    ::cdk::g_launches.fetch_add(1, std::memory_order_relaxed);   \
    cudaError_t _e = cudaGetLastError();                         \
    if (_e != cudaSuccess) return ::cdk::cuda_status(_e, what);  \
  } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// --- fork/join onto an auxiliary stream --------------------------------------
// Two independent kernels of one stage overlap instead of queueing: aux_fork
// makes the per-device auxiliary stream wait for everything issued on `st` so
// far and returns it (nullptr if it cannot be set up: the caller then stays
// on `st`); aux_join makes `st` wait for everything issued on it since.
struct AuxFork {
  cudaStream_t aux = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
inline AuxFork *aux_fork(cudaStream_t st) {
  static thread_local AuxFork f[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  AuxFork &x = f[dev];
  if (!x.aux) {
    int lo = 0, hi = 0;  // the side stream's (smaller) kernels go first when CTA slots free up
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&x.aux, cudaStreamNonBlocking, hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming) != cudaSuccess) {
      x = AuxFork{};
      cudaGetLastError();
      return nullptr;
    }
  }
  if (cudaEventRecord(x.fork, st) != cudaSuccess ||
      cudaStreamWaitEvent(x.aux, x.fork, 0) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return &x;
}
inline int aux_join(AuxFork *f, cudaStream_t st) {
  cudaError_t e = cudaEventRecord(f->join, f->aux);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st, f->join, 0);
  return cuda_status(e, "aux stream join");
}

// --- IEEE ops that must not be contracted into FMA (mirror numpy rounding) --
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

// wrap to (-pi, pi]: x - 2pi*ceil((x - pi)/(2pi)), same formula as oracle/cia.py
__device__ __forceinline__ double wrap_phase(double x) {
  const double PI = 3.141592653589793;
  const double TWO_PI = 6.283185307179586;
  double k = ceil(__ddiv_rn(__dsub_rn(x, PI), TWO_PI));
  return __dsub_rn(x, __dmul_rn(TWO_PI, k));
}

// --- loads ------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T ldg(const T *p) { return __ldg(p); }

__device__ __forceinline__ double2 ldcg2(const double2 *p) { return __ldcg(p); }

// L2 eviction-priority hints: streamed-once data (CSR index runs, row
// pointers, per-row scratch) is loaded evict-first so it does not push the
// randomly gathered state out of L2.
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t *a, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
               : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ int64_t ld_stream(const int64_t *a, uint64_t pol) {
  int64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b64 %0, [%1], %2;"
               : "=l"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t ld_stream(const uint64_t *a, uint64_t pol) {
  uint64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b64 %0, [%1], %2;"
               : "=l"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ uint4 ld_stream(const uint4 *a, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ldcg_stream(const double2 *a, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void stcg_stream(double2 *a, double2 v, uint64_t pol) {
  asm volatile("st.global.cg.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;"
               :: "l"(a), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}

// status.reserved bit 0 (Kuramoto paths): a peer barrier timed out; the run
// is aborted (kuramoto.cu peer_barrier)
__device__ __forceinline__ bool run_aborted(const cdk_run_status *st) {
  return (*reinterpret_cast<const volatile long long *>(&st->reserved) & 1ll) != 0;
}

// --- warp reductions (xor butterfly: every lane ends with the same bits) ----
__device__ __forceinline__ double warp_sum(double v, int width = 32) {
  for (int o = width >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

}  // namespace cdk
