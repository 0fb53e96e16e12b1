// TMA tile::gather4 throughput for random 16-byte rows of a table (double2),
// vs the LSU path (tools/gather_bench.cu: ~270 Ggathers/s L2-resident,
// bound by L1 miss processing).  One CTA per SM: P producer warps (lane 0
// issues gather4 into a ring of slots, each slot = B gather4 = 4B rows, one
// mbarrier per slot), the other warps consume (sum) and release slots.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -lcuda
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1;} } while (0)

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t *b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mb_expect(uint64_t *b, uint32_t tx) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(b)), "r"(tx) : "memory"); }
__device__ __forceinline__ void mb_arrive(uint64_t *b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mb_wait(uint64_t *b, uint32_t ph) {
  asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" :: "r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void gather4(void *dst, const CUtensorMap *tm, uint64_t *bar, int r0, int r1, int r2, int r3) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
               :: "r"(su32(dst)), "l"(tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(bar)) : "memory");
}

constexpr int THREADS = 1024;
template <int P, int S, int B>
__global__ void __launch_bounds__(THREADS, 1) tma_gather(const __grid_constant__ CUtensorMap tm, const int4 *idx, size_t n4_per_cta, double *out) {
  extern __shared__ __align__(128) unsigned char smem[];
  double2 *slots = reinterpret_cast<double2 *>(smem);               // [P][S][4B]
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + P * S * B * 128 * 32); // [P][S]
  uint64_t *empty = full + P * S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NCW = THREADS / 32 - P;  // consumer warps
  if (threadIdx.x == 0) {
    for (int i = 0; i < P * S; ++i) { mb_init(&full[i], 1); mb_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int4 *my = idx + blockIdx.x * n4_per_cta;
  // each producer p handles gather4 groups g = p, p+P, ... ; B per slot
  const size_t n_slots_total = n4_per_cta / B / 32;
  if (warp < P) {
    // producer warp: every lane issues B gather4 per slot (32*B per slot)
    int s = 0; uint32_t ph = 0;
    for (size_t k = warp; k < n_slots_total; k += P) {
      uint64_t *fb = &full[warp * S + s], *eb = &empty[warp * S + s];
      int4 r[B];
#pragma unroll
      for (int b = 0; b < B; ++b) r[b] = __ldg(my + (k * B + b) * 32 + lane);
      if (lane == 0) {
        mb_wait(eb, ph ^ 1);
        mb_expect(fb, 32 * B * 64);
      }
      __syncwarp();
      double2 *dst = slots + (size_t)(warp * S + s) * 8 * B * 32;
#pragma unroll
      for (int b = 0; b < B; ++b) gather4(dst + 8 * (b * 32 + lane), &tm, fb, r[b].x, r[b].y, r[b].z, r[b].w);
      if (++s == S) { s = 0; ph ^= 1; }
    }
  } else {
    const int cw = warp - P;
    double acc = 0;
    // consumer warp cw owns slots q = cw, cw + NCW, ... (q = p*S + sl) and
    // consumes them round by round (never waits more than one phase ahead)
    for (size_t rnd = 0;; ++rnd) {
      bool any = false;
      for (int q = cw; q < P * S; q += NCW) {
        const int p = q / S, sl = q % S;
        const size_t k = (size_t)p + (size_t)P * ((size_t)sl + (size_t)S * rnd);
        if (k >= n_slots_total) continue;
        any = true;
        uint64_t *fb = &full[q], *eb = &empty[q];
        mb_wait(fb, (uint32_t)(rnd & 1));
        const double2 *src = slots + (size_t)q * 8 * B * 32;
        for (int e = lane; e < 4 * B * 32; e += 32) acc += src[(e >> 2) * 8 + (e & 3)].x + src[(e >> 2) * 8 + (e & 3)].y;
        __syncwarp();
        if (lane == 0) mb_arrive(eb);
      }
      if (!any) break;
    }
    if (acc == 1.2345) *out = acc;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                             const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncodeFn encode = (EncodeFn)fn;
  for (size_t tb : {(size_t)32 << 20, (size_t)1 << 30}) {
    const size_t rows = tb / 16;
    double *tab; CK(cudaMalloc(&tab, tb)); CK(cudaMemset(tab, 0, tb));
    CUtensorMap tm;
    cuuint64_t dims[2] = {2, rows};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {2, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, tab, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    const size_t n_g = (size_t)64 << 20;  // gathers
    std::vector<int> h(n_g);
    uint64_t x = 88172645463325252ull;
    for (size_t i = 0; i < n_g; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = (int)(x % rows); }
    int *d; CK(cudaMalloc(&d, n_g * 4)); CK(cudaMemcpy(d, h.data(), n_g * 4, cudaMemcpyHostToDevice));
    double *out; CK(cudaMalloc(&out, 8));
    const size_t n4_per_cta = n_g / 4 / sms / 64 * 64;
    cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    float ms;
#define RUN(P, S, B)                                                                                   \
    {                                                                                                  \
      const int smem = P * S * B * 128 * 32 + 2 * P * S * 8;                                                 \
      CK(cudaFuncSetAttribute(tma_gather<P, S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
      tma_gather<P, S, B><<<sms, THREADS, smem>>>(tm, (const int4 *)d, n4_per_cta, out);               \
      CK(cudaDeviceSynchronize());                                                                     \
      CK(cudaEventRecord(e0));                                                                         \
      for (int it = 0; it < 3; ++it) tma_gather<P, S, B><<<sms, THREADS, smem>>>(tm, (const int4 *)d, n4_per_cta, out); \
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));      \
      printf("table %5zu MB P=%d S=%d B=%2d: %.1f Ggathers/s\n", tb >> 20, P, S, B,                      \
             3.0 * n4_per_cta * 4 * sms / (ms * 1e-3) / 1e9);                                           \
    }
    RUN(1, 4, 1); RUN(2, 4, 1); RUN(4, 4, 1); RUN(4, 2, 2); RUN(8, 2, 1); RUN(12, 2, 1); RUN(4, 4, 2);
    CK(cudaFree(tab)); CK(cudaFree(d));
  }
  return 0;
}
