// Microbenchmarks for the stage-kernel design (B200, sm_100a):
//  A) bulk async copy (TMA engine) streaming: 1 CTA/SM, one producer thread,
//     ring of S slots x B bytes, consumers release slots immediately.
//  B) plain LDG.128 streaming with all threads (reference).
//  C) shared-memory gather: random uint16 indices into a 64K-node window of
//     double2, 16-byte LDS per index, accumulate (with/without bank-conflict-
//     free index ordering).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mb tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile("{\n.reg .pred p;\nLAB_WAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra LAB_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// A) TMA streaming
template <int S>
__global__ void __launch_bounds__(256, 1) tma_stream(const char *src, size_t per_cta, int B, unsigned long long *sink) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int tid = threadIdx.x;
  if (tid == 0) { for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); } }
  __syncthreads();
  const char *base = src + (size_t)blockIdx.x * per_cta;
  const int ntiles = (int)(per_cta / B);
  if (tid == 0) {
    for (int k = 0; k < ntiles; ++k) {
      const int b = k % S, n = k / S;
      if (n > 0) mbar_wait(&empty[b], (n - 1) & 1);
      mbar_expect_tx(&full[b], B);
      bulk_g2s(sm + (size_t)b * B, base + (size_t)k * B, B, &full[b]);
    }
  } else if (tid == 32) {
    unsigned long long acc = 0;
    for (int k = 0; k < ntiles; ++k) {
      const int b = k % S, n = k / S;
      mbar_wait(&full[b], n & 1);
      acc += sm[(size_t)b * B + (k & 127)];
      mbar_arrive(&empty[b]);
    }
    atomicAdd(sink, acc);
  }
}

// B) LDG streaming (all threads, 16B loads, unrolled)
__global__ void __launch_bounds__(1024, 1) ldg_stream(const int4 *src, size_t n4_per_cta, unsigned long long *sink) {
  const int4 *base = src + (size_t)blockIdx.x * n4_per_cta;
  int acc = 0;
  for (size_t i = threadIdx.x; i < n4_per_cta; i += 4 * blockDim.x) {
    int4 v0 = __ldg(base + i);
    int4 v1 = (i + blockDim.x < n4_per_cta) ? __ldg(base + i + blockDim.x) : make_int4(0,0,0,0);
    int4 v2 = (i + 2*blockDim.x < n4_per_cta) ? __ldg(base + i + 2*blockDim.x) : make_int4(0,0,0,0);
    int4 v3 = (i + 3*blockDim.x < n4_per_cta) ? __ldg(base + i + 3*blockDim.x) : make_int4(0,0,0,0);
    acc ^= v0.x ^ v1.y ^ v2.z ^ v3.w;
  }
  if (acc == 0x7fffffff) atomicAdd(sink, 1ull);
}

// C) smem gather: window W double2 in smem, indices from global (uint16), each lane 8 per uint4
__global__ void __launch_bounds__(1024, 1) smem_gather(const uint4 *idx, size_t n_per_cta_u4, int W, double *out) {
  extern __shared__ __align__(128) double2 zs[];
  for (int i = threadIdx.x; i < W; i += blockDim.x) zs[i] = make_double2(i * 1e-3, -i * 1e-3);
  __syncthreads();
  const uint4 *base = idx + (size_t)blockIdx.x * n_per_cta_u4;
  double sr = 0, si = 0;
  for (size_t i = threadIdx.x; i < n_per_cta_u4; i += blockDim.x) {
    const uint4 w = __ldg(base + i);
    const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t u = (wv[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu;
      const double2 z = zs[u];
      sr -= z.x; si -= z.y;
    }
  }
  if (sr == 12345.0) out[0] = si;
}

int main() {
  const bool only_gather = getenv("ONLY_GATHER") != nullptr;
  int dev = 0; CK(cudaSetDevice(dev));
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const size_t total = (size_t)1 << 30;  // 1 GiB stream
  char *src; CK(cudaMalloc(&src, total)); CK(cudaMemset(src, 1, total));
  unsigned long long *sink; CK(cudaMalloc(&sink, 8));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const size_t per_cta = total / sms / 65536 * 65536;
  auto run_tma = [&](auto kern, int S, int B) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S * B));
    kern<<<sms, 256, S * B>>>(src, per_cta, B, sink);  // warm
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) kern<<<sms, 256, S * B>>>(src, per_cta, B, sink);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("TMA stream S=%d B=%6d: %.1f GB/s\n", S, B, 5.0 * per_cta * sms / (ms * 1e-3) / 1e9);
  };
  if (!only_gather) for (int B : {4096, 8192, 16384, 32768}) {
    run_tma(tma_stream<2>, 2, B);
    run_tma(tma_stream<4>, 4, B);
    if (B <= 16384) run_tma(tma_stream<8>, 8, B);
  }
  if (!only_gather) {
    const size_t n4 = per_cta / 16;
    ldg_stream<<<sms, 1024>>>((const int4 *)src, n4, sink);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) ldg_stream<<<sms, 1024>>>((const int4 *)src, n4, sink);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("LDG stream 1024thr: %.1f GB/s\n", 5.0 * per_cta * sms / (ms * 1e-3) / 1e9);
  }
  // C) gathers: 64 MB of indices (32M entries), window W nodes (WIN env, default 6000)
  {
    const int W = getenv("WIN") ? atoi(getenv("WIN")) : 6000;
    const size_t n_idx = (size_t)32 << 20;
    std::vector<uint16_t> h(n_idx);
    uint64_t x = 88172645463325252ull;
    for (size_t i = 0; i < n_idx; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = (uint16_t)(x % W); }
    uint16_t *d; CK(cudaMalloc(&d, n_idx * 2)); CK(cudaMemcpy(d, h.data(), n_idx * 2, cudaMemcpyHostToDevice));
    double *out; CK(cudaMalloc(&out, 8));
    const size_t per_cta_u4 = n_idx / 8 / sms;
    CK(cudaFuncSetAttribute(smem_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, W * 16));
    smem_gather<<<sms, 1024, W * 16>>>((const uint4 *)d, per_cta_u4, W, out);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) smem_gather<<<sms, 1024, W * 16>>>((const uint4 *)d, per_cta_u4, W, out);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    const double ent = 5.0 * per_cta_u4 * 8 * sms;
    printf("smem gather random: %.2f Gentries/s (%.3f ns per 1M... ) = %.3f cycles/entry/SM @1.9GHz\n",
           ent / (ms * 1e-3) / 1e9, 0.0, (ms * 1e-3) * 1.9e9 * sms / ent);
    // conflict-free ordering: within each group of 8 consecutive lanes' k-th entry make residues distinct
    for (size_t i = 0; i < n_idx; i += 64) {
      // block of 64 entries = 8 lanes x 8 entries (lane-major: lane l has entries i+8l..i+8l+7)
      for (int k = 0; k < 8; ++k)
        for (int l = 0; l < 8; ++l) {
          size_t pos = i + 8 * l + k;
          uint16_t v = h[pos];
          v = (uint16_t)((v / 8) * 8 + ((l + k) % 8));
          if (v >= W) v -= 8;
          h[pos] = v;
        }
    }
    CK(cudaMemcpy(d, h.data(), n_idx * 2, cudaMemcpyHostToDevice));
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) smem_gather<<<sms, 1024, W * 16>>>((const uint4 *)d, per_cta_u4, W, out);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("smem gather conflict-free(8-lane phases): %.2f Gentries/s = %.3f cycles/entry/SM\n",
           ent / (ms * 1e-3) / 1e9, (ms * 1e-3) * 1.9e9 * sms / ent);
  }
  return 0;
}
