// Device-side deterministic generator of large community graphs (BASELINE
// config 5: LFR-style N = 8e6, ~1e10 directed corrections; SURVEY §7.3.1,
// §8f rank 1).  Host generation/transfer of ~30 GB is impractical, so the
// decomposition is produced directly in the stage kernel's CSR layout.
//
// Model (documented in DESIGN.md):
//  * intra: pair {a, b} of community c (local indices) is MISSING iff
//    hash(seed, c, min(a,b), max(a,b)) < q_missing * 2^32  (symmetric,
//    counter-based: any row can be regenerated on its own);
//  * inter: n_edges undirected edges, endpoint k of edge e drawn from
//    hash(seed, e, k) by inverse CDF of per-node propensities (heavy-tailed
//    degrees); edges inside one community (and loops) are dropped,
//    duplicates removed after a per-row sort (so the graph is simple and the
//    row order canonical: identical on any GPU count).
#include "common.cuh"

namespace cdk {

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ uint32_t hash4(uint64_t seed, uint32_t a, uint32_t b, uint32_t c) {
  uint32_t h = mix32((uint32_t)seed ^ 0x9e3779b9U);
  h = mix32(h ^ (uint32_t)(seed >> 32) ^ 0x85ebca6bU);
  h = mix32(h ^ a);
  h = mix32(h ^ (b + 0x27d4eb2fU));
  h = mix32(h ^ (c + 0x165667b1U));
  return h;
}

__device__ __forceinline__ bool missing_pair(uint64_t seed, uint32_t c, uint32_t a, uint32_t b,
                                             uint32_t thr) {
  const uint32_t lo = min(a, b), hi = max(a, b);
  return hash4(seed, c, lo, hi) < thr;
}

__device__ __forceinline__ int find_comm64(const int64_t *off, int64_t m, int64_t node) {
  int64_t lo = 0, hi = m;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (off[mid] <= node) lo = mid; else hi = mid;
  }
  return (int)lo;
}

// Pass layout of a community (cdk_graph.intra_split): the community's staged
// window starts at w0 = c0 rounded down to 8 (plan.py win_lo); if it is wider
// than pass_nodes (and at most 4 passes), pass q covers global nodes
// [w0 + q*pass_nodes, w0 + (q+1)*pass_nodes).
struct PassGeom {
  int np;         // passes (1 = a single run)
  int64_t c0;     // community start
  uint32_t lam;   // community size
  int64_t w0;
  uint32_t wn;
  __device__ __forceinline__ uint32_t lo(int q) const {
    if (np == 1) return 0u;
    const int64_t v = w0 + (int64_t)q * wn - c0;
    return v < 0 ? 0u : (uint32_t)v;
  }
  __device__ __forceinline__ uint32_t hi(int q) const {
    if (np == 1) return lam;
    const int64_t v = w0 + (int64_t)(q + 1) * wn - c0;
    return v > (int64_t)lam ? lam : (uint32_t)v;
  }
};

__device__ __forceinline__ PassGeom pass_geom(const cdk_gen_params &p, int c) {
  PassGeom g;
  g.c0 = p.comm_off[c];
  g.lam = (uint32_t)(p.comm_off[c + 1] - g.c0);
  g.w0 = g.c0 & ~(int64_t)7;
  g.wn = p.pass_nodes;
  const int64_t width = ((g.c0 + g.lam + 7) & ~(int64_t)7) - g.w0;
  g.np = 1;
  if (g.wn && width > (int64_t)g.wn) {
    const int64_t q = (width + g.wn - 1) / g.wn;
    g.np = q <= 4 ? (int)q : 1;  // wider: unstaged global gathers, one run
  }
  return g;
}

// warp per row: count missing partners per pass (ballot)
__global__ void gen_intra_count_kernel(cdk_gen_params p, int64_t *padded, int64_t *raw,
                                       uint64_t *split) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_in = p.comm_off[p.n_comm];
  const int64_t i_lo = p.row_lo, i_hi = min(p.row_hi, n_in);
  for (int64_t i = i_lo + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < i_hi;
       i += warps) {
    const int c = find_comm64(p.comm_off, p.n_comm, i);
    const PassGeom G = pass_geom(p, c);
    const uint32_t a = (uint32_t)(i - G.c0);
    int64_t pad = 0, tot = 0;
    uint64_t sp = 0;
    for (int q = 0; q < G.np; ++q) {
      if (q > 0) sp |= (uint64_t)(pad >> 3) << (16 * (q - 1));
      const uint32_t lo = G.lo(q), hi = G.hi(q);
      int64_t count = 0;
      for (uint32_t base = lo; base < hi; base += 32) {
        const uint32_t b = base + lane;
        const bool m = b < hi && b != a && missing_pair(p.seed, (uint32_t)c, a, b, p.miss_thr);
        count += __popc(__ballot_sync(FULL, m));
      }
      tot += count;
      pad += (count + 7) & ~(int64_t)7;
    }
    if (lane == 0) {
      padded[i] = pad;
      if (raw) raw[i] = tot;
      if (split) split[i] = sp;
    }
  }
}

// warp per row: write local columns ascending per pass sub-run, pad with 0xFFFF
__global__ void gen_intra_fill_kernel(cdk_gen_params p, const int64_t *ptr, const uint64_t *split,
                                      uint16_t *col) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_in = p.comm_off[p.n_comm];
  const int64_t i_lo = p.row_lo, i_hi = min(p.row_hi, n_in);
  for (int64_t i = i_lo + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < i_hi;
       i += warps) {
    const int c = find_comm64(p.comm_off, p.n_comm, i);
    const PassGeom G = pass_geom(p, c);
    const uint32_t a = (uint32_t)(i - G.c0);
    const uint64_t sp = (G.np > 1) ? split[i] : 0ull;
    for (int q = 0; q < G.np; ++q) {
      int64_t pos = ptr[i] + (q ? 8 * (int64_t)((sp >> (16 * (q - 1))) & 0xFFFFu) : 0);
      const int64_t end = (q + 1 < G.np) ? ptr[i] + 8 * (int64_t)((sp >> (16 * q)) & 0xFFFFu)
                                         : ptr[i + 1];
      const uint32_t lo = G.lo(q), hi = G.hi(q);
      for (uint32_t base = lo; base < hi; base += 32) {
        const uint32_t b = base + lane;
        const bool m = b < hi && b != a && missing_pair(p.seed, (uint32_t)c, a, b, p.miss_thr);
        const unsigned bal = __ballot_sync(FULL, m);
        if (m) col[pos + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)b;
        pos += __popc(bal);
      }
      for (int64_t r = pos + lane; r < end; r += 32) col[r] = (uint16_t)0xFFFF;
    }
  }
}

// endpoint k of inter edge e: node by inverse CDF of the per-node inter
// propensities (node_cdf[i] = cumulative normalised weight up to node i,
// node_cdf[n-1] == 1): the first i with node_cdf[i] > u
__device__ __forceinline__ int64_t edge_end(const cdk_gen_params &p, int64_t e, uint32_t k,
                                            int *comm) {
  const uint32_t h = hash4(p.seed ^ 0xabcdef12345ULL, (uint32_t)e, (uint32_t)(e >> 32), k);
  const double u = ((double)h + 0.5) * (1.0 / 4294967296.0);
  int64_t lo = 0, hi = p.n_rows - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(p.node_cdf + mid) > u) hi = mid; else lo = mid + 1;
  }
  *comm = lo < p.comm_off[p.n_comm] ? find_comm64(p.comm_off, p.n_comm, lo) : -1 - (int)lo;
  return lo;
}

__global__ void gen_inter_count_kernel(cdk_gen_params p, unsigned long long *cnt) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < p.n_inter_edges; e += stride) {
    int cu, cv;
    const int64_t u = edge_end(p, e, 0, &cu), v = edge_end(p, e, 1, &cv);
    if (cu == cv) continue;
    if (u >= p.row_lo && u < p.row_hi) atomicAdd(cnt + u, 1ull);
    if (v >= p.row_lo && v < p.row_hi) atomicAdd(cnt + v, 1ull);
  }
}

__global__ void gen_inter_fill_kernel(cdk_gen_params p, unsigned long long *cursor, int32_t *col) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < p.n_inter_edges; e += stride) {
    int cu, cv;
    const int64_t u = edge_end(p, e, 0, &cu), v = edge_end(p, e, 1, &cv);
    if (cu == cv) continue;
    if (u >= p.row_lo && u < p.row_hi) col[atomicAdd(cursor + u, 1ull)] = (int32_t)v;
    if (v >= p.row_lo && v < p.row_hi) col[atomicAdd(cursor + v, 1ull)] = (int32_t)u;
  }
}

// per row: sort the inter run (block-wide bitonic in shared memory, rows up to
// 8192 entries; longer rows fall back to a serial insertion sort), drop
// duplicates, write the unique count
__global__ void __launch_bounds__(512) gen_inter_sort_kernel(int64_t n_rows, const int64_t *ptr,
                                                             int32_t *col, int64_t *uniq) {
  __shared__ int32_t buf[8192];
  for (int64_t i = blockIdx.x; i < n_rows; i += gridDim.x) {
    const int64_t b = ptr[i], e = ptr[i + 1];
    const int len = (int)(e - b);
    if (len <= 8192) {
      int n2 = 1;
      while (n2 < len) n2 <<= 1;
      for (int q = threadIdx.x; q < n2; q += blockDim.x) buf[q] = (q < len) ? col[b + q] : INT32_MAX;
      __syncthreads();
      for (int k = 2; k <= n2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
          for (int q = threadIdx.x; q < n2; q += blockDim.x) {
            const int l = q ^ j;
            if (l > q) {
              const bool up = (q & k) == 0;
              const int32_t x = buf[q], y = buf[l];
              if ((x > y) == up) {
                buf[q] = y;
                buf[l] = x;
              }
            }
          }
          __syncthreads();
        }
      }
      for (int q = threadIdx.x; q < len; q += blockDim.x) col[b + q] = buf[q];
      __syncthreads();
    } else if (threadIdx.x == 0) {
      for (int64_t q = b + 1; q < e; ++q) {
        const int32_t x = col[q];
        int64_t r = q - 1;
        while (r >= b && col[r] > x) {
          col[r + 1] = col[r];
          --r;
        }
        col[r + 1] = x;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // dedupe in place
      int64_t w = b;
      for (int64_t q = b; q < e; ++q)
        if (q == b || col[q] != col[q - 1]) col[w++] = col[q];
      uniq[i] = w - b;
    }
    __syncthreads();
  }
}

// compact rows to the deduplicated lengths
__global__ void gen_inter_compact_kernel(int64_t n_rows, const int64_t *ptr_raw,
                                         const int64_t *ptr_new, const int32_t *col_raw,
                                         int32_t *col_new) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_rows; i += warps) {
    const int64_t n = ptr_new[i + 1] - ptr_new[i];
    for (int64_t q = lane; q < n; q += 32) col_new[ptr_new[i] + q] = col_raw[ptr_raw[i] + q];
  }
}

static unsigned gen_grid(int64_t work, int per_block) {
  int64_t g = (work + per_block - 1) / per_block;
  if (g > 148 * 64) g = 148 * 64;
  return (unsigned)(g > 0 ? g : 1);
}

}  // namespace cdk

using namespace cdk;

extern "C" int cdk_gen_intra_count(const cdk_gen_params *p, int64_t *padded, int64_t *raw,
                                   uint64_t *split, void *stream) {
  if (!p || p->n_comm < 0 || !padded || p->row_lo < 0 || p->row_hi > p->n_rows ||
      p->row_lo > p->row_hi)
    return set_error("gen: bad params"), CDK_INPUT;
  gen_intra_count_kernel<<<gen_grid(p->n_rows, 8), 256, 0, as_stream(stream)>>>(*p, padded, raw,
                                                                                 split);
  CDK_CHECK_LAUNCH("gen_intra_count_kernel");
  return CDK_OK;
}

extern "C" int cdk_gen_intra_fill(const cdk_gen_params *p, const int64_t *ptr,
                                  const uint64_t *split, uint16_t *col, void *stream) {
  if (!p) return CDK_INPUT;
  gen_intra_fill_kernel<<<gen_grid(p->n_rows, 8), 256, 0, as_stream(stream)>>>(*p, ptr, split,
                                                                                col);
  CDK_CHECK_LAUNCH("gen_intra_fill_kernel");
  return CDK_OK;
}

extern "C" int cdk_gen_inter_count(const cdk_gen_params *p, int64_t *cnt, void *stream) {
  if (!p) return CDK_INPUT;
  gen_inter_count_kernel<<<gen_grid(p->n_inter_edges, 256), 256, 0, as_stream(stream)>>>(
      *p, reinterpret_cast<unsigned long long *>(cnt));
  CDK_CHECK_LAUNCH("gen_inter_count_kernel");
  return CDK_OK;
}

extern "C" int cdk_gen_inter_fill(const cdk_gen_params *p, int64_t *cursor, int32_t *col,
                                  void *stream) {
  if (!p) return CDK_INPUT;
  gen_inter_fill_kernel<<<gen_grid(p->n_inter_edges, 256), 256, 0, as_stream(stream)>>>(
      *p, reinterpret_cast<unsigned long long *>(cursor), col);
  CDK_CHECK_LAUNCH("gen_inter_fill_kernel");
  return CDK_OK;
}

extern "C" int cdk_gen_inter_sort(int64_t n_rows, const int64_t *ptr, int32_t *col, int64_t *uniq,
                                  void *stream) {
  gen_inter_sort_kernel<<<gen_grid(n_rows, 1), 512, 0, as_stream(stream)>>>(n_rows, ptr, col, uniq);
  CDK_CHECK_LAUNCH("gen_inter_sort_kernel");
  return CDK_OK;
}

extern "C" int cdk_gen_inter_compact(int64_t n_rows, const int64_t *ptr_raw,
                                     const int64_t *ptr_new, const int32_t *col_raw,
                                     int32_t *col_new, void *stream) {
  gen_inter_compact_kernel<<<gen_grid(n_rows, 8), 256, 0, as_stream(stream)>>>(
      n_rows, ptr_raw, ptr_new, col_raw, col_new);
  CDK_CHECK_LAUNCH("gen_inter_compact_kernel");
  return CDK_OK;
}

namespace cdk {
// add a per-row delta to every non-padding intra column (segment rebasing)
__global__ void gen_rebase_kernel(int64_t n_rows, const int64_t *ptr, const int32_t *delta,
                                  uint16_t *col) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_rows; i += warps) {
    const int32_t d = delta[i];
    if (d == 0) continue;
    for (int64_t q = ptr[i] + lane; q < ptr[i + 1]; q += 32) {
      const uint16_t v = col[q];
      if (v != (uint16_t)0xFFFF) col[q] = (uint16_t)(v + d);
    }
  }
}
}  // namespace cdk

extern "C" int cdk_gen_rebase(int64_t n_rows, const int64_t *ptr, const int32_t *delta,
                              uint16_t *col, void *stream) {
  cdk::gen_rebase_kernel<<<cdk::gen_grid(n_rows, 8), 256, 0, cdk::as_stream(stream)>>>(
      n_rows, ptr, delta, col);
  CDK_CHECK_LAUNCH("gen_rebase_kernel");
  return CDK_OK;
}

namespace cdk {
// warp per row: block sub-run starts of a sorted inter run (ballot counts)
__global__ void inter_split_kernel(int64_t n_rows, const int64_t *ptr, const int32_t *col,
                                   int blocks, int block_nodes, uint64_t *split, int *bad) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_rows; i += warps) {
    const int64_t b = ptr[i], e = ptr[i + 1];
    if (e - b > 0xFFFF) {
      if (lane == 0) atomicExch(bad, 1);
      continue;
    }
    int cnt[4] = {0, 0, 0, 0};  // entries below block boundary q+1
    for (int64_t q = b + lane; q < e; q += 32) {
      const int c = col[q];
#pragma unroll
      for (int k = 0; k < 3; ++k) cnt[k] += (k + 1 < blocks && c < (k + 1) * block_nodes) ? 1 : 0;
    }
    uint64_t w = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      int v = cnt[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
      if (k + 1 < blocks) w |= (uint64_t)v << (16 * k);
    }
    if (lane == 0) split[i] = w;
  }
}
}  // namespace cdk

extern "C" int cdk_inter_split(int64_t n_rows, const int64_t *ptr, const int32_t *col, int blocks,
                               int block_nodes, uint64_t *split, void *stream) {
  if (blocks < 2 || blocks > 4 || block_nodes <= 0) return set_error("inter_split: bad blocks"), CDK_INPUT;
  int *bad = nullptr;
  cudaError_t e = cudaMallocAsync(&bad, sizeof(int), as_stream(stream));
  if (e != cudaSuccess) return cuda_status(e, "inter_split alloc");
  cudaMemsetAsync(bad, 0, sizeof(int), as_stream(stream));
  cdk::inter_split_kernel<<<cdk::gen_grid(n_rows, 8), 256, 0, as_stream(stream)>>>(
      n_rows, ptr, col, blocks, block_nodes, split, bad);
  CDK_CHECK_LAUNCH("inter_split_kernel");
  int hbad = 0;
  cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, as_stream(stream));
  cudaFreeAsync(bad, as_stream(stream));
  e = cudaStreamSynchronize(as_stream(stream));
  if (e != cudaSuccess) return cuda_status(e, "inter_split");
  if (hbad) return set_error("inter_split: a row has more than 65535 inter entries"), CDK_INPUT;
  return CDK_OK;
}

namespace cdk {
// Device twin of cdk_host_bank_order (csrc/host_plan.cpp), out of place: per
// run (a row, or a pass sub-run of cdk_graph.intra_split) a stable counting
// sort by bank group (column mod 8, pads -> pad_bank), then the sorted s-th
// entry is dealt to phase j of round r in closed form (rounds 0..c-1 cover
// all P = 8*nblk phases, later rounds only the full blocks' phases) and
// written to position 64*(j/8) + 8*r + j%8 of the run.
__global__ void bank_order_kernel(int64_t n_rows, const int64_t *ptr, const uint64_t *split,
                                  const uint16_t *src, uint16_t *dst, int pad_bank) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_rows; i += warps) {
    const int64_t a = ptr[i], e = ptr[i + 1];
    const uint64_t sw = split ? split[i] : 0ull;
    int64_t bnd[5];
    int nr = 0;
    bnd[nr++] = a;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int64_t o = (int64_t)((sw >> (16 * q)) & 0xFFFFu);
      if (o) bnd[nr++] = a + 8 * o;
    }
    bnd[nr] = e;
    for (int r = 0; r < nr; ++r) {
      const int64_t rs = bnd[r], re = bnd[r + 1];
      const int64_t L = re - rs;
      if (L <= 8) {
        for (int64_t q = rs + lane; q < re; q += 32) dst[q] = src[q];
        continue;
      }
      int cnt[8];
#pragma unroll
      for (int b = 0; b < 8; ++b) cnt[b] = 0;
      for (int64_t q0 = rs; q0 < re; q0 += 32) {
        const int64_t q = q0 + lane;
        const uint16_t v = q < re ? src[q] : (uint16_t)0;
        const int bank = q < re ? (v == (uint16_t)0xFFFF ? pad_bank : (v & 7)) : -1;
#pragma unroll
        for (int b = 0; b < 8; ++b) cnt[b] += __popc(__ballot_sync(FULL, bank == b));
      }
      int base[8];
      int acc = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        base[b] = acc;
        acc += cnt[b];
      }
      const int64_t nblk = (L + 63) / 64, P = 8 * nblk, Pf = P - 8;
      const int64_t c = (L % 64 == 0) ? 8 : (L % 64) / 8;
      for (int64_t q0 = rs; q0 < re; q0 += 32) {
        const int64_t q = q0 + lane;
        const uint16_t v = q < re ? src[q] : (uint16_t)0;
        const int bank = q < re ? (v == (uint16_t)0xFFFF ? pad_bank : (v & 7)) : -1;
        int64_t sidx = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          const unsigned m = __ballot_sync(FULL, bank == b);
          if (bank == b) sidx = base[b] + __popc(m & lt);
          base[b] += __popc(m);
        }
        if (q < re) {
          int64_t rd, j;
          if (sidx < c * P) {
            rd = sidx / P;
            j = sidx % P;
          } else {
            const int64_t s2 = sidx - c * P;
            rd = c + s2 / Pf;
            j = s2 % Pf;
          }
          dst[rs + 64 * (j >> 3) + 8 * rd + (j & 7)] = v;
        }
      }
    }
  }
}
}  // namespace cdk

extern "C" int cdk_bank_order(int64_t n_rows, const int64_t *ptr, const uint64_t *split,
                              const uint16_t *src, uint16_t *dst, int pad_bank, void *stream) {
  if (n_rows < 0 || !ptr || !src || !dst || src == dst) return set_error("bank_order: bad args"), CDK_INPUT;
  cdk::bank_order_kernel<<<cdk::gen_grid(n_rows, 8), 256, 0, as_stream(stream)>>>(
      n_rows, ptr, split, src, dst, pad_bank & 7);
  CDK_CHECK_LAUNCH("bank_order_kernel");
  return CDK_OK;
}
