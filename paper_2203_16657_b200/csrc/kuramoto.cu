// Fused CIA Kuramoto right-hand side inside RK4 stages (sm_100a).
//
// Replaces, per RHS evaluation, the reference chain
//   order_params_blocks (_kernels.py:34-51)  -> community sums R_c = sum_{l in c} z_l
//   dense_complex       (_kernels.py:124-149) -> K/N Im(R_c conj z_m)
//   pairs_trig          (_kernels.py:246-283) -> K/N sum_l s_ml sin(x_l - x_m)
// with ONE kernel per RK4 stage over a directed CSR of S (diagonal dropped: it
// contributes sin(0) = 0).  Per row i of community c:
//   acc_i = -sum_{j intra-missing} z_j + sum_{j inter} z_j        (gathers)
//   k_i   = omega_i + K/N Im(R_c conj z_i) + K/N Im(acc_i conj z_i)
// then the RK4 stage update, z_next = exp(i theta_next) and the per-rblock
// partial of R for the next stage.  The last CTA to finish a community
// reduces its rblock partials (fixed order) into R_next[c], so the next stage
// kernel starts with every community observable ready: no extra launch.
//
// Gathers of intra-community neighbours hit a shared-memory copy of the
// community's z (staged once per segment); inter-community gathers go to
// global memory (L2).  8 lanes per row, 4 rows per warp pass, 32-row rblocks
// per warp; all accumulation orders are fixed => bitwise deterministic and
// independent of the CTA schedule (and so of the GPU count).
#include "common.cuh"

namespace cdk {

#ifdef CDK_DEBUG
#define DBG_CHECK(cond, fmt, ...)                                                  \
  do {                                                                             \
    if (!(cond)) {                                                                 \
      printf("CDK_DEBUG %s:%d block %d thread %d: " fmt "\n", __FILE__, __LINE__, \
             blockIdx.x, threadIdx.x, __VA_ARGS__);                                \
      __trap();                                                                    \
    }                                                                              \
  } while (0)
#else
#define DBG_CHECK(cond, fmt, ...) \
  do {                            \
  } while (0)
#endif


struct Workspace {
  double2 *z[2];
  double *ksum;
  double2 *part[2];  // canonical rblock partials of z (ping-pong with z)
  cdk_run_status *status;
  unsigned int *bar;  // grid-barrier counter of the persistent kernel
  double2 *xacc;      // per-row inter sums (block-phased inter sweep only)
  unsigned int *peer_bar;  // fused multi-GPU exchange: this rank's barrier counter
};

static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static Workspace carve(const cdk_graph *g, void *base, size_t *total) {
  Workspace w{};
  size_t off = 0;
  char *b = reinterpret_cast<char *>(base);
  auto take = [&](size_t bytes) {
    void *p = b ? b + off : nullptr;
    off = align_up(off + bytes, 256);
    return p;
  };
  const size_t n = (size_t)g->n_rows;
  // +16: staged windows are rounded out to 8-node (128-byte) boundaries
  w.z[0] = (double2 *)take((n + 16) * sizeof(double2));
  w.z[1] = (double2 *)take((n + 16) * sizeof(double2));
  w.ksum = (double *)take((n + 4) * sizeof(double));  // bulk copies read 16-byte units
  w.part[0] = (double2 *)take(((size_t)g->n_rblk + 1) * sizeof(double2));
  w.part[1] = (double2 *)take(((size_t)g->n_rblk + 1) * sizeof(double2));
  w.status = (cdk_run_status *)take(sizeof(cdk_run_status));
  w.bar = (unsigned int *)take(256);
  w.xacc = g->inter_blocks > 0 ? (double2 *)take(n * sizeof(double2)) : nullptr;
  w.peer_bar = (unsigned int *)take(256);
  if (total) *total = off;
  return w;
}

struct StageArgs {
  cdk_graph g;
  const double2 *z_in;
  double2 *z_out;
  const double2 *part_in;  // rblock partials of z_in (community sums are reduced in-kernel)
  double2 *part_out;       // rblock partials of z_out
  cdk_run_status *status;
  double *theta;
  const double *omega;
  double *ksum;
  double *out;  // MODE 0
  double2 *xacc;  // block-phased inter sums (g.inter_blocks > 0)
  // fused multi-GPU exchange: the epilogue also stores z_out rows into every
  // peer's buffer (peer_out[q], q != rank)
  double2 *const *peer_out;
  int n_peers, rank;
  int sweep_mode;  // inter sweep lanes/unroll variant (CDK_SWEEP, experiments)
  int debug_flags; // CDK_DEBUG_FLAGS (timing experiments only; results invalid):
                   // 1 = skip the inter sweep, 2 = skip the segments,
                   // 4 = drop inline inter entries, 8 = drop intra gathers
  double k_over_n;
  double h;     // stage increment (dt/2, dt/2, dt) or dt/6 at stage 4
  int64_t step_rel;
  unsigned long long *prof;  // CDK_PROFILE builds: per-CTA phase cycles
  unsigned long long *cta_cycles;  // ELL stage kernels: per-CTA cycles (planner calibration)
};

// Canonical community sum R_c of the rblock partials: 8 lanes, lane t sums
// partials b0+t, b0+t+8, ... in order, then a fixed xor butterfly (4, 2, 1).
// Used by every producer of R (prepare and all stage kernels) so R is
// bitwise independent of which CTA/GPU reduces it.
__device__ __forceinline__ double2 reduce_comm8(const double2 *part, int b0, int b1, int t,
                                                unsigned mask) {
  double sr = 0.0, si = 0.0;
  for (int b = b0 + t; b < b1; b += 8) {
    double2 v = ldcg2(part + b);
    sr += v.x;
    si += v.y;
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    sr += __shfl_xor_sync(mask, sr, o);
    si += __shfl_xor_sync(mask, si, o);
  }
  return make_double2(sr, si);
}

// ---- bulk async copy (TMA engine, non-tensor form) + mbarrier helpers -----
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LAB_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra LAB_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ double2 lds_d2(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

// 8 uint16 intra columns (one 16-byte chunk): subtract their z (sign -1).
// Staged: explicit ld.shared from the window (32-bit shared address),
// branch-free, padding (0xFFFF) clamped onto a zero slot one past the window
// capacity.  Unstaged (global, huge communities / NONE pool): predicated loads.
#ifndef CDK_LDS_BATCH
#define CDK_LDS_BATCH 8
#endif
__device__ __forceinline__ void gather8_smem(const uint4 w, uint32_t zs_addr, uint32_t zero_slot,
                                             double &sr, double &si) {
  // all loads of a batch issued before any add: the shared-memory latency is
  // paid once per batch, not once per pair of entries (measured: with two
  // loads in flight per warp the gather was latency-bound at ~0.45
  // cycles/entry/SM); fixed combine order
  const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
  constexpr int B = CDK_LDS_BATCH;
  double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
#pragma unroll
  for (int k0 = 0; k0 < 8; k0 += B) {
    double2 z[B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const uint32_t u = (wv[(k0 + k) >> 1] >> (((k0 + k) & 1) * 16)) & 0xFFFFu;
      z[k] = lds_d2(zs_addr + (min(u, zero_slot) << 4));
    }
#pragma unroll
    for (int k = 0; k < B; k += 2) {
      ar += z[k].x;
      ai += z[k].y;
      br += z[k + 1].x;
      bi += z[k + 1].y;
    }
  }
  sr -= ar + br;
  si -= ai + bi;
}

__device__ __forceinline__ void gather8_global(const uint4 w, const double2 *__restrict__ zbase,
                                               double &sr, double &si) {
  const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t u = (wv[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu;
    if (u != CDK_INTRA_PAD) {
      const double2 z = __ldcg(zbase + u);
      sr -= z.x;
      si -= z.y;
    }
  }
}

// ---------------------------------------------------------------------------
// Stage kernel.  One CTA (1024 threads = 128 groups of 8 lanes) per SM,
// persistent over its cost-balanced segments.  Per segment:
//  1. one thread issues bulk async copies (TMA engine) of the segment's node
//     window of z_in, its row-pointer slices and the epilogue inputs (theta,
//     omega, ksum) into shared memory, all completing on one mbarrier;
//  2. gather: groups claim rows from a shared counter (dynamic balance); each
//     lane streams 16-byte chunks (8 uint16 columns) of the row's intra run
//     with the next row's chunks already in flight (1-row-ahead prefetch) and
//     gathers z from the window (bank-conflict-free entry order, host-side);
//     inter entries gather z from global memory (L2); the group reduces (fixed
//     butterfly) into a shared row accumulator;
//  3. epilogue (after a CTA barrier): warps take rblocks, lane = row:
//     k = omega + K/N Im((R_c + acc) conj z), RK4 stage update, z_next =
//     exp(i theta_next), canonical rblock partial; the warp that completes a
//     community's last rblock reduces R_next[c].
// Communities above the window capacity (and the NONE pool) gather intra
// neighbours from global memory; everything else is identical.
// ---------------------------------------------------------------------------
#ifndef CDK_STAGE_THREADS
#define CDK_STAGE_THREADS 896  // measured: 896 ~ 768 > 640 > 1024 threads (register room)
#endif
#ifndef CDK_STAGE_MINBLOCKS
#define CDK_STAGE_MINBLOCKS 1  // resident stage CTAs per SM the build targets
#endif
constexpr int NTHREADS = CDK_STAGE_THREADS;
constexpr int NWARPS = NTHREADS / 32;
constexpr int NGROUPS = NTHREADS / 8;
constexpr int SWEEP_THREADS = 1024;  // inter sweep launch (no shared memory, own config)

struct SegSmem {  // carve-up of dynamic shared memory (all 16-byte aligned)
  double2 *acc;     // [cap4]   row sums, index i - row0
  int64_t *sip;     // [cap4]   intra_ptr[row0a ..]
  int64_t *sxp;     // [cap4]   inter_ptr[row0a ..]
  double *sth;      // [cap4]   theta[row0a ..]
  double *som;      // [cap4]   omega[row0a ..]
  double *sks;      // [cap4]   ksum[row0a ..]
  double2 *zs;      // [smem_nodes + 8] window + zero slot
  int32_t *sxc;     // [xs_cap + 4] staged inter columns of the segment (xs_cap > 0)
};

__host__ __device__ inline size_t cap4_of(int cap) { return (size_t)cap + 4; }

__host__ __device__ inline size_t stage_smem_bytes(int cap, int smem_nodes, int xs_cap = 0) {
  return cap4_of(cap) * (16 + 5 * 8) + ((size_t)smem_nodes + 8) * 16 +
         (xs_cap > 0 ? ((size_t)xs_cap + 4) * 4 : 0);
}

__device__ __forceinline__ SegSmem carve_smem(unsigned char *base, int cap, int smem_nodes) {
  SegSmem m;
  const size_t c4 = cap4_of(cap);
  m.acc = reinterpret_cast<double2 *>(base);
  m.sip = reinterpret_cast<int64_t *>(m.acc + c4);
  m.sxp = m.sip + c4;
  m.sth = reinterpret_cast<double *>(m.sxp + c4);
  m.som = m.sth + c4;
  m.sks = m.som + c4;
  m.zs = reinterpret_cast<double2 *>(m.sks + c4);
  m.sxc = reinterpret_cast<int32_t *>(m.zs + smem_nodes + 8);
  return m;
}

constexpr int SEG_MAX_COMM = 64;  // communities per segment (planner cap)

// one row of the group's software pipeline (offsets relative to the segment)
struct RowPipe {
  int e1, p;    // intra run end, this lane's first chunk position
  int x0, x1;   // inter run
  int j;        // this lane's first inter column (or -1)
  uint4 c0, c1; // this lane's first two 16-byte column chunks
  double2 z;    // z of column j
};

// z_in / partial reads: L2-coherent (.cg) so a persistent multi-stage launch
// never sees a stale L1 line of a buffer another CTA rewrote since.
__device__ __forceinline__ double2 ldz(const double2 *p) { return __ldcg(p); }

// Gather phase of one segment: rows r = grp, grp + NG, ... (NG = 1024/LPR
// groups of LPR lanes); 3-deep pipeline per group:
//   C: pointers + first inter column (2 rows ahead)
//   B: first two column chunks + z of the inter column (1 row ahead)
//   A: gathers, tails, reduction -> acc[r]
// Lane t of a row reads the 8 entries [8t, 8t+8) of every 8*LPR-entry block,
// so for LPR >= 8 one quarter-warp phase (8 lanes) covers one 64-entry block
// and the host bank ordering (cdk_host_bank_order) is conflict-free; for
// LPR = 4 a phase spans two rows (distinct within each row).
// MULTI: the segment is staged in window passes (sub-runs per row); INLINE:
// inter entries ride in the row pipeline (else: separate phase / sweep).
// Compile-time so the common single-pass inline path carries no extra state.
template <int LPR, bool MULTI, bool INLINE>
__device__ __forceinline__ void gather_phase(const StageArgs &a, const SegSmem &sm, int nrows,
                                             int64_t row0, int64_t row0a, int64_t ebase,
                                             int64_t xbase, bool staged, uint32_t zs_addr,
                                             uint32_t zero_slot, const double2 *zglob,
                                             const uint4 *__restrict__ colv,
                                             const int32_t *__restrict__ xcol, int pass,
                                             int npass, const int32_t *sxc) {
  constexpr int NG = NTHREADS / LPR;
  constexpr int STRIDE = 8 * LPR;
  const int tid = threadIdx.x, lane = tid & 31;
  const int t = lane & (LPR - 1);
  const int grp = tid / LPR;
  const unsigned gmask = (LPR == 32) ? FULL : (((1u << LPR) - 1u) << (lane & ~(LPR - 1)));
  const double2 *__restrict__ z_in = a.z_in;
  const uint4 padv = make_uint4(~0u, ~0u, ~0u, ~0u);
  auto stage_ptr = [&](int r, RowPipe &R) {
    if (r < nrows) {
      const int64_t li = row0 + r - row0a;
      int e0 = (int)(sm.sip[li] - ebase);
      R.e1 = (int)(sm.sip[li + 1] - ebase);
      if (MULTI) {  // this pass's sub-run (cdk_graph.intra_split)
        const uint64_t sw = __ldg(a.g.intra_split + row0 + r);
        if (pass + 1 < npass) R.e1 = e0 + 8 * (int)((sw >> (16 * pass)) & 0xFFFFu);
        if (pass > 0) e0 += 8 * (int)((sw >> (16 * (pass - 1))) & 0xFFFFu);
      }
      if (INLINE) {  // inter entries: in pass 0
        R.x0 = (int)(sm.sxp[li] - xbase);
        R.x1 = (!MULTI || pass == 0) ? (int)(sm.sxp[li + 1] - xbase) : R.x0;
      } else {
        R.x0 = R.x1 = 0;
      }
      R.p = e0 + 8 * t;
      if (sxc) {  // staged inter columns: the z gather goes out two rows ahead
        R.j = (R.x0 + t < R.x1) ? sxc[R.x0 + t] : -1;
        R.z = (R.j >= 0) ? ldz(z_in + R.j) : make_double2(0.0, 0.0);
      } else {
        R.j = (R.x0 + t < R.x1) ? ldg(xcol + R.x0 + t) : -1;
      }
    }
  };
  auto stage_data = [&](int r, RowPipe &R) {
    if (r < nrows) {
      R.c0 = (R.p < R.e1) ? ldg(colv + (R.p >> 3)) : padv;
      R.c1 = (R.p + STRIDE < R.e1) ? ldg(colv + ((R.p + STRIDE) >> 3)) : padv;
      if (!sxc) R.z = (R.j >= 0) ? ldz(z_in + R.j) : make_double2(0.0, 0.0);
    }
  };
  RowPipe A{}, B{}, C{};
  int r = grp;
  stage_ptr(r, A);
  stage_ptr(r + NG, B);
  stage_data(r, A);
  for (; r < nrows; r += NG) {
    stage_ptr(r + 2 * NG, C);
    stage_data(r + NG, B);
    double sr = 0.0, si = 0.0;
    if (staged) {
      if (A.p < A.e1) gather8_smem(A.c0, zs_addr, zero_slot, sr, si);  // skip all-pad chunks
      if (A.p + STRIDE < A.e1) gather8_smem(A.c1, zs_addr, zero_slot, sr, si);
      for (int p = A.p + 2 * STRIDE; p < A.e1; p += STRIDE)
        gather8_smem(ldg(colv + (p >> 3)), zs_addr, zero_slot, sr, si);
    } else {
      gather8_global(A.c0, zglob, sr, si);
      gather8_global(A.c1, zglob, sr, si);
      for (int p = A.p + 2 * STRIDE; p < A.e1; p += STRIDE)
        gather8_global(ldg(colv + (p >> 3)), zglob, sr, si);
    }
    sr += A.z.x;
    si += A.z.y;
    for (int p = A.x0 + LPR + t; p < A.x1; p += LPR) {
      const double2 z = ldz(z_in + (sxc ? sxc[p] : ldg(xcol + p)));
      sr += z.x;
      si += z.y;
    }
    // group reduction with a transposed first level: lanes of the low half
    // keep the real part, the high half the imaginary part, so every level
    // moves ONE double (2 SHFL) instead of two (fixed order, deterministic)
    const bool hi_half = (t & (LPR / 2)) != 0;
    double v = hi_half ? si : sr;
    v += __shfl_xor_sync(gmask, hi_half ? sr : si, LPR / 2);
#pragma unroll
    for (int o = LPR / 4; o > 0; o >>= 1) v += __shfl_xor_sync(gmask, v, o);
    if (t == 0 || t == LPR / 2) {  // t = 0 owns .x, t = LPR/2 owns .y
      double *dst = reinterpret_cast<double *>(sm.acc + r) + (t ? 1 : 0);
      if (!MULTI || pass == 0) {
        *dst = v;
      } else {
        *dst = *dst + v;
      }
    }
    A = B;
    B = C;
  }
}

// Separate inter phase (segments whose rows carry many inter entries, e.g.
// config 5's ~400 per row): 8 lanes per row, each lane keeps IU independent
// random z gathers in flight (the inline path keeps one), fixed per-lane
// order + 8-lane butterfly, added onto the row's intra sum.
template <int IU>
__device__ __forceinline__ void inter_phase(const StageArgs &a, const SegSmem &sm, int nrows,
                                            int64_t row0, int64_t row0a, int64_t xbase,
                                            const int32_t *__restrict__ xcol) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int t = lane & 7, grp = tid >> 3;
  const unsigned gmask = 0xFFu << (lane & 24);
  const double2 *__restrict__ z_in = a.z_in;
  for (int r = grp; r < nrows; r += NGROUPS) {
    const int64_t li = row0 + r - row0a;
    const int x0 = (int)(sm.sxp[li] - xbase), x1 = (int)(sm.sxp[li + 1] - xbase);
    double sr = 0.0, si = 0.0;
    for (int p = x0 + t; p < x1; p += 8 * IU) {
      int j[IU];
#pragma unroll
      for (int k = 0; k < IU; ++k) j[k] = (p + 8 * k < x1) ? ldg(xcol + p + 8 * k) : -1;
      double2 z[IU];
#pragma unroll
      for (int k = 0; k < IU; ++k) z[k] = (j[k] >= 0) ? ldz(z_in + j[k]) : make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < IU; ++k) {
        sr += z[k].x;
        si += z[k].y;
      }
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      sr += __shfl_xor_sync(gmask, sr, o);
      si += __shfl_xor_sync(gmask, si, o);
    }
    if (t == 0) {
      const double2 prev = sm.acc[r];
      sm.acc[r] = make_double2(prev.x + sr, prev.y + si);
    }
  }
}

// Block-phased inter sweep (g.inter_blocks > 0; config 5): before its
// segments, the CTA sums the inter entries of all its rows, column block by
// column block, into xacc (one 8-lane group per row, IU independent gathers
// per lane; block q adds onto block q-1's sum in a fixed order).  All CTAs
// walk the blocks at about the same pace, so the random z gathers of the
// whole GPU fall into one ~inter_block_nodes*16-byte slice of z that stays
// L2-resident instead of thrashing HBM.
template <int LPR, int IU, bool HINT = false>
__device__ __forceinline__ void inter_sweep(const StageArgs &a) {
  const cdk_graph &g = a.g;
  const int segA = g.cta_seg[blockIdx.x], segB = g.cta_seg[blockIdx.x + 1];
  if (segA == segB) return;
  const int64_t rA = g.rblk_row0[g.seg_rblk[segA]], rB = g.rblk_row0[g.seg_rblk[segB]];
  constexpr int NG = SWEEP_THREADS / LPR;
  const int tid = threadIdx.x, lane = tid & 31;
  const int t = lane & (LPR - 1), grp = tid / LPR;
  const unsigned gmask = (LPR == 32) ? FULL : (((1u << LPR) - 1u) << (lane & ~(LPR - 1)));
  const double2 *__restrict__ z_in = a.z_in;
  const int nb = g.inter_blocks;
  const uint64_t pol = l2_evict_first();
  for (int q = 0; q < nb; ++q) {
    for (int64_t i = rA + grp; i < rB; i += NG) {
      const int64_t xb = HINT ? ld_stream(g.inter_ptr + i, pol) : __ldg(g.inter_ptr + i);
      const int64_t xe = HINT ? ld_stream(g.inter_ptr + i + 1, pol) : __ldg(g.inter_ptr + i + 1);
      const uint64_t sw =
          nb > 1 ? (HINT ? ld_stream(g.inter_split + i, pol) : __ldg(g.inter_split + i)) : 0ull;
      const int64_t s0 = xb + (q ? (int64_t)((sw >> (16 * (q - 1))) & 0xFFFFu) : 0);
      const int64_t s1 = (q + 1 < nb) ? xb + (int64_t)((sw >> (16 * q)) & 0xFFFFu) : xe;
      double sr = 0.0, si = 0.0;
      for (int64_t p = s0 + t; p < s1; p += LPR * IU) {
        int j[IU];
#pragma unroll
        for (int k = 0; k < IU; ++k)
          j[k] = (p + LPR * k < s1)
                     ? (HINT ? ld_stream(g.inter_col + p + LPR * k, pol) : ldg(g.inter_col + p + LPR * k))
                     : -1;
        double2 z[IU];
#pragma unroll
        for (int k = 0; k < IU; ++k)
          z[k] = (j[k] >= 0) ? ldz(z_in + j[k]) : make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < IU; ++k) {
          sr += z[k].x;
          si += z[k].y;
        }
      }
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) {
        sr += __shfl_xor_sync(gmask, sr, o);
        si += __shfl_xor_sync(gmask, si, o);
      }
      if (t == 0) {
        if (q > 0) {
          const double2 prev = HINT ? ldcg_stream(a.xacc + i, pol) : ldcg2(a.xacc + i);
          sr = prev.x + sr;
          si = prev.y + si;
        }
        if (HINT) stcg_stream(a.xacc + i, make_double2(sr, si), pol);
        else __stcg(a.xacc + i, make_double2(sr, si));
      }
    }
  }
  __syncthreads();
}

// Software-pipelined variant: the next row's pointers, split word, first
// index batch and previous-block sum are loaded while the current row's
// gathers are in flight, so a group always has gathers or index loads
// outstanding instead of serialising pointer -> index -> gather per row.
template <int IU>
__device__ __forceinline__ void inter_sweep_pipe(const StageArgs &a) {
  constexpr int LPR = 8;
  const cdk_graph &g = a.g;
  const int segA = g.cta_seg[blockIdx.x], segB = g.cta_seg[blockIdx.x + 1];
  if (segA == segB) return;
  const int64_t rA = g.rblk_row0[g.seg_rblk[segA]], rB = g.rblk_row0[g.seg_rblk[segB]];
  const int tid = threadIdx.x, lane = tid & 31;
  const int t = lane & (LPR - 1), grp = tid / LPR;
  const unsigned gmask = 0xFFu << (lane & 24);
  const double2 *__restrict__ z_in = a.z_in;
  const int32_t *__restrict__ xc = g.inter_col;
  const int nb = g.inter_blocks;
  auto span = [&](int64_t i, int q, int64_t &s0, int64_t &s1) {
    const int64_t xb = __ldg(g.inter_ptr + i), xe = __ldg(g.inter_ptr + i + 1);
    const uint64_t sw = nb > 1 ? __ldg(g.inter_split + i) : 0ull;
    s0 = xb + (q ? (int64_t)((sw >> (16 * (q - 1))) & 0xFFFFu) : 0);
    s1 = (q + 1 < nb) ? xb + (int64_t)((sw >> (16 * q)) & 0xFFFFu) : xe;
  };
  for (int q = 0; q < nb; ++q) {
    int64_t i = rA + grp;
    if (i >= rB) continue;
    int64_t c0, c1;
    span(i, q, c0, c1);
    int jn[IU];
#pragma unroll
    for (int k = 0; k < IU; ++k) jn[k] = (c0 + t + LPR * k < c1) ? ldg(xc + c0 + t + LPR * k) : -1;
    while (i < rB) {
      const int64_t i2 = i + SWEEP_THREADS / LPR;
      int64_t n0 = 0, n1 = 0;
      if (i2 < rB) span(i2, q, n0, n1);  // next row's span: in flight with this row's gathers
      double2 prev = make_double2(0.0, 0.0);
      if (q > 0 && t == 0) prev = ldcg2(a.xacc + i);
      double sr = 0.0, si = 0.0;
      int j[IU];
#pragma unroll
      for (int k = 0; k < IU; ++k) j[k] = jn[k];
      for (int64_t p = c0 + t;;) {
        double2 z[IU];
#pragma unroll
        for (int k = 0; k < IU; ++k)
          z[k] = (j[k] >= 0) ? ldz(z_in + j[k]) : make_double2(0.0, 0.0);
        p += LPR * IU;
        const bool more = p < c1;
        if (more) {
#pragma unroll
          for (int k = 0; k < IU; ++k) j[k] = (p + LPR * k < c1) ? ldg(xc + p + LPR * k) : -1;
        }
#pragma unroll
        for (int k = 0; k < IU; ++k) {
          sr += z[k].x;
          si += z[k].y;
        }
        if (!more) break;
      }
      // next row's first index batch (its span has landed by now)
      if (i2 < rB) {
#pragma unroll
        for (int k = 0; k < IU; ++k) jn[k] = (n0 + t + LPR * k < n1) ? ldg(xc + n0 + t + LPR * k) : -1;
      }
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) {
        sr += __shfl_xor_sync(gmask, sr, o);
        si += __shfl_xor_sync(gmask, si, o);
      }
      if (t == 0) {
        if (q > 0) {
          sr = prev.x + sr;
          si = prev.y + si;
        }
        __stcg(a.xacc + i, make_double2(sr, si));
      }
      i = i2;
      c0 = n0;
      c1 = n1;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void inter_sweep_dispatch(const StageArgs &a) {
  switch (a.sweep_mode) {
    case 1: inter_sweep<8, 8>(a); break;
    case 2: inter_sweep<8, 16>(a); break;
    case 3: inter_sweep<4, 16>(a); break;
    case 4: inter_sweep<8, 4>(a); break;
    case 5: inter_sweep<2, 16>(a); break;
    case 6: inter_sweep<16, 8>(a); break;
    case 7: inter_sweep_pipe<8>(a); break;
    case 8: inter_sweep_pipe<4>(a); break;
    case 9: inter_sweep_pipe<12>(a); break;
    case 10: inter_sweep<8, 8, true>(a); break;
    case 11: inter_sweep<8, 16, true>(a); break;
    default: inter_sweep<4, 8>(a);  // measured best on config 5 (tools/sweep_modes.sh)
  }
}

struct ProfAcc {
  unsigned long long t_stage = 0, t_gather = 0, t_epi = 0, t_mark = 0;
};

// One stage over this CTA's segments (see the kernel comment above).
template <int MODE>
__device__ __forceinline__ void stage_body(const StageArgs &a, const SegSmem &sm,
                                           uint64_t &bar_seg, uint64_t &bar_epi, double2 *sR,
                                           uint32_t &parity, ProfAcc &pa) {
  const cdk_graph &g = a.g;
  const uint32_t zero_slot = (uint32_t)g.smem_nodes;  // zs[smem_nodes] == 0
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t = lane & 7;
  const int grp = tid >> 3;
  const int leader = lane & 24;
  const unsigned gmask = 0xFFu << leader;  // this 8-lane group only
  const int segA = g.cta_seg[blockIdx.x], segB = g.cta_seg[blockIdx.x + 1];
  const double2 *__restrict__ z_in = a.z_in;
  const int wn = g.smem_nodes;
  // mbarrier phases: bar_seg completes once per pass, bar_epi once per segment
  uint32_t pseg = (parity >> 1) & 1u, pepi = parity & 1u;
  const bool swept = g.inter_blocks > 0;  // inter sums precomputed (inter_sweep_kernel)
  const int segEnd = (a.debug_flags & 2) ? segA : segB;
#ifdef CDK_PROFILE
#define PROF_MARK(acc)                           \
  do {                                           \
    const unsigned long long _n = clock64();     \
    pa.acc += _n - pa.t_mark;                    \
    pa.t_mark = _n;                              \
  } while (0)
#else
#define PROF_MARK(acc) \
  do {                 \
  } while (0)
#endif
  for (int s = segA; s < segEnd; ++s) {
    const int rbA = g.seg_rblk[s], rbB = g.seg_rblk[s + 1];
    const int64_t row0 = g.rblk_row0[rbA];
    const int64_t row1 = g.rblk_row0[rbB];
    const int64_t row0a = row0 & ~(int64_t)1;
    const int64_t w0 = g.seg_win[2 * s], w1 = g.seg_win[2 * s + 1];
    const bool staged = w1 > w0;
    const int npass = staged ? (int)((w1 - w0 + wn - 1) / wn) : 1;  // window passes (<= 4)
    const int nrows = (int)(row1 - row0);
    const int cA = g.rblk_comm[rbA];
    const bool inter_inline0 = !swept && (g.seg_lpr[s] & CDK_SEG_INTER_PHASE) == 0;
    const bool inter_inline = inter_inline0 && !(a.debug_flags & 4);
    const bool inter_phased = !swept && !inter_inline0 && !(a.debug_flags & 4);

    // staged inter columns (xs): the segment's inter run, 4-entry aligned
    int64_t xs_beg = 0;
    bool xs_ok = false;
    if (g.xs_cap > 0 && g.seg_xr != nullptr && inter_inline) {
      xs_beg = g.seg_xr[2 * s] & ~(int64_t)3;
      xs_ok = g.seg_xr[2 * s + 1] - xs_beg <= (int64_t)g.xs_cap;
    }
    // ---- 1. stage window, pointer slices, epilogue inputs (async) ----------
    if (tid == 0) {
      fence_proxy_async_smem();  // earlier generic accesses before the async overwrite
      const uint32_t bw = staged ? (uint32_t)(min(w1 - w0, (int64_t)wn) * 16) : 0u;
      const uint32_t bp = (uint32_t)((((row1 + 2) & ~(int64_t)1) - row0a) * 8);
      const uint32_t br = (uint32_t)((((row1 + 1) & ~(int64_t)1) - row0a) * 8);
      const uint32_t bx =
          xs_ok ? (uint32_t)(((g.seg_xr[2 * s + 1] - xs_beg + 3) & ~(int64_t)3) * 4) : 0u;
      const int nr_in = (MODE == 0) ? 1 : ((MODE == 1 || MODE == 5) ? 2 : 3);
      mbar_expect_tx(&bar_seg, bw + 2 * bp + bx);
      if (bx) bulk_g2s(sm.sxc, g.inter_col + xs_beg, bx, &bar_seg);
      if (bw) bulk_g2s(sm.zs, z_in + w0, bw, &bar_seg);
      bulk_g2s(sm.sip, g.intra_ptr + row0a, bp, &bar_seg);
      bulk_g2s(sm.sxp, g.inter_ptr + row0a, bp, &bar_seg);
      // epilogue inputs on their own barrier: they land during the gathers
      mbar_expect_tx(&bar_epi, (uint32_t)nr_in * br);
      bulk_g2s(sm.som, a.omega + row0a, br, &bar_epi);
      if (MODE != 0) bulk_g2s(sm.sth, a.theta + row0a, br, &bar_epi);
      if (MODE >= 2 && MODE <= 4) bulk_g2s(sm.sks, a.ksum + row0a, br, &bar_epi);
    }
    // community observables R_c of the segment's communities, reduced (in the
    // canonical 8-lane order) from the previous stage's rblock partials while
    // the copies fly: all threads load the partials into the (still unused)
    // accumulator buffer at once, then one 8-lane group per community reduces.
    if (cA >= 0) {
      const int cB = g.rblk_comm[rbB - 1];
      const int cLast = cB >= 0 ? cB : (int)g.n_comm - 1;
      const int ncomm = cLast - cA + 1;
      const int pb0 = g.comm_rblk_off[cA], pb1 = g.comm_rblk_off[cLast + 1];
      const int np = pb1 - pb0;
      const bool fits = np <= (int)cap4_of(g.seg_rows_cap);
      if (fits) {
        for (int q = tid; q < np; q += NTHREADS) sm.acc[q] = ldcg2(a.part_in + pb0 + q);
        __syncthreads();
      }
      for (int q = grp; q < ncomm; q += NGROUPS) {
        const int c = cA + q;
        const int b0 = g.comm_rblk_off[c], b1 = g.comm_rblk_off[c + 1];
        double2 Rc;
        if (fits) {
          double sr = 0.0, si = 0.0;
          for (int b = b0 + t; b < b1; b += 8) {
            const double2 v = sm.acc[b - pb0];
            sr += v.x;
            si += v.y;
          }
#pragma unroll
          for (int o = 4; o > 0; o >>= 1) {
            sr += __shfl_xor_sync(gmask, sr, o);
            si += __shfl_xor_sync(gmask, si, o);
          }
          Rc = make_double2(sr, si);
        } else {
          Rc = reduce_comm8(a.part_in, b0, b1, t, gmask);
        }
        if (t == 0) sR[q] = Rc;
      }
      __syncthreads();  // accumulator buffer free for the gather phase
    }
    mbar_wait(&bar_seg, pseg);
    pseg ^= 1u;
    PROF_MARK(t_stage);
    const uint32_t zs_addr = smem_u32(sm.zs);
    const double2 *__restrict__ zglob = z_in + g.seg_base[s];
    const int64_t ebase = sm.sip[row0 - row0a], xbase = sm.sxp[row0 - row0a];
    const uint4 *__restrict__ colv = reinterpret_cast<const uint4 *>(g.intra_col + ebase);
    const int32_t *__restrict__ xcol = g.inter_col + xbase;
    const int lpr = g.seg_lpr[s] & 0xFF;
    // inter column p of the segment (relative to xbase) lives at sxc[p + xbase - xs_beg]
    const int32_t *sxc_rel = xs_ok ? sm.sxc + (xbase - xs_beg) : nullptr;

    // ---- 2. gather: lanes per row chosen per segment (4 / 8 / 16 / 32); a
    //         community wider than the window is gathered in passes, each
    //         with its slice of the window restaged (rebased columns of pass
    //         q lie in [q*wn, (q+1)*wn): the window base address is shifted)
    for (int pass = 0; pass < npass; ++pass) {
      if (pass > 0) {
        __syncthreads();  // every gather of the previous pass is done with zs
        if (tid == 0) {
          fence_proxy_async_smem();
          const int64_t q0 = w0 + (int64_t)pass * wn, q1 = min(w1, q0 + wn);
          const uint32_t bq = (uint32_t)((q1 - q0) * 16);
          mbar_expect_tx(&bar_seg, bq);
          bulk_g2s(sm.zs, z_in + q0, bq, &bar_seg);
        }
        mbar_wait(&bar_seg, pseg);
        pseg ^= 1u;
      }
      const uint32_t zs_p = zs_addr - (uint32_t)pass * (uint32_t)wn * 16u;
      const uint32_t zero_p = zero_slot + (uint32_t)pass * (uint32_t)wn;
#define CDK_GATHER(L, M, I)                                                                  \
  gather_phase<L, M, I>(a, sm, nrows, row0, row0a, ebase, xbase, staged, zs_p, zero_p, zglob, \
                        colv, xcol, pass, npass, sxc_rel)
      const bool multi = npass > 1;
      if (a.debug_flags & 8) {
        for (int r = tid; r < nrows; r += NTHREADS) sm.acc[r] = make_double2(0.0, 0.0);
      } else if (lpr == 4) {
        if (multi) {
          if (inter_inline) CDK_GATHER(4, true, true); else CDK_GATHER(4, true, false);
        } else {
          if (inter_inline) CDK_GATHER(4, false, true); else CDK_GATHER(4, false, false);
        }
      } else {
        if (multi) {
          if (inter_inline) CDK_GATHER(8, true, true); else CDK_GATHER(8, true, false);
        } else {
          if (inter_inline) CDK_GATHER(8, false, true); else CDK_GATHER(8, false, false);
        }
      }
#undef CDK_GATHER
    }
    __syncthreads();
    if (inter_phased) {
      inter_phase<8>(a, sm, nrows, row0, row0a, xbase, xcol);
      __syncthreads();
    }
    PROF_MARK(t_gather);

    // ---- 3. epilogue: warp per rblock, lane = row ---------------------------
    mbar_wait(&bar_epi, pepi);
    pepi ^= 1u;
    const double kn = a.k_over_n;
    for (int rb = rbA + warp; rb < rbB; rb += NWARPS) {
      const int64_t rrow0 = g.rblk_row0[rb];
      const int64_t rrow1 = g.rblk_row0[rb + 1];
      const int nr = (int)(rrow1 - rrow0);
      const int c = g.rblk_comm[rb];
      double zr = 0.0, zim = 0.0;
      if (lane < nr) {
        const int64_t i = rrow0 + lane;
        const int64_t li = i - row0a;
        double2 ac = sm.acc[i - row0];
        if (swept) {
          const double2 xa = ldcg2(a.xacc + i);
          ac = make_double2(ac.x + xa.x, ac.y + xa.y);
        }
        const double2 zi = (staged && npass == 1) ? sm.zs[i - w0] : ldz(z_in + i);
        const double2 R = (c >= 0) ? sR[c - cA] : make_double2(0.0, 0.0);
        double k = sm.som[li] + kn * (R.y * zi.x - R.x * zi.y);
        k = k + kn * (ac.y * zi.x - ac.x * zi.y);
        if (MODE == 0) {
          a.out[i] = k;
        } else {
          const double th0 = sm.sth[li];
          double thn;
          if (MODE == 1) {
            a.ksum[i] = k;
            thn = add_rn(th0, mul_rn(a.h, k));
          } else if (MODE == 2 || MODE == 3) {
            a.ksum[i] = add_rn(sm.sks[li], mul_rn(2.0, k));
            thn = add_rn(th0, mul_rn(a.h, k));
          } else {  // MODE 4: x + dt/6 (k1 + 2k2 + 2k3 + k4); MODE 5: Euler x + dt k
            const double ks = (MODE == 4) ? add_rn(sm.sks[li], k) : k;
            thn = wrap_phase(add_rn(th0, mul_rn(a.h, ks)));
            a.theta[i] = thn;
            if (!isfinite(thn)) {
              atomicAdd(reinterpret_cast<unsigned long long *>(&a.status->nonfinite), 1ull);
              atomicMin(reinterpret_cast<long long *>(&a.status->first_bad_step),
                        (long long)(a.status->steps_done + a.step_rel + 1));
            }
          }
          sincos(thn, &zim, &zr);
          const double2 zn = make_double2(zr, zim);
          a.z_out[i] = zn;
          for (int q = 0; q < a.n_peers; ++q)  // NVLink P2P stores (fused all-gather)
            if (q != a.rank) a.peer_out[q][i] = zn;
        }
      }
      if (MODE != 0) {
        // canonical rblock partial: lane t < 8 sums rows t, t+8, t+16, t+24 in
        // order (absent rows = +0), then the 8-lane xor butterfly
        const double r8 = __shfl_down_sync(FULL, zr, 8), i8 = __shfl_down_sync(FULL, zim, 8);
        const double r16 = __shfl_down_sync(FULL, zr, 16), i16 = __shfl_down_sync(FULL, zim, 16);
        const double r24 = __shfl_down_sync(FULL, zr, 24), i24 = __shfl_down_sync(FULL, zim, 24);
        double pr = ((zr + r8) + r16) + r24, pim = ((zim + i8) + i16) + i24;
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
          pr += __shfl_xor_sync(FULL, pr, o);
          pim += __shfl_xor_sync(FULL, pim, o);
        }
        if (lane == 0) a.part_out[rb] = make_double2(pr, pim);
      }
    }
    __syncthreads();  // shared segment buffers reused by the next segment
    PROF_MARK(t_epi);
  }
  if (a.n_peers > 1) __threadfence_system();  // peer stores before the barrier signal
  parity = (pseg << 1) | pepi;
}

__device__ __forceinline__ void init_cta(const cdk_graph &g, const SegSmem &sm, uint64_t &bar_seg,
                                         uint64_t &bar_epi) {
  if (threadIdx.x == 0) {
    mbar_init(&bar_seg, 1);
    mbar_init(&bar_epi, 1);
    sm.zs[g.smem_nodes] = make_double2(0.0, 0.0);
  }
  __syncthreads();
}

// Block-phased inter sweep as its own launch: it must run with (almost) no
// shared memory — measured on B200, a 200+ KB shared-memory carve-out halves
// the random-gather rate (124 vs 240 Ggathers/s, tools/sweep_bench.cu), the
// L1 left for in-flight misses being too small.  Same CTA row ranges as the
// stage kernel (cta_seg).
__global__ void __launch_bounds__(SWEEP_THREADS, 1) inter_sweep_kernel(const StageArgs a) {
  inter_sweep_dispatch(a);
}

// single stage launch (MODE 0: RHS, 1..4: RK4 stage, 5: Euler)
template <int MODE>
__global__ void __launch_bounds__(NTHREADS, CDK_STAGE_MINBLOCKS) kuramoto_stage_kernel(const StageArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bar_seg, bar_epi;
  __shared__ double2 sR[SEG_MAX_COMM];
  if (a.n_peers > 1 && run_aborted(a.status)) return;  // a peer barrier timed out earlier
  const SegSmem sm = carve_smem(smem_raw, a.g.seg_rows_cap, a.g.smem_nodes);
  init_cta(a.g, sm, bar_seg, bar_epi);
  uint32_t parity = 0;
  ProfAcc pa;
#ifdef CDK_PROFILE
  pa.t_mark = clock64();
  const unsigned long long t_begin = pa.t_mark;
  unsigned long long g_begin;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_begin));
#endif
  stage_body<MODE>(a, sm, bar_seg, bar_epi, sR, parity, pa);
#ifdef CDK_PROFILE
  if (threadIdx.x == 0 && a.prof) {
    unsigned long long *p = a.prof + 6 * blockIdx.x;
    p[0] = clock64() - t_begin;
    p[1] = pa.t_stage;
    p[2] = pa.t_gather;
    p[3] = pa.t_epi;
    unsigned long long g_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
    p[4] = g_begin;  // ns: launch skew and tail across CTAs
    p[5] = g_end;
  }
#endif
}

#ifndef CDK_GRID_SLEEP_NS
#define CDK_GRID_SLEEP_NS 0  // grid-barrier poll back-off (64 ns: release ~0.2 us later)
#endif
// grid-wide barrier for the cooperative (co-resident) persistent kernel:
// monotone arrival counter, target = (sync index + 1) * gridDim.x.  The test
// is wrap-safe (serial-number arithmetic), so a launch may run more than
// 2^32 / gridDim.x barriers.
__device__ __forceinline__ void grid_sync(unsigned int *counter, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(counter, 1u);
    unsigned int v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
      if ((int)(v - target) >= 0) break;
      __nanosleep(CDK_GRID_SLEEP_NS);
    }
    __threadfence();
  }
  __syncthreads();
}

// System-scope counter barrier of the fused exchange: signal every rank
// (its counter gets +1 from each rank per stage), then wait until this
// rank's counter reaches `target`.  A 20 s watchdog turns a lost peer into
// an ABORT: status.reserved bit 0 is set, the persistent kernels return at
// their next grid barrier, later stage launches return at entry and later
// peer barriers do not wait — one timeout ends the run (the host raises).
struct PeerBar {
  unsigned int *const *bar;
  unsigned int *mine;
  int n, wait;
};

__device__ __forceinline__ void peer_barrier(const PeerBar &pb, unsigned int target,
                                             cdk_run_status *st) {
  if (run_aborted(st)) return;
  __threadfence_system();
  for (int q = 0; q < pb.n; ++q) atomicAdd_system(pb.bar[q], 1u);
  if (!pb.wait) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned int v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(pb.mine) : "memory");
    if ((int)(v - target) >= 0) break;
    uint64_t t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (t1 - t0 > 20000000000ull) {
      atomicOr(reinterpret_cast<unsigned long long *>(&st->reserved), 1ull);
      break;
    }
    __nanosleep(100);
  }
  __threadfence_system();
}

__global__ void peer_barrier_kernel(PeerBar pb, unsigned int target, cdk_run_status *st) {
  peer_barrier(pb, target, st);
}

struct StepPtrs {
  double2 *z[2];
  double2 *part[2];
  unsigned int *bar;
  double2 *const *peer_z[2];  // fused exchange: every rank's z[0] / z[1] (n_peers > 1)
  PeerBar pb;
  unsigned int pb_base;
};

// Persistent RK4: n_steps x 4 stages in ONE cooperative launch, grid barrier
// between stages (no launch gaps; the CSR slices and window reloads are the
// only per-stage traffic).
template <bool PEERS>
__global__ void __launch_bounds__(NTHREADS, CDK_STAGE_MINBLOCKS) kuramoto_rk4_kernel(StageArgs a, StepPtrs ptr,
                                                                   int64_t n_steps, double dt) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bar_seg, bar_epi;
  __shared__ double2 sR[SEG_MAX_COMM];
  const SegSmem sm = carve_smem(smem_raw, a.g.seg_rows_cap, a.g.smem_nodes);
  init_cta(a.g, sm, bar_seg, bar_epi);
  uint32_t parity = 0;
  ProfAcc pa;
  unsigned int sync_idx = 0;
  const double h2 = dt / 2.0, h6 = dt / 6.0;
  unsigned int peer_target = ptr.pb_base;
  // after a stage: grid barrier, and with peers the cross-GPU barrier (one
  // thread) followed by a second grid barrier that releases every CTA
#define CDK_STAGE_SYNC(last)                                                           \
  do {                                                                                 \
    if (PEERS) {                                                                       \
      grid_sync(ptr.bar, ++sync_idx * gridDim.x);                                      \
      peer_target += (unsigned int)a.n_peers;                                          \
      if (blockIdx.x == 0 && threadIdx.x == 0) peer_barrier(ptr.pb, peer_target, a.status); \
      if (!(last)) grid_sync(ptr.bar, ++sync_idx * gridDim.x);                         \
      if (run_aborted(a.status)) return;                                               \
    } else if (!(last)) {                                                              \
      grid_sync(ptr.bar, ++sync_idx * gridDim.x);                                      \
    }                                                                                  \
  } while (0)
  for (int64_t step = 0; step < n_steps; ++step) {
    a.step_rel = step;
    a.z_in = ptr.z[0]; a.z_out = ptr.z[1]; a.part_in = ptr.part[0]; a.part_out = ptr.part[1];
    a.peer_out = ptr.peer_z[1];
    a.h = h2;
    stage_body<1>(a, sm, bar_seg, bar_epi, sR, parity, pa);
    CDK_STAGE_SYNC(false);
    a.z_in = ptr.z[1]; a.z_out = ptr.z[0]; a.part_in = ptr.part[1]; a.part_out = ptr.part[0];
    a.peer_out = ptr.peer_z[0];
    stage_body<2>(a, sm, bar_seg, bar_epi, sR, parity, pa);
    CDK_STAGE_SYNC(false);
    a.z_in = ptr.z[0]; a.z_out = ptr.z[1]; a.part_in = ptr.part[0]; a.part_out = ptr.part[1];
    a.peer_out = ptr.peer_z[1];
    a.h = dt;
    stage_body<3>(a, sm, bar_seg, bar_epi, sR, parity, pa);
    CDK_STAGE_SYNC(false);
    a.z_in = ptr.z[1]; a.z_out = ptr.z[0]; a.part_in = ptr.part[1]; a.part_out = ptr.part[0];
    a.peer_out = ptr.peer_z[0];
    a.h = h6;
    stage_body<4>(a, sm, bar_seg, bar_epi, sR, parity, pa);
    CDK_STAGE_SYNC(step + 1 == n_steps);
  }
#undef CDK_STAGE_SYNC
}

// ===========================================================================
// ELL stage kernels (cdk_graph.ell_off set; layout: cdk_host_ell_intra).
// One warp per rblock, lane = row, persistent CTAs over the same segments as
// the kernels above.  Per segment: one bulk copy (TMA engine) stages the
// window of z_in, the segment's chunk and inter-column ranges are prefetched
// into L2, and each 8-lane group reduces one community's R_c from the
// previous stage's rblock partials.  Warps then claim rblocks (shared
// counter); per rblock every lane streams its row's 16-byte chunks (8 uint16
// columns, 512 contiguous bytes per warp per chunk, two chunks in flight) and
// gathers z from the window — the layout schedules each quarter-warp step
// onto 8 distinct bank groups, padding included (zero slots per bank group),
// so every LDS.128 is 4 wavefronts — sums its inter columns (global z, the
// first four issued before the intra loop), and runs the same epilogue as
// above (same arithmetic, lane = row).  No row reductions, no per-row
// pointers, no barrier between gathers and epilogue.  Accumulation order is
// fixed by the layout: deterministic and independent of the CTA schedule.
// ===========================================================================
#ifndef CDK_ELL_THREADS
#define CDK_ELL_THREADS 512  // measured (config 2, 8192-node window): 512 > 640 > 448 > 384 > 768
#endif
#ifndef CDK_ELL_WINDOW
#define CDK_ELL_WINDOW 8192  // nodes: (8192 + 8) * 16 B = 128 KB; the rest of the SM stays L1
                             // (measured: 14336 nodes, 224 KB, is 3% slower on config 2)
#endif
#ifndef CDK_ELL_DEPTH
#define CDK_ELL_DEPTH 4  // chunks per lane in flight (cp.async ring in shared memory; measured 4 > 8 on config 2)
#endif
#ifndef CDK_ELL_XCOLS
#define CDK_ELL_XCOLS 12  // inter columns per lane loaded before the intra loop (multiple of 4)
#endif
#ifndef CDK_ELL_RK4_RT
#define CDK_ELL_RK4_RT 1  // persistent RK4: one stage body with a runtime mode (0: four inlined)
#endif
constexpr int ELL_THREADS = CDK_ELL_THREADS;
constexpr int ELL_XCOLS = CDK_ELL_XCOLS;
#ifndef CDK_ELL_XEARLY
#define CDK_ELL_XEARLY 4  // inter z gathers issued before the intra loop (4 <= . <= XCOLS)
#endif
constexpr int ELL_XEARLY = CDK_ELL_XEARLY;
#ifndef CDK_ELL_MINBLOCKS
#define CDK_ELL_MINBLOCKS 1  // resident ELL CTAs per SM (the planner launches SMs x this many)
#endif
constexpr int ELL_PART_CAP = 512 / CDK_ELL_MINBLOCKS;  // a segment's rblock partials in smem
#ifndef CDK_ELL_META_CAP
#define CDK_ELL_META_CAP 256  // unit records of a staged segment held in shared memory
#endif
constexpr int ELL_META_CAP = CDK_ELL_META_CAP;
constexpr int ELL_DEPTH = CDK_ELL_DEPTH;
constexpr int ELL_WARPS = ELL_THREADS / 32;
constexpr int ELL_GROUPS = ELL_THREADS / 8;

static_assert((CDK_ELL_DEPTH & (CDK_ELL_DEPTH - 1)) == 0, "CDK_ELL_DEPTH: a power of two");
// dynamic shared memory: the z window (+ one zero slot per bank group), then
// each warp's chunk ring (ELL_DEPTH x 512 bytes: one 16-byte chunk per lane)
__host__ __device__ inline size_t ell_ring_offset(int smem_nodes) {
  return ((size_t)smem_nodes + 8) * 16;  // smem_nodes is a multiple of 8: 128-byte aligned
}
__host__ __device__ inline size_t ell_smem_bytes(int smem_nodes) {
  return ell_ring_offset(smem_nodes) + (size_t)ELL_WARPS * ELL_DEPTH * 512;
}

// cp.async (16 bytes, L2 only): the chunk stream lands in shared memory
// without occupying registers while in flight
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint4 lds_u4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}

__device__ __forceinline__ void prefetch_l2(const void *p, uint64_t bytes) {
  // cp.async.bulk.prefetch.L2: 16-byte granules, issued in <= 64 KB pieces
  uint64_t a = reinterpret_cast<uint64_t>(p) & ~(uint64_t)15;
  const uint64_t end = reinterpret_cast<uint64_t>(p) + bytes;
  while (a < end) {
    const uint64_t left = (end - a + 15) & ~(uint64_t)15;
    const uint32_t n = (uint32_t)(left < 65536 ? left : 65536);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(n) : "memory");
    a += n;
  }
}

// 8 entries of one chunk from the window: unconditional (pads hit zero slots);
// all 8 loads in flight, then their adds
__device__ __forceinline__ void ell_gather8_smem(const uint4 w, uint32_t zs_addr, double &ar,
                                                 double &ai, double &br, double &bi) {
  const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
  double2 z[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t u = (wv[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu;
    z[k] = lds_d2(zs_addr + (u << 4));
  }
#pragma unroll
  for (int k = 0; k < 8; k += 2) {
    ar += z[k].x;
    ai += z[k].y;
    br += z[k + 1].x;
    bi += z[k + 1].y;
  }
}

// unstaged rblocks (community wider than the window): global gathers, pads skipped
__device__ __forceinline__ void ell_gather8_global(const uint4 w, const double2 *__restrict__ zb,
                                                   double &ar, double &ai, double &br,
                                                   double &bi) {
  const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t u = (wv[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu;
    if (u != CDK_INTRA_PAD) {
      const double2 z = ldz(zb + u);
      if (k & 1) {
        br += z.x;
        bi += z.y;
      } else {
        ar += z.x;
        ai += z.y;
      }
    }
  }
}

// per-stage values (the kernel parameter StageArgs stays untouched, so the
// persistent kernel reads the graph from the parameter bank, not a local copy)
struct StageVar {
  const double2 *z_in;
  double2 *z_out;
  const double2 *part_in;
  double2 *part_out;
  double2 *const *peer_out;
  double h;
  int64_t step_rel;
  __device__ static StageVar of(const StageArgs &a) {
    return StageVar{a.z_in, a.z_out, a.part_in, a.part_out, a.peer_out, a.h, a.step_rel};
  }
};

// chunk stream of work unit u (this lane's column): first chunk, chunk count
struct UnitChunks {
  const uint4 *cp;
  int nch;
};
__device__ __forceinline__ UnitChunks unit_chunks(const cdk_graph &g, int u, int lane) {
  if (g.ell_meta) {  // packed unit metadata: one round trip
    const int4 m0 = ldg(reinterpret_cast<const int4 *>(g.ell_meta) + 2 * u);
    const int4 m1 = ldg(reinterpret_cast<const int4 *>(g.ell_meta) + 2 * u + 1);
    UnitChunks r;
    r.cp = reinterpret_cast<const uint4 *>(g.ell_col) + (uint32_t)m0.x + lane;
    r.nch = m1.x;
    return r;
  }
  const int rb = g.ell_units[u];
  UnitChunks r;
  r.cp = reinterpret_cast<const uint4 *>(g.ell_col) + g.ell_off[rb] + lane;
  r.nch = (int)((g.ell_off[rb + 1] - g.ell_off[rb]) >> 5);
  return r;
}

// One work unit (an rblock): lane = row.  The
// unit's chunk stream runs through the warp's ring in shared memory
// (cp.async, ELL_DEPTH chunks in flight per lane, one commit group per
// chunk): no registers held by loads in flight, no register moves between
// queue slots (a move of a register whose load is pending stalls the warp on
// that load), and the depth is free of register pressure.
template <bool STAGED>
__device__ __forceinline__ void ell_rblock(const int MODE, const StageArgs &a, const StageVar &v,
                                           int rb, uint32_t zs_addr, const double2 *zs, int64_t w0,
                                           const double2 *__restrict__ zglob, double2 R,
                                           const UnitChunks &uc, uint32_t ring,
                                           const int4 *mt = nullptr) {
  const cdk_graph &g = a.g;
  const int lane = threadIdx.x & 31;
  int64_t r0, r1, x0;
  int nx;
  if (mt) {  // packed unit metadata (cdk_graph.ell_meta)
    r0 = (uint32_t)mt->z;
    r1 = r0 + (mt[1].z & 0xFF);
    x0 = (uint32_t)mt->y;
    nx = mt[1].y;
  } else {
    r0 = g.rblk_row0[rb];
    r1 = g.rblk_row0[rb + 1];
    x0 = g.xell_off[rb];
    nx = (int)((g.xell_off[rb + 1] - x0) >> 5);
  }
  const int64_t i = r0 + lane;
  const bool valid = i < r1;
  DBG_CHECK(r1 <= g.n_rows && r1 - r0 <= 32, "rblock %d: rows [%lld, %lld) vs n_rows %lld", rb,
            (long long)r0, (long long)r1, (long long)g.n_rows);
  const int nch = uc.nch;
  // epilogue inputs: in flight during the gathers
  double om = 0.0, th0 = 0.0, ks0 = 0.0;
  if (valid) {
    om = a.omega[i];
    if (MODE != 0) th0 = a.theta[i];
    if (MODE >= 2 && MODE <= 4) ks0 = a.ksum[i];
  }
  // inter entries: the first ELL_XCOLS columns load before the intra loop and
  // the z of the first four go out with them; after the loop the z of the
  // remaining columns go out together (one exposed L2 round trip, not one
  // column + one z round trip per batch of four)
  const int32_t *__restrict__ xc = g.xell_col + x0 + lane;
  const double2 *__restrict__ z_in = v.z_in;
  int jx[ELL_XCOLS];
#pragma unroll
  for (int q = 0; q < ELL_XCOLS; ++q) jx[q] = (q < nx) ? ldg(xc + 32 * q) : -1;
#ifdef CDK_DEBUG
  for (int q = 0; q < ELL_XCOLS; ++q)
    DBG_CHECK(jx[q] < g.n_rows, "rblock %d: inter column %d >= n_rows %lld", rb, jx[q],
              (long long)g.n_rows);
#endif
  double2 xz[ELL_XEARLY];
#pragma unroll
  for (int q = 0; q < ELL_XEARLY; ++q)
    xz[q] = (jx[q] >= 0) ? ldz(z_in + jx[q]) : make_double2(0.0, 0.0);
  // intra chunks: ELL_DEPTH in flight ahead of the one being gathered
  const uint4 *__restrict__ cp = uc.cp;
#pragma unroll
  for (int d = 0; d < ELL_DEPTH; ++d) {
    if (d < nch) cp_async16(ring + d * 512, cp + 32 * d);
    cp_async_commit();
  }
  double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
  double2 xw[ELL_XCOLS > 4 ? ELL_XCOLS - 4 : 1];
  auto issue_xw = [&]() {
#pragma unroll
    for (int q = 4; q < ELL_XCOLS; ++q)
      xw[q - 4] = (jx[q] >= 0) ? ldz(z_in + jx[q]) : make_double2(0.0, 0.0);
  };
  for (int c = 0; c < nch; ++c) {
    cp_async_wait<ELL_DEPTH - 1>();  // chunk c has landed (groups complete in order)
    const uint32_t slot = ring + (uint32_t)(c & (ELL_DEPTH - 1)) * 512u;
    const uint4 w = lds_u4(slot);
#ifdef CDK_DEBUG
    if (STAGED) {  // every window index lands in the window or its 8 zero slots
      const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
      for (int k = 0; k < 8; ++k) {
        const uint32_t u = (wv[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu;
        DBG_CHECK(u < (uint32_t)g.smem_nodes + 8u, "rblock %d chunk %d: window index %u >= %d + 8",
                  rb, c, u, g.smem_nodes);
      }
    }
#endif
    if (STAGED) {
      ell_gather8_smem(w, zs_addr, ar, ai, br, bi);
    } else {
      ell_gather8_global(w, zglob, ar, ai, br, bi);
    }
    // refill after the gathers issued: their addresses came from w, so the
    // slot has been read before the async copy overwrites it
    if (c + ELL_DEPTH < nch) cp_async16(slot, cp + 32 * (c + ELL_DEPTH));
    cp_async_commit();
  }
  double sr = -(ar + br), si = -(ai + bi);  // intra-missing entries: sign -1
#pragma unroll
  for (int q = 0; q < ELL_XEARLY; ++q) {
    sr += xz[q].x;
    si += xz[q].y;
  }
  if (ELL_XCOLS > ELL_XEARLY && nx > ELL_XEARLY) {
    if (ELL_XEARLY == 4) {
      issue_xw();
#pragma unroll
      for (int q = 4; q < ELL_XCOLS; ++q) {
        sr += xw[q - 4].x;
        si += xw[q - 4].y;
      }
    } else {
      double2 xl[ELL_XCOLS > ELL_XEARLY ? ELL_XCOLS - ELL_XEARLY : 1];
#pragma unroll
      for (int q = ELL_XEARLY; q < ELL_XCOLS; ++q)
        xl[q - ELL_XEARLY] = (jx[q] >= 0) ? ldz(z_in + jx[q]) : make_double2(0.0, 0.0);
#pragma unroll
      for (int q = ELL_XEARLY; q < ELL_XCOLS; ++q) {
        sr += xl[q - ELL_XEARLY].x;
        si += xl[q - ELL_XEARLY].y;
      }
    }
  }
  for (int k = ELL_XCOLS; k < nx; k += 4) {
#pragma unroll
    for (int q = 0; q < 4; ++q) jx[q] = (k + q < nx) ? ldg(xc + 32 * (k + q)) : -1;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      xz[q] = (jx[q] >= 0) ? ldz(z_in + jx[q]) : make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      sr += xz[q].x;
      si += xz[q].y;
    }
  }
  // epilogue (same arithmetic as stage_body's)
  double zr = 0.0, zim = 0.0;
  if (valid) {
    const double2 zi = STAGED ? zs[i - w0] : ldz(z_in + i);
    const double kn = a.k_over_n;
    double k = om + kn * (R.y * zi.x - R.x * zi.y);
    k = k + kn * (si * zi.x - sr * zi.y);
    if (MODE == 0) {
      a.out[i] = k;
    } else {
      double thn;
      if (MODE == 1) {
        a.ksum[i] = k;
        thn = add_rn(th0, mul_rn(v.h, k));
      } else if (MODE == 2 || MODE == 3) {
        a.ksum[i] = add_rn(ks0, mul_rn(2.0, k));
        thn = add_rn(th0, mul_rn(v.h, k));
      } else {
        const double ks = (MODE == 4) ? add_rn(ks0, k) : k;
        thn = wrap_phase(add_rn(th0, mul_rn(v.h, ks)));
        a.theta[i] = thn;
        if (!isfinite(thn)) {
          atomicAdd(reinterpret_cast<unsigned long long *>(&a.status->nonfinite), 1ull);
          atomicMin(reinterpret_cast<long long *>(&a.status->first_bad_step),
                    (long long)(a.status->steps_done + v.step_rel + 1));
        }
      }
      sincos(thn, &zim, &zr);
      const double2 zn = make_double2(zr, zim);
      v.z_out[i] = zn;
      for (int q = 0; q < a.n_peers; ++q)  // NVLink P2P stores (fused all-gather)
        if (q != a.rank) v.peer_out[q][i] = zn;
    }
  }
  if (MODE != 0) {  // canonical rblock partial (same shape as stage_body's)
    const double r8 = __shfl_down_sync(FULL, zr, 8), i8 = __shfl_down_sync(FULL, zim, 8);
    const double r16 = __shfl_down_sync(FULL, zr, 16), i16 = __shfl_down_sync(FULL, zim, 16);
    const double r24 = __shfl_down_sync(FULL, zr, 24), i24 = __shfl_down_sync(FULL, zim, 24);
    double pr = ((zr + r8) + r16) + r24, pim = ((zim + i8) + i16) + i24;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      pr += __shfl_xor_sync(FULL, pr, o);
      pim += __shfl_xor_sync(FULL, pim, o);
    }
    if (lane == 0) v.part_out[rb] = make_double2(pr, pim);
  }
}

struct EllSmem {
  double2 *zs;  // [smem_nodes + 8]: window, then one zero slot per bank group
  uint64_t *bar;
  double2 *sR;  // [SEG_MAX_COMM]
  int *next;    // rblock claim counter
  double2 *sP;  // [ELL_PART_CAP] the segment's rblock partials (community sums)
  int4 *meta;   // [2 * ELL_META_CAP] the segment's unit records (cdk_graph.ell_meta)
  uint32_t ring;  // this lane's slot 0 of its warp's chunk ring (shared address)
};

// MODE: 0 RHS, 1..4 RK4 stage, 5 Euler (a runtime value: constant-folded in
// the per-stage kernels, one uniform branch per row in the persistent one)
#ifdef CDK_PROFILE
// intra-CTA drain of one segment: each warp's finish time after the segment
// became ready; prof[14 n_cta + 4 cta + {0: sum over warps of (last finish -
// own finish), 1: (last finish - ready) x warps, 2: segments}] (ns)
__device__ void ell_prof_drain(const StageArgs &a, unsigned long long t_ready) {
  __shared__ unsigned long long fin[ELL_WARPS];
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if ((threadIdx.x & 31) == 0) fin[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0 && a.prof) {
    unsigned long long mx = 0, sum = 0;
    for (int w = 0; w < ELL_WARPS; ++w) mx = fin[w] > mx ? fin[w] : mx;
    for (int w = 0; w < ELL_WARPS; ++w) sum += mx - fin[w];
    unsigned long long *p = a.prof + 14 * gridDim.x + 4 * blockIdx.x;
    atomicAdd(p, sum);
    atomicAdd(p + 1, (mx - t_ready) * ELL_WARPS);
    atomicAdd(p + 2, 1ull);
  }
}
#endif

__device__ __forceinline__ void ell_body(const int MODE, const StageArgs &a, const StageVar &v,
                                         const EllSmem &sm, uint32_t &phase) {
  const cdk_graph &g = a.g;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t = lane & 7, grp = tid >> 3;
  const unsigned gmask = 0xFFu << (lane & 24);
  const int segA = g.cta_seg[blockIdx.x], segB = g.cta_seg[blockIdx.x + 1];
  const uint32_t zs_addr = smem_u32(sm.zs);
  for (int s = segA; s < segB; ++s) {
    const int rbA = g.seg_rblk[s], rbB = g.seg_rblk[s + 1];
    const int64_t w0 = g.seg_win[2 * s], w1 = g.seg_win[2 * s + 1];
    const bool staged = w1 > w0;
    const int cA = g.rblk_comm[rbA];
    if (tid == 0) {
      fence_proxy_async_smem();  // earlier generic accesses before the async overwrite
      if (staged) {
        const uint32_t bw = (uint32_t)((w1 - w0) * 16);
        // the segment's unit records ride along with the window (read from
        // shared memory at each claim instead of L2)
        const int nu = g.seg_unit[s + 1] - g.seg_unit[s];
        const uint32_t bm = (g.ell_meta && nu <= ELL_META_CAP) ? (uint32_t)nu * 32u : 0u;
        mbar_expect_tx(sm.bar, bw + bm);
        bulk_g2s(sm.zs, v.z_in + w0, bw, sm.bar);
        if (bm) bulk_g2s(sm.meta, g.ell_meta + 8 * (int64_t)g.seg_unit[s], bm, sm.bar);
      }
      const int64_t eA = g.ell_off[rbA], eB = g.ell_off[rbB];
      prefetch_l2(g.ell_col + 8 * eA, (uint64_t)(eB - eA) * 16);
      const int64_t xA = g.xell_off[rbA], xB = g.xell_off[rbB];
      prefetch_l2(g.xell_col + xA, (uint64_t)(xB - xA) * 4);
      *sm.next = g.seg_unit[s] + ELL_WARPS;
    }
    if (cA >= 0) {  // community observables of the segment (canonical order)
      const int cB = g.rblk_comm[rbB - 1];
      const int cLast = cB >= 0 ? cB : (int)g.n_comm - 1;
      const int pb0 = g.comm_rblk_off[cA], np = g.comm_rblk_off[cLast + 1] - pb0;
      if (np <= ELL_PART_CAP) {  // all partials in one round trip, then the 8-lane sums
        for (int q = tid; q < np; q += ELL_THREADS) sm.sP[q] = ldcg2(v.part_in + pb0 + q);
        __syncthreads();
      }
      for (int q = grp; q < cLast - cA + 1; q += ELL_GROUPS) {
        const int c = cA + q;
        const int b0 = g.comm_rblk_off[c], b1 = g.comm_rblk_off[c + 1];
        double2 Rc;
        if (np <= ELL_PART_CAP) {  // same order as reduce_comm8
          double sr = 0.0, si = 0.0;
          for (int b = b0 + t; b < b1; b += 8) {
            const double2 pv = sm.sP[b - pb0];
            sr += pv.x;
            si += pv.y;
          }
#pragma unroll
          for (int o = 4; o > 0; o >>= 1) {
            sr += __shfl_xor_sync(gmask, sr, o);
            si += __shfl_xor_sync(gmask, si, o);
          }
          Rc = make_double2(sr, si);
        } else {
          Rc = reduce_comm8(v.part_in, b0, b1, t, gmask);
        }
        if (t == 0) sm.sR[q] = Rc;
      }
    }
    __syncthreads();
    if (staged) {
      mbar_wait(sm.bar, phase);
      phase ^= 1u;
    }
#ifdef CDK_PROFILE
    if (tid == 0 && a.prof && s == segA) a.prof[6 * blockIdx.x + 1] = clock64();  // ready (raw)
    unsigned long long t_ready;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_ready));
#endif
    const double2 *zglob = v.z_in + g.seg_base[s];
    const int uB = g.seg_unit[s + 1];
    int u = g.seg_unit[s] + warp;
    if (g.ell_meta) {  // packed metadata: the unit's description travels in registers
      const bool mloc = staged && uB - g.seg_unit[s] <= ELL_META_CAP;  // records in smem
      const int4 *meta = mloc ? sm.meta - 2 * g.seg_unit[s]
                              : reinterpret_cast<const int4 *>(g.ell_meta);
      int4 ma = make_int4(0, 0, 0, 0), mb = ma;
      if (u < uB) {
        ma = meta[2 * u];
        mb = meta[2 * u + 1];
      }
      while (u < uB) {
        const int ci = mb.w & 0xFF;  // community relative to the segment's first (255: pool)
        const double2 R = (ci != 0xFF) ? sm.sR[ci] : make_double2(0.0, 0.0);
        const UnitChunks uc{reinterpret_cast<const uint4 *>(g.ell_col) + (uint32_t)ma.x + lane,
                            mb.x};
        const int4 mt[2] = {ma, mb};
        if (staged) {
          ell_rblock<true>(MODE, a, v, ma.w, zs_addr, sm.zs, w0, zglob, R, uc, sm.ring, mt);
        } else {
          ell_rblock<false>(MODE, a, v, ma.w, zs_addr, sm.zs, w0, zglob, R, uc, sm.ring, mt);
        }
        int nxt = 0;
        if (lane == 0) nxt = atomicAdd(sm.next, 1);
        nxt = __shfl_sync(FULL, nxt, 0);
        int4 na = make_int4(0, 0, 0, 0), nb = na;
        if (nxt < uB) {
          na = meta[2 * nxt];
          nb = meta[2 * nxt + 1];
        }
        u = nxt;
        ma = na;
        mb = nb;
      }
#ifdef CDK_PROFILE
      ell_prof_drain(a, t_ready);
#endif
      __syncthreads();  // window and counters reused by the next segment
      continue;
    }
    while (u < uB) {
      const UnitChunks uc = unit_chunks(g, u, lane);
      const int rb = g.ell_units[u];
      const int c = g.rblk_comm[rb];
      const double2 R = (c >= 0) ? sm.sR[c - cA] : make_double2(0.0, 0.0);
      if (staged) {
        ell_rblock<true>(MODE, a, v, rb, zs_addr, sm.zs, w0, zglob, R, uc, sm.ring);
      } else {
        ell_rblock<false>(MODE, a, v, rb, zs_addr, sm.zs, w0, zglob, R, uc, sm.ring);
      }
      int nxt = 0;
      if (lane == 0) nxt = atomicAdd(sm.next, 1);
      u = __shfl_sync(FULL, nxt, 0);
    }
    __syncthreads();  // window and counters reused by the next segment
  }
  if (a.n_peers > 1) __threadfence_system();  // peer stores before the barrier signal
}

__device__ __forceinline__ EllSmem ell_init(unsigned char *smem_raw, uint64_t *bar, double2 *sR,
                                            int *next, double2 *sP, int4 *meta,
                                            int smem_nodes) {
  EllSmem sm;
  sm.sP = sP;
  sm.meta = meta;
  sm.zs = reinterpret_cast<double2 *>(smem_raw);
  sm.bar = bar;
  sm.sR = sR;
  sm.next = next;
  sm.ring = smem_u32(smem_raw + ell_ring_offset(smem_nodes)) +
            (uint32_t)((threadIdx.x >> 5) * ELL_DEPTH * 512 + (threadIdx.x & 31) * 16);
  if (threadIdx.x == 0) mbar_init(bar, 1);
  if (threadIdx.x < 8) sm.zs[smem_nodes + threadIdx.x] = make_double2(0.0, 0.0);
  __syncthreads();
  return sm;
}

template <int MODE>
__global__ void __launch_bounds__(ELL_THREADS, CDK_ELL_MINBLOCKS) ell_stage_kernel(const StageArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ double2 sR[SEG_MAX_COMM];
  __shared__ int next;
  __shared__ double2 sP[ELL_PART_CAP];
  __shared__ __align__(16) int4 smeta[2 * ELL_META_CAP];
  if (a.n_peers > 1 && run_aborted(a.status)) return;  // a peer barrier timed out earlier
  const EllSmem sm = ell_init(smem_raw, &bar, sR, &next, sP, smeta, a.g.smem_nodes);
  uint32_t phase = 0;
  const unsigned long long t_cal = a.cta_cycles ? clock64() : 0ull;
#ifdef CDK_PROFILE
  const unsigned long long t_begin = clock64();
  unsigned long long g_begin;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_begin));
#endif
  ell_body(MODE, a, StageVar::of(a), sm, phase);
  if (a.cta_cycles) {  // calibration launches only
    __syncthreads();
    if (threadIdx.x == 0) a.cta_cycles[blockIdx.x] = clock64() - t_cal;
  }
#ifdef CDK_PROFILE
  __syncthreads();
  if (threadIdx.x == 0 && a.prof) {
    unsigned long long *p = a.prof + 6 * blockIdx.x;
    p[0] = clock64() - t_begin;
    p[1] = p[1] - t_begin;  // first segment ready (window + community sums)
    p[2] = p[3] = 0;
    unsigned long long g_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
    p[4] = g_begin;
    p[5] = g_end;
  }
#endif
}

// Persistent RK4 over the ELL layout (cooperative launch, grid barrier
// between stages; same sequencing as kuramoto_rk4_kernel).
template <bool PEERS>
__global__ void __launch_bounds__(ELL_THREADS, CDK_ELL_MINBLOCKS) ell_rk4_kernel(const __grid_constant__ StageArgs a,
                                                                 StepPtrs ptr,
                                                                 int64_t n_steps, double dt) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ double2 sR[SEG_MAX_COMM];
  __shared__ int next;
  __shared__ double2 sP[ELL_PART_CAP];
  __shared__ __align__(16) int4 smeta[2 * ELL_META_CAP];
  const EllSmem sm = ell_init(smem_raw, &bar, sR, &next, sP, smeta, a.g.smem_nodes);
  uint32_t phase = 0;
  unsigned int sync_idx = 0;
  const double h2 = dt / 2.0, h6 = dt / 6.0;
  unsigned int peer_target = ptr.pb_base;
#define CDK_STAGE_SYNC(last)                                                                 \
  do {                                                                                       \
    if (PEERS) {                                                                             \
      grid_sync(ptr.bar, ++sync_idx * gridDim.x);                                            \
      peer_target += (unsigned int)a.n_peers;                                                \
      if (blockIdx.x == 0 && threadIdx.x == 0) peer_barrier(ptr.pb, peer_target, a.status);  \
      if (!(last)) grid_sync(ptr.bar, ++sync_idx * gridDim.x);                               \
      if (run_aborted(a.status)) return;                                                     \
    } else if (!(last)) {                                                                    \
      grid_sync(ptr.bar, ++sync_idx * gridDim.x);                                            \
    }                                                                                        \
  } while (0)
  StageVar v = StageVar::of(a);
  for (int64_t step = 0; step < n_steps; ++step) {
    v.step_rel = step;
#if CDK_ELL_RK4_RT
    for (int st = 1; st <= 4; ++st) {  // z / partial buffers ping-pong: odd stages read [0]
      const int in = (st & 1) ? 0 : 1;
      v.z_in = ptr.z[in]; v.z_out = ptr.z[in ^ 1];
      v.part_in = ptr.part[in]; v.part_out = ptr.part[in ^ 1];
      v.peer_out = ptr.peer_z[in ^ 1];
      v.h = (st <= 2) ? h2 : (st == 3 ? dt : h6);
#ifdef CDK_PROFILE
      unsigned long long t0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#endif
      ell_body(st, a, v, sm, phase);
#ifdef CDK_PROFILE
      __syncthreads();
      if (a.prof && step == 1 && threadIdx.x == 0) {  // second step: stage timeline per CTA
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        a.prof[6 * gridDim.x + 8 * blockIdx.x + 2 * (st - 1)] = t0;
        a.prof[6 * gridDim.x + 8 * blockIdx.x + 2 * (st - 1) + 1] = t1;
      }
#endif
      CDK_STAGE_SYNC(st == 4 && step + 1 == n_steps);
    }
#else
#define CDK_ELL_STAGE(st, hh)                                                                \
  do {                                                                                       \
    const int in = ((st) & 1) ? 0 : 1;                                                       \
    v.z_in = ptr.z[in]; v.z_out = ptr.z[in ^ 1];                                             \
    v.part_in = ptr.part[in]; v.part_out = ptr.part[in ^ 1];                                 \
    v.peer_out = ptr.peer_z[in ^ 1];                                                         \
    v.h = (hh);                                                                              \
    ell_body((st), a, v, sm, phase);                                                         \
    CDK_STAGE_SYNC((st) == 4 && step + 1 == n_steps);                                        \
  } while (0)
    CDK_ELL_STAGE(1, h2);
    CDK_ELL_STAGE(2, h2);
    CDK_ELL_STAGE(3, dt);
    CDK_ELL_STAGE(4, h6);
#undef CDK_ELL_STAGE
#endif
  }
#undef CDK_STAGE_SYNC
}

// z = exp(i theta) and the canonical rblock partials (prepare).  One 8-lane
// group per rblock, lane t owns rows t, t+8, t+16, t+24 (same shape as the
// stage epilogue).
__global__ void __launch_bounds__(256) prepare_kernel(cdk_graph g, const double *theta,
                                                      double2 *z, double2 *part) {
  const int t = threadIdx.x & 7;
  const int rb = blockIdx.x * (blockDim.x >> 3) + (threadIdx.x >> 3);
  if (rb >= g.n_rblk) return;  // whole 8-lane groups exit together
  const unsigned gmask = 0xFFu << (threadIdx.x & 24);
  const int64_t row0 = g.rblk_row0[rb];
  const int64_t row1 = g.rblk_row0[rb + 1];
  const int nr = (int)(row1 - row0);
  double zr[4], zi[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int l = t + 8 * m;
    zr[m] = 0.0;
    zi[m] = 0.0;
    if (l < nr) {
      sincos(theta[row0 + l], &zi[m], &zr[m]);
      z[row0 + l] = make_double2(zr[m], zi[m]);
    }
  }
  double pr = ((zr[0] + zr[1]) + zr[2]) + zr[3], pim = ((zi[0] + zi[1]) + zi[2]) + zi[3];
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    pr += __shfl_xor_sync(gmask, pr, o);
    pim += __shfl_xor_sync(gmask, pim, o);
  }
  if (t == 0) part[rb] = make_double2(pr, pim);
}

__global__ void reset_status_kernel(cdk_run_status *st) {
  st->nonfinite = 0;
  st->first_bad_step = INT64_MAX;
  st->steps_done = 0;
  st->reserved = 0;
}

__global__ void advance_kernel(cdk_run_status *st, int64_t n) { st->steps_done += n; }

// ---------------------------------------------------------------------------

static int check_graph(const cdk_graph *g) {
  if (!g || g->n_rows < 0 || g->n_comm < 0 || g->n_rblk < 0 || g->n_seg < 0 || g->n_cta <= 0) {
    set_error("cdk_graph: invalid sizes");
    return CDK_INPUT;
  }
  if (g->ell_off) {
    if (g->cta_threads != ELL_THREADS || !g->xell_off || !g->ell_units || !g->seg_unit ||
        g->inter_blocks != 0 || g->intra_split) {
      set_error("cdk_graph (ELL): cta_threads must equal cdk_kuramoto_ell_threads(), xell_off "
                "set, no inter_blocks / intra_split");
      return CDK_INPUT;
    }
  } else if (g->cta_threads != NTHREADS) {
    set_error("cdk_graph: cta_threads must equal cdk_kuramoto_stage_threads()");
    return CDK_INPUT;
  }
  if (g->smem_nodes < 0 || (g->smem_nodes & 7) || g->seg_rows_cap <= 0) {
    set_error("cdk_graph: bad shared-memory capacities");
    return CDK_INPUT;
  }
  if (g->inter_blocks < 0 || g->inter_blocks > 4 ||
      (g->inter_blocks >= 2 && (!g->inter_split || g->inter_block_nodes <= 0))) {
    set_error("cdk_graph: inter_blocks must be 0..4 (inter_split set when >= 2)");
    return CDK_INPUT;
  }
  return CDK_OK;
}

static size_t stage_smem(const cdk_graph *g) {
  if (g->ell_off) return ell_smem_bytes(g->smem_nodes);
  return stage_smem_bytes(g->seg_rows_cap, g->smem_nodes, g->xs_cap);
}

// opt a kernel into the largest dynamic shared memory its static use leaves
template <typename K>
static int smem_optin(K kernel, int &attr_bytes, const char *what) {
  if (attr_bytes >= 0) return CDK_OK;
  cudaFuncAttributes fa{};
  cudaError_t e = cudaFuncGetAttributes(&fa, kernel);
  if (e != cudaSuccess) return cuda_status(e, what);
  const int dyn_max = cdk_max_smem_optin() - (int)fa.sharedSizeBytes;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max);
  if (e != cudaSuccess) return cuda_status(e, what);
  attr_bytes = dyn_max;
  return CDK_OK;
}

template <int MODE>
static int launch_ell_stage(const StageArgs &a, cudaStream_t st) {
  static int attr_bytes = -1;
  const size_t smem = stage_smem(&a.g);
  int rc = smem_optin(ell_stage_kernel<MODE>, attr_bytes, "cudaFuncSetAttribute(ell stage)");
  if (rc) return rc;
  if ((int)smem > attr_bytes) {
    set_error("ELL window does not fit the shared-memory opt-in limit");
    return CDK_INPUT;
  }
  ell_stage_kernel<MODE><<<a.g.n_cta, a.g.cta_threads, smem, st>>>(a);
  CDK_CHECK_LAUNCH("ell_stage_kernel");
  return CDK_OK;
}

template <int MODE>
static int launch_stage(const StageArgs &a, cudaStream_t st) {
  if (a.g.ell_off) return launch_ell_stage<MODE>(a, st);
  static int attr_bytes = -1;  // opt-in set once per instantiation (single-device process)
  const size_t smem = stage_smem(&a.g);
  if (attr_bytes < 0) {
    cudaFuncAttributes fa{};
    cudaError_t e = cudaFuncGetAttributes(&fa, kuramoto_stage_kernel<MODE>);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncGetAttributes(stage)");
    const int dyn_max = cdk_max_smem_optin() - (int)fa.sharedSizeBytes;
    e = cudaFuncSetAttribute(kuramoto_stage_kernel<MODE>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(stage)");
    attr_bytes = dyn_max;
  }
  if ((int)smem > attr_bytes) {
    set_error("community state does not fit the shared-memory opt-in limit");
    return CDK_INPUT;
  }
  if (a.g.inter_blocks > 0 && !(a.debug_flags & 1)) {
    inter_sweep_kernel<<<a.g.n_cta, SWEEP_THREADS, 0, st>>>(a);
    CDK_CHECK_LAUNCH("inter_sweep_kernel");
  }
  kuramoto_stage_kernel<MODE><<<a.g.n_cta, a.g.cta_threads, smem, st>>>(a);
  CDK_CHECK_LAUNCH("kuramoto_stage_kernel");
  return CDK_OK;
}

static int prepare(const cdk_graph *g, const double *theta, const Workspace &w, cudaStream_t st) {
  if (g->n_rblk > 0) {
    const int gpb = 32;  // 8-lane groups per block
    prepare_kernel<<<(g->n_rblk + gpb - 1) / gpb, 8 * gpb, 0, st>>>(*g, theta, w.z[0], w.part[0]);
    CDK_CHECK_LAUNCH("prepare_kernel");
  }
  reset_status_kernel<<<1, 1, 0, st>>>(w.status);
  CDK_CHECK_LAUNCH("reset_status_kernel");
  return CDK_OK;
}

static unsigned long long *g_prof = nullptr;

static StageArgs base_args(const cdk_graph *g, const Workspace &w, double *theta,
                           const double *omega, double k_over_n) {
  StageArgs a{};
  a.prof = g_prof;
  a.g = *g;
  a.status = w.status;
  a.theta = theta;
  a.omega = omega;
  a.ksum = w.ksum;
  a.xacc = w.xacc;
  a.peer_out = nullptr;
  a.n_peers = 1;
  a.rank = 0;
  {
    const char *e = getenv("CDK_SWEEP");
    a.sweep_mode = e ? atoi(e) : 0;
    const char *f = getenv("CDK_DEBUG_FLAGS");
    a.debug_flags = f ? atoi(f) : 0;
  }
  a.k_over_n = k_over_n;
  return a;
}

}  // namespace cdk

using namespace cdk;

extern "C" size_t cdk_kuramoto_workspace_bytes(const cdk_graph *g) {
  size_t total = 0;
  carve(g, nullptr, &total);
  return total;
}

extern "C" int cdk_kuramoto_prepare(const cdk_graph *g, const double *theta, void *workspace,
                                    void *stream) {
  int rc = check_graph(g);
  if (rc) return rc;
  Workspace w = carve(g, workspace, nullptr);
  return prepare(g, theta, w, as_stream(stream));
}

extern "C" int cdk_kuramoto_rhs(const cdk_graph *g, const double *theta, const double *omega,
                                double k_over_n, double *out, void *workspace, void *stream) {
  int rc = check_graph(g);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  Workspace w = carve(g, workspace, nullptr);
  rc = prepare(g, theta, w, st);
  if (rc) return rc;
  StageArgs a = base_args(g, w, const_cast<double *>(theta), omega, k_over_n);
  a.z_in = w.z[0];
  a.part_in = w.part[0];
  a.out = out;
  return launch_stage<0>(a, st);
}

static int launch_rk4_persistent(const StageArgs &a, const Workspace &w, int64_t n_steps,
                                 double dt, cudaStream_t st, const cdk_peers *peers = nullptr) {
  static int attr_bytes = -1, ell_attr = -1, ell_attr_peers = -1;
  const size_t smem = stage_smem(&a.g);
  const bool ell = a.g.ell_off != nullptr;
  if (ell) {
    int rc = smem_optin(ell_rk4_kernel<false>, ell_attr, "cudaFuncSetAttribute(ell rk4)");
    if (!rc) rc = smem_optin(ell_rk4_kernel<true>, ell_attr_peers, "cudaFuncSetAttribute(ell rk4)");
    if (rc) return rc;
    if ((int)smem > ell_attr) {
      set_error("ELL window does not fit the shared-memory opt-in limit");
      return CDK_INPUT;
    }
  } else if (attr_bytes < 0) {
    cudaFuncAttributes fa{};
    cudaError_t e = cudaFuncGetAttributes(&fa, kuramoto_rk4_kernel<false>);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncGetAttributes(rk4)");
    const int dyn_max = cdk_max_smem_optin() - (int)fa.sharedSizeBytes;
    e = cudaFuncSetAttribute(kuramoto_rk4_kernel<false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(kuramoto_rk4_kernel<true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(rk4)");
    attr_bytes = dyn_max;
  }
  if (!ell && (int)smem > attr_bytes) {
    set_error("community state does not fit the shared-memory opt-in limit");
    return CDK_INPUT;
  }
  StepPtrs ptr{};
  ptr.z[0] = w.z[0];
  ptr.z[1] = w.z[1];
  ptr.part[0] = w.part[0];
  ptr.part[1] = w.part[1];
  ptr.bar = w.bar;
  if (peers && peers->n_ranks > 1) {
    ptr.peer_z[0] = reinterpret_cast<double2 *const *>(peers->z0);
    ptr.peer_z[1] = reinterpret_cast<double2 *const *>(peers->z1);
    ptr.pb.bar = peers->bar;
    ptr.pb.mine = w.peer_bar;
    ptr.pb.n = peers->n_ranks;
    ptr.pb.wait = peers->wait;
    ptr.pb_base = peers->bar_base;
  }
  cudaError_t e = cudaMemsetAsync(w.bar, 0, sizeof(unsigned int), st);
  if (e != cudaSuccess) return cuda_status(e, "cudaMemsetAsync(grid barrier)");
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)a.g.n_cta);
  cfg.blockDim = dim3((unsigned)a.g.cta_threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (grid barrier)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const bool pe = peers && peers->n_ranks > 1;
  if (ell)
    e = pe ? cudaLaunchKernelEx(&cfg, ell_rk4_kernel<true>, a, ptr, n_steps, dt)
           : cudaLaunchKernelEx(&cfg, ell_rk4_kernel<false>, a, ptr, n_steps, dt);
  else
    e = pe ? cudaLaunchKernelEx(&cfg, kuramoto_rk4_kernel<true>, a, ptr, n_steps, dt)
           : cudaLaunchKernelEx(&cfg, kuramoto_rk4_kernel<false>, a, ptr, n_steps, dt);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (e != cudaSuccess) return cuda_status(e, "cudaLaunchKernelEx(kuramoto_rk4_kernel)");
  return CDK_OK;
}

extern "C" int cdk_kuramoto_rk4(const cdk_graph *g, double *theta, const double *omega,
                                double k_over_n, double dt, int64_t n_steps, void *workspace,
                                void *stream) {
  int rc = check_graph(g);
  if (rc) return rc;
  if (n_steps < 0) {
    set_error("n_steps < 0");
    return CDK_INPUT;
  }
  if (n_steps == 0) return CDK_OK;
  cudaStream_t st = as_stream(stream);
  Workspace w = carve(g, workspace, nullptr);
  StageArgs a = base_args(g, w, theta, omega, k_over_n);
  if (g->inter_blocks > 0) {
    // large graphs: per-stage launches (sweep + stage); launch gaps are
    // negligible against ~10 ms stages and the sweep needs its own smem config
    for (int64_t s = 0; s < n_steps; ++s) {
      a.step_rel = s;
      a.z_in = w.z[0]; a.z_out = w.z[1]; a.part_in = w.part[0]; a.part_out = w.part[1];
      a.h = dt / 2.0;
      if ((rc = launch_stage<1>(a, st))) return rc;
      a.z_in = w.z[1]; a.z_out = w.z[0]; a.part_in = w.part[1]; a.part_out = w.part[0];
      if ((rc = launch_stage<2>(a, st))) return rc;
      a.z_in = w.z[0]; a.z_out = w.z[1]; a.part_in = w.part[0]; a.part_out = w.part[1];
      a.h = dt;
      if ((rc = launch_stage<3>(a, st))) return rc;
      a.z_in = w.z[1]; a.z_out = w.z[0]; a.part_in = w.part[1]; a.part_out = w.part[0];
      a.h = dt / 6.0;
      if ((rc = launch_stage<4>(a, st))) return rc;
    }
  } else if ((rc = launch_rk4_persistent(a, w, n_steps, dt, st))) {
    return rc;
  }
  advance_kernel<<<1, 1, 0, st>>>(w.status, n_steps);
  CDK_CHECK_LAUNCH("advance_kernel");
  return CDK_OK;
}

extern "C" int cdk_kuramoto_status(const cdk_graph *g, const void *workspace, cdk_run_status *out,
                                   void *stream) {
  int rc = check_graph(g);
  if (rc) return rc;
  Workspace w = carve(g, const_cast<void *>(workspace), nullptr);
  cudaStream_t st = as_stream(stream);
  cudaError_t e = cudaMemcpyAsync(out, w.status, sizeof(cdk_run_status), cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return cuda_status(e, "cudaMemcpyAsync(status)");
  e = cudaStreamSynchronize(st);
  return cuda_status(e, "cudaStreamSynchronize(status)");
}

extern "C" int cdk_kuramoto_euler(const cdk_graph *g, double *theta, const double *omega,
                                  double k_over_n, double dt, int64_t n_steps, void *workspace,
                                  void *stream) {
  int rc = check_graph(g);
  if (rc) return rc;
  if (n_steps < 0) {
    set_error("n_steps < 0");
    return CDK_INPUT;
  }
  cudaStream_t st = as_stream(stream);
  Workspace w = carve(g, workspace, nullptr);
  StageArgs a = base_args(g, w, theta, omega, k_over_n);
  a.h = dt;
  for (int64_t s = 0; s < n_steps; ++s) {
    const int src = (int)(s & 1);
    a.step_rel = s;
    a.z_in = w.z[src]; a.z_out = w.z[src ^ 1];
    a.part_in = w.part[src]; a.part_out = w.part[src ^ 1];
    if ((rc = launch_stage<5>(a, st))) return rc;
  }
  if (n_steps & 1) {  // leave the current state in buffer 0 (the rk4/euler entry invariant)
    cudaError_t e = cudaMemcpyAsync(w.z[0], w.z[1], sizeof(double2) * (size_t)g->n_rows,
                                    cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(w.part[0], w.part[1], sizeof(double2) * (size_t)(g->n_rblk + 1),
                          cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_status(e, "cudaMemcpyAsync(euler parity)");
  }
  if (n_steps > 0) {
    advance_kernel<<<1, 1, 0, st>>>(w.status, n_steps);
    CDK_CHECK_LAUNCH("advance_kernel");
  }
  return CDK_OK;
}

extern "C" int cdk_kuramoto_rk4_stage(const cdk_graph *g, double *theta, const double *omega,
                                      double k_over_n, double dt, int stage, void *workspace,
                                      void *stream) {
  int rc = check_graph(g);
  if (rc) return rc;
  if (stage < 1 || stage > 4) {
    set_error("stage must be 1..4");
    return CDK_INPUT;
  }
  cudaStream_t st = as_stream(stream);
  Workspace w = carve(g, workspace, nullptr);
  StageArgs a = base_args(g, w, theta, omega, k_over_n);
  const int src = (stage - 1) & 1;
  a.z_in = w.z[src]; a.z_out = w.z[src ^ 1];
  a.part_in = w.part[src]; a.part_out = w.part[src ^ 1];
  a.step_rel = 0;
  switch (stage) {
    case 1: a.h = dt / 2.0; return launch_stage<1>(a, st);
    case 2: a.h = dt / 2.0; return launch_stage<2>(a, st);
    case 3: a.h = dt; return launch_stage<3>(a, st);
    default: a.h = dt / 6.0; return launch_stage<4>(a, st);
  }
}

// Planner calibration: one RK4 stage-1 launch of the ELL stage kernel with
// per-CTA cycle counts written to cycles[n_cta] (device).  Touches only the
// workspace's stage buffers (ksum, z[1], partials[1]); theta is unchanged.
extern "C" int cdk_kuramoto_stage_cycles(const cdk_graph *g, double *theta, const double *omega,
                                         double k_over_n, double dt, void *workspace,
                                         unsigned long long *cycles, void *stream) {
  int rc = check_graph(g);
  if (rc) return rc;
  if (!g->ell_off || !cycles) {
    set_error("cdk_kuramoto_stage_cycles: ELL graphs only, cycles required");
    return CDK_INPUT;
  }
  cudaStream_t st = as_stream(stream);
  Workspace w = carve(g, workspace, nullptr);
  StageArgs a = base_args(g, w, theta, omega, k_over_n);
  a.z_in = w.z[0]; a.z_out = w.z[1];
  a.part_in = w.part[0]; a.part_out = w.part[1];
  a.step_rel = 0;
  a.h = dt / 2.0;
  a.cta_cycles = cycles;
  return launch_stage<1>(a, st);
}

// CDK_PROFILE builds only: per-CTA phase cycles [total, staging, gather, epilogue]
// of the most recent stage launch are written to prof (device, 6*n_cta u64).
extern "C" CDK_API void cdk_debug_set_profile_buffer(void *prof) {
  g_prof = reinterpret_cast<unsigned long long *>(prof);
}

// Byte offsets of the workspace views (z[0], z[1], ksum, part[0], part[1],
// status) so a host driver can exchange stage state between ranks.
extern "C" int cdk_kuramoto_workspace_layout(const cdk_graph *g, int64_t *offsets) {
  if (!g || !offsets) return CDK_INPUT;
  char *base = reinterpret_cast<char *>(0x1000);  // any non-null base
  Workspace w = carve(g, base, nullptr);
  offsets[0] = reinterpret_cast<char *>(w.z[0]) - base;
  offsets[1] = reinterpret_cast<char *>(w.z[1]) - base;
  offsets[2] = reinterpret_cast<char *>(w.ksum) - base;
  offsets[3] = reinterpret_cast<char *>(w.part[0]) - base;
  offsets[4] = reinterpret_cast<char *>(w.part[1]) - base;
  offsets[5] = reinterpret_cast<char *>(w.status) - base;
  offsets[6] = reinterpret_cast<char *>(w.peer_bar) - base;
  return CDK_OK;
}

// advance the workspace's step counter (drivers that run stages one by one)
extern "C" int cdk_kuramoto_advance(const cdk_graph *g, void *workspace, int64_t n_steps,
                                    void *stream) {
  int rc = check_graph(g);
  if (rc) return rc;
  Workspace w = carve(g, workspace, nullptr);
  advance_kernel<<<1, 1, 0, as_stream(stream)>>>(w.status, n_steps);
  CDK_CHECK_LAUNCH("advance_kernel");
  return CDK_OK;
}

extern "C" int cdk_kuramoto_stage_threads(void) { return cdk::NTHREADS; }
extern "C" int cdk_kuramoto_stage_ctas_per_sm(void) { return CDK_STAGE_MINBLOCKS; }
extern "C" int cdk_kuramoto_ell_threads(void) { return cdk::ELL_THREADS; }
extern "C" int cdk_kuramoto_ell_ctas_per_sm(void) { return CDK_ELL_MINBLOCKS; }
extern "C" int cdk_kuramoto_ell_window_nodes(void) { return CDK_ELL_WINDOW; }

static int check_peers(const cdk_peers *p) {
  if (!p || p->n_ranks < 1 || p->rank < 0 || p->rank >= p->n_ranks ||
      (p->n_ranks > 1 && (!p->z0 || !p->z1 || !p->bar))) {
    set_error("cdk_peers: invalid table");
    return CDK_INPUT;
  }
  return CDK_OK;
}

static void apply_peers(StageArgs &a, const cdk_peers *p) {
  a.n_peers = p->n_ranks;
  a.rank = p->rank;
}

extern "C" int cdk_kuramoto_rk4_peers(const cdk_graph *g, double *theta, const double *omega,
                                      double k_over_n, double dt, int64_t n_steps,
                                      void *workspace, const cdk_peers *peers, void *stream) {
  int rc = check_graph(g);
  if (rc || (rc = check_peers(peers))) return rc;
  if (n_steps < 0) return set_error("n_steps < 0"), CDK_INPUT;
  if (n_steps == 0) return CDK_OK;
  cudaStream_t st = as_stream(stream);
  Workspace w = carve(g, workspace, nullptr);
  StageArgs a = base_args(g, w, theta, omega, k_over_n);
  apply_peers(a, peers);
  if (g->inter_blocks > 0) {  // per-stage launches: stage kernel, then the peer barrier
    PeerBar pb{peers->bar, w.peer_bar, peers->n_ranks, peers->wait};
    unsigned int target = peers->bar_base;
    auto z = [&](int k) { return k ? peers->z1 : peers->z0; };
    for (int64_t s = 0; s < n_steps; ++s) {
      a.step_rel = s;
      for (int stg = 1; stg <= 4; ++stg) {
        const int src = (stg - 1) & 1;
        a.z_in = w.z[src]; a.z_out = w.z[src ^ 1];
        a.part_in = w.part[src]; a.part_out = w.part[src ^ 1];
        a.peer_out = reinterpret_cast<double2 *const *>(z(src ^ 1));
        a.h = (stg == 3) ? dt : (stg == 4 ? dt / 6.0 : dt / 2.0);
        switch (stg) {
          case 1: rc = launch_stage<1>(a, st); break;
          case 2: rc = launch_stage<2>(a, st); break;
          case 3: rc = launch_stage<3>(a, st); break;
          default: rc = launch_stage<4>(a, st);
        }
        if (rc) return rc;
        if (peers->n_ranks > 1) {
          target += (unsigned int)peers->n_ranks;
          peer_barrier_kernel<<<1, 1, 0, st>>>(pb, target, w.status);
          CDK_CHECK_LAUNCH("peer_barrier_kernel");
        }
      }
    }
  } else if ((rc = launch_rk4_persistent(a, w, n_steps, dt, st, peers))) {
    return rc;
  }
  advance_kernel<<<1, 1, 0, st>>>(w.status, n_steps);
  CDK_CHECK_LAUNCH("advance_kernel");
  return CDK_OK;
}

extern "C" int cdk_kuramoto_rk4_stage_peers(const cdk_graph *g, double *theta, const double *omega,
                                            double k_over_n, double dt, int stage, void *workspace,
                                            const cdk_peers *peers, void *stream) {
  int rc = check_graph(g);
  if (rc || (rc = check_peers(peers))) return rc;
  if (stage < 1 || stage > 4) return set_error("stage must be 1..4"), CDK_INPUT;
  cudaStream_t st = as_stream(stream);
  Workspace w = carve(g, workspace, nullptr);
  StageArgs a = base_args(g, w, theta, omega, k_over_n);
  apply_peers(a, peers);
  const int src = (stage - 1) & 1;
  a.z_in = w.z[src]; a.z_out = w.z[src ^ 1];
  a.part_in = w.part[src]; a.part_out = w.part[src ^ 1];
  a.peer_out = reinterpret_cast<double2 *const *>(src ^ 1 ? peers->z1 : peers->z0);
  a.step_rel = 0;
  switch (stage) {
    case 1: a.h = dt / 2.0; rc = launch_stage<1>(a, st); break;
    case 2: a.h = dt / 2.0; rc = launch_stage<2>(a, st); break;
    case 3: a.h = dt; rc = launch_stage<3>(a, st); break;
    default: a.h = dt / 6.0; rc = launch_stage<4>(a, st);
  }
  if (rc) return rc;
  if (peers->n_ranks > 1) {
    PeerBar pb{peers->bar, w.peer_bar, peers->n_ranks, peers->wait};
    peer_barrier_kernel<<<1, 1, 0, st>>>(pb, peers->bar_base + (unsigned int)peers->n_ranks,
                                         w.status);
    CDK_CHECK_LAUNCH("peer_barrier_kernel");
  }
  return CDK_OK;
}
