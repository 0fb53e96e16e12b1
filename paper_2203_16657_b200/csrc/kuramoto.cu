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
  double2 *R[2];
  double2 *part;
  int32_t *cnt;
  cdk_run_status *status;
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
  const size_t n = (size_t)g->n_rows, m = (size_t)g->n_comm;
  // +16: staged windows are rounded out to 8-node (128-byte) boundaries
  w.z[0] = (double2 *)take((n + 16) * sizeof(double2));
  w.z[1] = (double2 *)take((n + 16) * sizeof(double2));
  w.ksum = (double *)take(n * sizeof(double));
  w.R[0] = (double2 *)take((m + 1) * sizeof(double2));
  w.R[1] = (double2 *)take((m + 1) * sizeof(double2));
  w.part = (double2 *)take(((size_t)g->n_rblk + 1) * sizeof(double2));
  w.cnt = (int32_t *)take((m + 1) * sizeof(int32_t));
  w.status = (cdk_run_status *)take(sizeof(cdk_run_status));
  if (total) *total = off;
  return w;
}

struct StageArgs {
  cdk_graph g;
  const double2 *z_in;
  double2 *z_out;
  const double2 *R_in;
  double2 *R_out;
  double2 *part;
  int32_t *cnt;
  cdk_run_status *status;
  double *theta;
  const double *omega;
  double *ksum;
  double *out;  // MODE 0
  double k_over_n;
  double h;     // stage increment (dt/2, dt/2, dt) or dt/6 at stage 4
  int64_t step_rel;
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

// 8 uint16 intra columns (one 16-byte chunk): subtract their z (sign -1).
// Staged (shared memory): branch-free, padding (0xFFFF) is clamped onto a zero
// slot one past the window capacity.  Unstaged (global, huge communities):
// predicated loads.
template <bool STAGED>
__device__ __forceinline__ void gather8(const uint4 w, const double2 *__restrict__ zbase,
                                        uint32_t zero_slot, double &sr, double &si) {
  const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t u = (wv[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu;
    if (STAGED) {
      const double2 z = zbase[min(u, zero_slot)];
      sr -= z.x;
      si -= z.y;
    } else if (u != CDK_INTRA_PAD) {
      const double2 z = ldg(zbase + u);
      sr -= z.x;
      si -= z.y;
    }
  }
}

// sparse sums of two rows (A, B) of an unstaged segment (global gathers)
__device__ __forceinline__ void gather_rows_global(const cdk_graph &g,
                                                   const double2 *__restrict__ z_in,
                                                   const double2 *__restrict__ zbase, int64_t iA,
                                                   int64_t iB, bool hasB, int t, double &ar,
                                                   double &ai, double &br, double &bi) {
  const int64_t eA0 = ldg(g.intra_ptr + iA), eA1 = ldg(g.intra_ptr + iA + 1);
  const int64_t xA0 = ldg(g.inter_ptr + iA), xA1 = ldg(g.inter_ptr + iA + 1);
  const int64_t eB0 = ldg(g.intra_ptr + iB);
  const int64_t eB1 = hasB ? ldg(g.intra_ptr + iB + 1) : eB0;
  const int64_t xB0 = ldg(g.inter_ptr + iB);
  const int64_t xB1 = hasB ? ldg(g.inter_ptr + iB + 1) : xB0;
  const uint4 *colv = reinterpret_cast<const uint4 *>(g.intra_col);
  for (int64_t p = eA0 + 8 * t; p < eA1; p += 64)
    gather8<false>(ldg(colv + (p >> 3)), zbase, 0, ar, ai);
  for (int64_t p = eB0 + 8 * t; p < eB1; p += 64)
    gather8<false>(ldg(colv + (p >> 3)), zbase, 0, br, bi);
  for (int64_t p = xA0 + t; p < xA1; p += 8) {
    const double2 z = ldg(z_in + ldg(g.inter_col + p));
    ar += z.x;
    ai += z.y;
  }
  for (int64_t p = xB0 + t; p < xB1; p += 8) {
    const double2 z = ldg(z_in + ldg(g.inter_col + p));
    br += z.x;
    bi += z.y;
  }
}

// ---------------------------------------------------------------------------
// TMA-pipelined, barrier-free stage kernel.  One CTA per SM, 32 warps:
//   warp 31 (one lane) = producer: streams each tile's CSR slices (uint16
//     intra columns, int32 inter columns, int32 row table) into a 2-slot
//     shared-memory ring with bulk async copies (full/empty mbarriers);
//   warps 0..30 = 124 consumer groups of 8 lanes.  Per segment, one bulk copy
//     stages the node window of z_in in shared memory.  Per tile, groups claim
//     rows from a shared counter (dynamic balance, no CTA barrier), gather
//     the row from the window, store the row sum, and count the row into its
//     rblock; the group that completes an rblock runs its epilogue (RK4 stage
//     update, sincos, canonical rblock partial, community completion).  The
//     slot is refilled once every group has left the tile and the tile's last
//     epilogue is done (empty barrier expects NGROUPS + 1 arrivals).
// Unstaged segments (communities above the window capacity, NONE pool) are
// processed from global memory with CTA barriers (rare path).
// All reductions have a fixed shape => bitwise deterministic and independent
// of the schedule (and so of the GPU count).
// ---------------------------------------------------------------------------
constexpr int TILE_ROWS = 128;
constexpr int TILE_E = 8192;
constexpr int TILE_X = 1024;
constexpr int TILE_TAB = 2 * (TILE_ROWS + 4) + TILE_ROWS;
constexpr int RING = 4;
constexpr int NTHREADS = 1024;
constexpr int NCONS_WARPS = 31;
constexpr int NCONS = NCONS_WARPS * 32;
constexpr int NGROUPS = NCONS / 8;
constexpr int CNT_STRIDE = TILE_ROWS + 4;

struct TileSlot {
  uint16_t cols[TILE_E];
  int32_t xcol[TILE_X];
  int32_t tab[TILE_TAB];
};
static_assert(sizeof(TileSlot) % 16 == 0, "tile slot must keep 16-byte alignment");

__device__ __forceinline__ void consumer_bar() {
  asm volatile("bar.sync 1, %0;" ::"r"(NCONS) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Epilogue of one rblock by an 8-lane group: lane t owns rows t, t+8, t+16,
// t+24 of the rblock.  Canonical rblock partial: per-lane sum in row order,
// then the 8-lane butterfly.  The group that completes community c reduces R.
template <int MODE>
__device__ __forceinline__ void epilogue_group(const StageArgs &a, int rb, int t, unsigned gmask,
                                               const double2 *acc, int64_t accrow0, bool staged,
                                               const double2 *zs, int64_t w0) {
  const cdk_graph &g = a.g;
  const int64_t rrow0 = g.rblk_row0[rb];
  const int64_t rrow1 = (rb + 1 < g.n_rblk) ? g.rblk_row0[rb + 1] : g.n_rows;
  const int nr = (int)(rrow1 - rrow0);
  const int c = g.rblk_comm[rb];
  const double2 R = (c >= 0) ? ldcg2(a.R_in + c) : make_double2(0.0, 0.0);
  const double kn = a.k_over_n;
  double pr = 0.0, pim = 0.0;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int l = t + 8 * m;
    if (l < nr) {
      const int64_t i = rrow0 + l;
      const double2 ac = acc[i - accrow0];
      const double2 zi = staged ? zs[i - w0] : ldg(a.z_in + i);
      double k = ldg(a.omega + i) + kn * (R.y * zi.x - R.x * zi.y);
      k = k + kn * (ac.y * zi.x - ac.x * zi.y);
      if (MODE == 0) {
        a.out[i] = k;
      } else {
        const double th0 = a.theta[i];
        double thn;
        if (MODE == 1) {
          a.ksum[i] = k;
          thn = add_rn(th0, mul_rn(a.h, k));
        } else if (MODE == 2 || MODE == 3) {
          a.ksum[i] = add_rn(a.ksum[i], mul_rn(2.0, k));
          thn = add_rn(th0, mul_rn(a.h, k));
        } else {  // MODE 4: x + dt/6 (k1 + 2k2 + 2k3 + k4); MODE 5: Euler x + dt k
          const double ks = (MODE == 4) ? add_rn(a.ksum[i], k) : k;
          thn = wrap_phase(add_rn(th0, mul_rn(a.h, ks)));
          a.theta[i] = thn;
          if (!isfinite(thn)) {
            atomicAdd(reinterpret_cast<unsigned long long *>(&a.status->nonfinite), 1ull);
            atomicMin(reinterpret_cast<long long *>(&a.status->first_bad_step),
                      (long long)(a.status->steps_done + a.step_rel + 1));
          }
        }
        double sn, cs;
        sincos(thn, &sn, &cs);
        a.z_out[i] = make_double2(cs, sn);
        pr += cs;
        pim += sn;
      }
    }
  }
  if (MODE != 0 && c >= 0) {
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      pr += __shfl_xor_sync(gmask, pr, o);
      pim += __shfl_xor_sync(gmask, pim, o);
    }
    const int leader = (threadIdx.x & 31) & 24;
    int last = 0;
    if (t == 0) {
      a.part[rb] = make_double2(pr, pim);
      __threadfence();
      const int total = g.comm_rblk_off[c + 1] - g.comm_rblk_off[c];
      last = (atomicAdd(a.cnt + c, 1) + 1 == total);
    }
    last = __shfl_sync(gmask, last, leader);
    if (last) {  // this group finished community c: reduce its partials
      __threadfence();
      const double2 Rn =
          reduce_comm8(a.part, g.comm_rblk_off[c], g.comm_rblk_off[c + 1], t, gmask);
      if (t == 0) {
        a.R_out[c] = Rn;
        a.cnt[c] = 0;
      }
    }
  }
}

// MODE 0: out = f(theta) (single RHS).  MODE 1..4: RK4 stage.  MODE 5: Euler step.
template <int MODE>
__global__ void __launch_bounds__(NTHREADS, 1) kuramoto_stage_kernel(const StageArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // full: tile data landed (TMA tx); empty: all rows of the tile gathered
  // (slot reusable).  A group only waits for tiles it has rows in, so it may
  // skip fills: s_slot_tag[b] names the tile currently filling/filled in slot
  // b (set by the producer before the copies) and is checked before the
  // parity wait; s_acc_owner[b] names the tile allowed to use accumulator
  // slot b (advanced by the tile's last epilogue).
  __shared__ __align__(8) uint64_t bar_full[RING], bar_empty[RING], bar_win;
  __shared__ int s_rows_done[RING], s_rb_done[RING];
  __shared__ volatile int s_slot_tag[RING], s_acc_owner[RING];
  const cdk_graph &g = a.g;
  TileSlot *ring = reinterpret_cast<TileSlot *>(smem_raw);
  double2 *accs = reinterpret_cast<double2 *>(smem_raw + RING * sizeof(TileSlot));
  int *cnt_rb = reinterpret_cast<int *>(accs + RING * TILE_ROWS);
  double2 *zs = reinterpret_cast<double2 *>(cnt_rb + RING * CNT_STRIDE);
  const uint32_t zero_slot = (uint32_t)g.smem_nodes;  // zs[smem_nodes] == 0
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int segA = g.cta_seg[blockIdx.x], segB = g.cta_seg[blockIdx.x + 1];
  for (int i = tid; i < RING * CNT_STRIDE; i += NTHREADS) cnt_rb[i] = 0;
  if (tid == 0) {
    for (int b = 0; b < RING; ++b) {
      mbar_init(&bar_full[b], 1);
      mbar_init(&bar_empty[b], 1);
      s_rows_done[b] = 0;
      s_rb_done[b] = 0;
      s_slot_tag[b] = -1;
      s_acc_owner[b] = b;
    }
    mbar_init(&bar_win, 1);
    zs[zero_slot] = make_double2(0.0, 0.0);
  }
  __syncthreads();

  if (warp == NCONS_WARPS) {  // ---------------- producer ----------------
    if (lane == 0) {
      int k = 0;
      for (int s = segA; s < segB; ++s) {
        for (int ti = g.seg_tile[s]; ti < g.seg_tile[s + 1]; ++ti, ++k) {
          const int b = k % RING, n = k / RING;
          if (n > 0) mbar_wait(&bar_empty[b], (n - 1) & 1);
          s_slot_tag[b] = k;
          const cdk_tile T = g.tiles[ti];
          const int64_t r0 = g.rblk_row0[T.rblk0];
          const int64_t r1 = (T.rblk1 < g.n_rblk) ? g.rblk_row0[T.rblk1] : g.n_rows;
          const int nrow = (int)(r1 - r0);
          const int half = (nrow + 1 + 3) & ~3;
          const uint32_t be = (uint32_t)T.ne * 2u, bx = (uint32_t)T.nxa * 4u,
                         bt = (uint32_t)(2 * half + ((nrow + 3) & ~3)) * 4u;
          mbar_expect_tx(&bar_full[b], be + bx + bt);
          if (be) bulk_g2s(ring[b].cols, g.intra_col + T.e0, be, &bar_full[b]);
          if (bx) bulk_g2s(ring[b].xcol, g.inter_col + T.x0a, bx, &bar_full[b]);
          bulk_g2s(ring[b].tab, g.tile_tab + T.tab_off, bt, &bar_full[b]);
        }
      }
    }
    return;
  }

  // ---------------- consumers (warps 0..30) ----------------
  const int t = lane & 7;
  const int grp = tid >> 3;
  const int leader = lane & 24;
  const unsigned gmask = 0xFFu << leader;  // this 8-lane group only
  const double2 *__restrict__ z_in = a.z_in;
  int k = 0;
  int rot = 0;  // rows of the CTA's earlier tiles, mod NGROUPS (rotating row assignment)
  uint32_t win_par = 0;
  for (int s = segA; s < segB; ++s) {
    const int rbA = g.seg_rblk[s], rbB = g.seg_rblk[s + 1];
    const int64_t w0 = g.seg_win[2 * s], w1 = g.seg_win[2 * s + 1];
    const bool staged = w1 > w0;
    if (staged) {
      if (tid == 0) {
        fence_proxy_async_smem();  // prior generic reads of zs before the async overwrite
        const uint32_t bytes = (uint32_t)((w1 - w0) * sizeof(double2));
        mbar_expect_tx(&bar_win, bytes);
        bulk_g2s(zs, z_in + w0, bytes, &bar_win);
      }
      mbar_wait(&bar_win, win_par);
      win_par ^= 1;
      for (int ti = g.seg_tile[s]; ti < g.seg_tile[s + 1]; ++ti, ++k) {
        const cdk_tile T = g.tiles[ti];
        const int64_t r0 = g.rblk_row0[T.rblk0];
        const int64_t r1 = (T.rblk1 < g.n_rblk) ? g.rblk_row0[T.rblk1] : g.n_rows;
        const int nrow = (int)(r1 - r0);
        int r = grp - rot;
        if (r < 0) r += NGROUPS;
        rot += nrow;
        rot %= NGROUPS;
        if (r >= nrow) continue;  // no row of this tile for this group
        const int b = k % RING, n = k / RING;
        while (s_slot_tag[b] != k) __nanosleep(32);
        mbar_wait(&bar_full[b], n & 1);
        while (s_acc_owner[b] != k) __nanosleep(32);
        __threadfence_block();
        const TileSlot &S = ring[b];
        const int half = (nrow + 1 + 3) & ~3;
        const int nrb = T.rblk1 - T.rblk0;
        double2 *acc = accs + b * TILE_ROWS;
        int *cnt = cnt_rb + b * CNT_STRIDE;
        for (; r < nrow; r += NGROUPS) {
          const int ie0 = S.tab[r], ie1 = S.tab[r + 1];
          const int xe0 = S.tab[half + r], xe1 = S.tab[half + r + 1];
          const int lrb = S.tab[2 * half + r];
          DBG_CHECK(ie0 >= 0 && ie0 <= ie1 && ie1 <= T.ne && xe0 >= 0 && xe0 <= xe1 &&
                        xe1 <= T.nxa && lrb >= 0 && lrb < nrb,
                    "tab r=%d nrow=%d ie %d %d xe %d %d lrb %d k=%d ti=%d", r, nrow, ie0, ie1, xe0,
                    xe1, lrb, k, ti);
          const int32_t j = (xe0 + t < xe1) ? S.xcol[xe0 + t] : -1;
          DBG_CHECK(j < (int32_t)g.n_rows, "inter col %d r=%d k=%d ti=%d", j, r, k, ti);
          const double2 zx = (j >= 0) ? ldg(z_in + j) : make_double2(0.0, 0.0);
          double sr = 0.0, si = 0.0;
          for (int p = ie0 + 8 * t; p < ie1; p += 64)
            gather8<true>(*reinterpret_cast<const uint4 *>(S.cols + p), zs, zero_slot, sr, si);
          sr += zx.x;
          si += zx.y;
          for (int p = xe0 + 8 + t; p < xe1; p += 8) {
            const double2 z = ldg(z_in + S.xcol[p]);
            sr += z.x;
            si += z.y;
          }
#pragma unroll
          for (int o = 4; o > 0; o >>= 1) {
            sr += __shfl_xor_sync(gmask, sr, o);
            si += __shfl_xor_sync(gmask, si, o);
          }
          int last = 0;
          if (t == 0) {
            acc[r] = make_double2(sr, si);
            __threadfence_block();
            const int rb = T.rblk0 + lrb;
            const int64_t e = (rb + 1 < g.n_rblk) ? g.rblk_row0[rb + 1] : g.n_rows;
            last = (atomicAdd(&cnt[lrb], 1) + 1 == (int)(e - g.rblk_row0[rb]));
            DBG_CHECK(cnt[lrb] <= 32, "rblock counter overflow %d", cnt[lrb]);
            if (atomicAdd(&s_rows_done[b], 1) + 1 == nrow) {  // slot data fully consumed
              s_rows_done[b] = 0;
              mbar_arrive(&bar_empty[b]);
            }
          }
          last = __shfl_sync(gmask, last, leader);
          if (last) {
            __threadfence_block();
            epilogue_group<MODE>(a, T.rblk0 + lrb, t, gmask, acc, r0, true, zs, w0);
            if (t == 0 && atomicAdd(&s_rb_done[b], 1) + 1 == nrb) {  // accumulators free
              for (int i = 0; i < nrb; ++i) cnt[i] = 0;
              s_rb_done[b] = 0;
              __threadfence_block();
              s_acc_owner[b] = k + RING;
            }
          }
        }
      }
    } else {
      const int64_t row0 = g.rblk_row0[rbA];
      const int64_t row1 = (rbB < g.n_rblk) ? g.rblk_row0[rbB] : g.n_rows;
      const int nrows = (int)(row1 - row0);
      const double2 *zbase = z_in + g.seg_base[s];
      double2 *acc = accs;  // all staged tiles' epilogues finished (segment barrier)
      for (int r = grp; r < nrows; r += 2 * NGROUPS) {
        const int rB = r + NGROUPS;
        const bool hasB = rB < nrows;
        double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
        gather_rows_global(g, z_in, zbase, row0 + r, row0 + (hasB ? rB : r), hasB, t, ar, ai, br,
                           bi);
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
          ar += __shfl_xor_sync(gmask, ar, o);
          ai += __shfl_xor_sync(gmask, ai, o);
          br += __shfl_xor_sync(gmask, br, o);
          bi += __shfl_xor_sync(gmask, bi, o);
        }
        if (t == 0) {
          acc[r] = make_double2(ar, ai);
          if (hasB) acc[rB] = make_double2(br, bi);
        }
      }
      consumer_bar();
      for (int rb = rbA + grp; rb < rbB; rb += NGROUPS)
        epilogue_group<MODE>(a, rb, t, gmask, acc, row0, false, zs, 0);
    }
    consumer_bar();  // zs / accs reuse by the next segment
  }
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
  const int64_t row1 = (rb + 1 < g.n_rblk) ? g.rblk_row0[rb + 1] : g.n_rows;
  const int nr = (int)(row1 - row0);
  double pr = 0.0, pim = 0.0;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int l = t + 8 * m;
    if (l < nr) {
      double sn, cs;
      sincos(theta[row0 + l], &sn, &cs);
      z[row0 + l] = make_double2(cs, sn);
      pr += cs;
      pim += sn;
    }
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    pr += __shfl_xor_sync(gmask, pr, o);
    pim += __shfl_xor_sync(gmask, pim, o);
  }
  if (t == 0) part[rb] = make_double2(pr, pim);
}

__global__ void comm_reduce_kernel(cdk_graph g, const double2 *part, double2 *R, int32_t *cnt,
                                   cdk_run_status *st) {
  const int c = blockIdx.x;
  const int lane = threadIdx.x;  // blockDim.x == 8
  if (c < g.n_comm) {
    const double2 Rc = reduce_comm8(part, g.comm_rblk_off[c], g.comm_rblk_off[c + 1], lane, 0xFFu);
    if (lane == 0) {
      R[c] = Rc;
      cnt[c] = 0;
    }
  }
  if (c == 0 && lane == 0) {
    st->nonfinite = 0;
    st->first_bad_step = INT64_MAX;
    st->steps_done = 0;
    st->reserved = 0;
  }
}

__global__ void advance_kernel(cdk_run_status *st, int64_t n) { st->steps_done += n; }

// ---------------------------------------------------------------------------

static int check_graph(const cdk_graph *g) {
  if (!g || g->n_rows < 0 || g->n_comm < 0 || g->n_rblk < 0 || g->n_seg < 0 || g->n_cta <= 0) {
    set_error("cdk_graph: invalid sizes");
    return CDK_INPUT;
  }
  if (g->cta_threads != NTHREADS) {
    set_error("cdk_graph: cta_threads must be 1024");
    return CDK_INPUT;
  }
  if (g->smem_nodes < 0 || g->seg_rows_cap <= 0 || g->seg_rows_cap > TILE_ROWS) {
    set_error("cdk_graph: bad shared-memory capacities");
    return CDK_INPUT;
  }
  return CDK_OK;
}

static size_t stage_smem(const cdk_graph *g) {
  return RING * sizeof(TileSlot) + (size_t)RING * TILE_ROWS * sizeof(double2) +
         RING * CNT_STRIDE * sizeof(int) + ((size_t)g->smem_nodes + 8) * sizeof(double2);
}

template <int MODE>
static int launch_stage(const StageArgs &a, cudaStream_t st) {
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
  kuramoto_stage_kernel<MODE><<<a.g.n_cta, a.g.cta_threads, smem, st>>>(a);
  CDK_CHECK_LAUNCH("kuramoto_stage_kernel");
  return CDK_OK;
}

static int prepare(const cdk_graph *g, const double *theta, const Workspace &w, cudaStream_t st) {
  if (g->n_rblk > 0) {
    const int gpb = 32;  // 8-lane groups per block
    prepare_kernel<<<(g->n_rblk + gpb - 1) / gpb, 8 * gpb, 0, st>>>(*g, theta, w.z[0], w.part);
    CDK_CHECK_LAUNCH("prepare_kernel");
  }
  const int m = (int)g->n_comm;
  comm_reduce_kernel<<<m > 0 ? m : 1, 8, 0, st>>>(*g, w.part, w.R[0], w.cnt, w.status);
  CDK_CHECK_LAUNCH("comm_reduce_kernel");
  return CDK_OK;
}

static StageArgs base_args(const cdk_graph *g, const Workspace &w, double *theta,
                           const double *omega, double k_over_n) {
  StageArgs a{};
  a.g = *g;
  a.part = w.part;
  a.cnt = w.cnt;
  a.status = w.status;
  a.theta = theta;
  a.omega = omega;
  a.ksum = w.ksum;
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
  a.R_in = w.R[0];
  a.out = out;
  return launch_stage<0>(a, st);
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
  cudaStream_t st = as_stream(stream);
  Workspace w = carve(g, workspace, nullptr);
  StageArgs a = base_args(g, w, theta, omega, k_over_n);
  const double h2 = dt / 2.0, h6 = dt / 6.0;
  for (int64_t s = 0; s < n_steps; ++s) {
    a.step_rel = s;
    // stage 1: z0 -> z1
    a.z_in = w.z[0]; a.z_out = w.z[1]; a.R_in = w.R[0]; a.R_out = w.R[1]; a.h = h2;
    if ((rc = launch_stage<1>(a, st))) return rc;
    a.z_in = w.z[1]; a.z_out = w.z[0]; a.R_in = w.R[1]; a.R_out = w.R[0]; a.h = h2;
    if ((rc = launch_stage<2>(a, st))) return rc;
    a.z_in = w.z[0]; a.z_out = w.z[1]; a.R_in = w.R[0]; a.R_out = w.R[1]; a.h = dt;
    if ((rc = launch_stage<3>(a, st))) return rc;
    a.z_in = w.z[1]; a.z_out = w.z[0]; a.R_in = w.R[1]; a.R_out = w.R[0]; a.h = h6;
    if ((rc = launch_stage<4>(a, st))) return rc;
  }
  if (n_steps > 0) {
    advance_kernel<<<1, 1, 0, st>>>(w.status, n_steps);
    CDK_CHECK_LAUNCH("advance_kernel");
  }
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
    a.z_in = w.z[src]; a.z_out = w.z[src ^ 1]; a.R_in = w.R[src]; a.R_out = w.R[src ^ 1];
    if ((rc = launch_stage<5>(a, st))) return rc;
  }
  if (n_steps & 1) {  // leave the current state in buffer 0 (the rk4/euler entry invariant)
    cudaError_t e = cudaMemcpyAsync(w.z[0], w.z[1], sizeof(double2) * (size_t)g->n_rows,
                                    cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(w.R[0], w.R[1], sizeof(double2) * (size_t)(g->n_comm + 1),
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
  a.z_in = w.z[src]; a.z_out = w.z[src ^ 1]; a.R_in = w.R[src]; a.R_out = w.R[src ^ 1];
  a.step_rel = 0;
  switch (stage) {
    case 1: a.h = dt / 2.0; return launch_stage<1>(a, st);
    case 2: a.h = dt / 2.0; return launch_stage<2>(a, st);
    case 3: a.h = dt; return launch_stage<3>(a, st);
    default: a.h = dt / 6.0; return launch_stage<4>(a, st);
  }
}
