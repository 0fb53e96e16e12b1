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

constexpr int RB = 32;  // rows per rblock

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

// Sum of rblock partials of community c, fixed order (lane-strided, butterfly).
__device__ __forceinline__ double2 reduce_comm(const double2 *part, int b0, int b1, int lane) {
  double sr = 0.0, si = 0.0;
  for (int b = b0 + lane; b < b1; b += 32) {
    double2 v = ldcg2(part + b);
    sr += v.x;
    si += v.y;
  }
  sr = warp_sum(sr);
  si = warp_sum(si);
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
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra LAB_WAIT;\n"
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

// MODE 0: out = f(theta) (single RHS).  MODE 1..4: RK4 stage.  MODE 5: Euler step.
//
// Per segment (a run of whole rblocks, see cdk_graph):
//  1. one thread bulk-copies the segment's node window of z_in into shared
//     memory (async proxy, mbarrier completion);
//  2. gather: 8-lane groups take rows round-robin; each lane streams 16-byte
//     chunks (8 uint16 columns) of the row's intra run and gathers z from
//     shared memory, then the row's inter entries from global memory (L2); the
//     group reduces (fixed butterfly) and writes the row's sparse sum to a
//     shared-memory accumulator;
//  3. epilogue: warps take rblocks; lane = row: k = omega + K/N Im((R_c + acc) conj z),
//     RK4 stage update, z_next = exp(i theta_next), rblock partial of R_next;
//     the warp that completes a community's last rblock reduces R_next[c].
template <int MODE>
__global__ void __launch_bounds__(512, 2) kuramoto_stage_kernel(const StageArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bar;
  const cdk_graph &g = a.g;
  double2 *zs = reinterpret_cast<double2 *>(smem_raw);
  double2 *accs = zs + g.smem_nodes;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  const int t = lane & 7;                 // lane within the 8-lane row group
  const int grp = tid >> 3, ngrp = blockDim.x >> 3;
  const int segA = g.cta_seg[blockIdx.x], segB = g.cta_seg[blockIdx.x + 1];
  if (tid == 0) mbar_init(&bar, 1);
  __syncthreads();
  uint32_t parity = 0;

  for (int s = segA; s < segB; ++s) {
    const int rbA = g.seg_rblk[s], rbB = g.seg_rblk[s + 1];
    const int64_t row0 = g.rblk_row0[rbA];
    const int64_t row1 = (rbB < g.n_rblk) ? g.rblk_row0[rbB] : g.n_rows;
    const int64_t w0 = g.seg_win[2 * s], w1 = g.seg_win[2 * s + 1];
    const int64_t base = g.seg_base[s];
    const bool staged = w1 > w0;
    if (staged) {
      if (tid == 0) {
        fence_proxy_async_smem();  // prior generic reads of zs ordered before the async write
        const uint32_t bytes = (uint32_t)((w1 - w0) * sizeof(double2));
        mbar_expect_tx(&bar, bytes);
        bulk_g2s(zs, a.z_in + w0, bytes, &bar);
      }
      mbar_wait(&bar, parity);
      parity ^= 1;
    }
    const double2 *zsrc = staged ? zs : a.z_in + base;

    // ---- gather phase --------------------------------------------------
    const int nrows = (int)(row1 - row0);
    for (int r = grp; r < nrows; r += ngrp) {
      const int64_t i = row0 + r;
      const int64_t e0 = ldg(g.intra_ptr + i), e1 = ldg(g.intra_ptr + i + 1);
      const int64_t x0 = ldg(g.inter_ptr + i), x1 = ldg(g.inter_ptr + i + 1);
      double sr = 0.0, si = 0.0;
      for (int64_t p = e0 + 8 * t; p < e1; p += 64) {
        const uint4 w = ldg(reinterpret_cast<const uint4 *>(g.intra_col + p));
        const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t u = (wv[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu;
          if (u != CDK_INTRA_PAD) {
            const double2 z = staged ? zs[u] : ldg(zsrc + u);
            sr -= z.x;
            si -= z.y;
          }
        }
      }
      for (int64_t p = x0 + t; p < x1; p += 8) {
        const double2 z = ldg(a.z_in + ldg(g.inter_col + p));
        sr += z.x;
        si += z.y;
      }
      // only this 8-lane group is guaranteed to be here (rows may end mid-warp)
      const unsigned gmask = 0xFFu << (lane & 24);
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        sr += __shfl_xor_sync(gmask, sr, o);
        si += __shfl_xor_sync(gmask, si, o);
      }
      if (t == 0) accs[r] = make_double2(sr, si);
    }
    __syncthreads();

    // ---- epilogue: one warp per rblock, lane = row ------------------------
    for (int rb = rbA + warp; rb < rbB; rb += nwarp) {
      const int64_t rrow0 = g.rblk_row0[rb];
      const int64_t rrow1 = (rb + 1 < g.n_rblk) ? g.rblk_row0[rb + 1] : g.n_rows;
      const int nr = (int)(rrow1 - rrow0);
      const int c = g.rblk_comm[rb];
      double2 znew = make_double2(0.0, 0.0);
      if (lane < nr) {
        const int64_t i = rrow0 + lane;
        const double2 acc = accs[i - row0];
        const double2 zi = staged ? zs[i - w0] : ldg(a.z_in + i);
        const double2 R = (c >= 0) ? ldcg2(a.R_in + c) : make_double2(0.0, 0.0);
        const double kn = a.k_over_n;
        double k = ldg(a.omega + i) + kn * (R.y * zi.x - R.x * zi.y);
        k = k + kn * (acc.y * zi.x - acc.x * zi.y);
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
          znew = make_double2(cs, sn);
          a.z_out[i] = znew;
        }
      }
      if (MODE != 0 && c >= 0) {
        const double pr = warp_sum(znew.x), pim = warp_sum(znew.y);
        int last = 0;
        if (lane == 0) {
          a.part[rb] = make_double2(pr, pim);
          __threadfence();
          const int total = g.comm_rblk_off[c + 1] - g.comm_rblk_off[c];
          last = (atomicAdd(a.cnt + c, 1) + 1 == total);
        }
        last = __shfl_sync(FULL, last, 0);
        if (last) {  // this warp finished community c: reduce its partials (fixed order)
          __threadfence();
          const double2 Rn =
              reduce_comm(a.part, g.comm_rblk_off[c], g.comm_rblk_off[c + 1], lane);
          if (lane == 0) {
            a.R_out[c] = Rn;
            a.cnt[c] = 0;
          }
        }
      }
    }
    __syncthreads();  // zs / accs reused by the next segment
  }
}

// z = exp(i theta) per rblock and the rblock partials (prepare).
__global__ void __launch_bounds__(256) prepare_kernel(cdk_graph g, const double *theta,
                                                      double2 *z, double2 *part) {
  const int lane = threadIdx.x & 31;
  const int rb = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (rb >= g.n_rblk) return;
  const int64_t row0 = g.rblk_row0[rb];
  const int c = g.rblk_comm[rb];
  const int64_t cend = (c >= 0) ? g.comm_off[c + 1] : g.n_rows;
  const int nr = (int)min((int64_t)RB, cend - row0);
  double2 zz = make_double2(0.0, 0.0);
  if (lane < nr) {
    double sn, cs;
    sincos(theta[row0 + lane], &sn, &cs);
    zz = make_double2(cs, sn);
    z[row0 + lane] = zz;
  }
  const double pr = warp_sum(zz.x), pi = warp_sum(zz.y);
  if (lane == 0) part[rb] = make_double2(pr, pi);
}

__global__ void comm_reduce_kernel(cdk_graph g, const double2 *part, double2 *R, int32_t *cnt,
                                   cdk_run_status *st) {
  const int c = blockIdx.x;
  const int lane = threadIdx.x;
  if (c < g.n_comm) {
    const double2 Rc = reduce_comm(part, g.comm_rblk_off[c], g.comm_rblk_off[c + 1], lane);
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
  if (g->cta_threads != 256 && g->cta_threads != 512) {
    set_error("cdk_graph: cta_threads must be 256 or 512");
    return CDK_INPUT;
  }
  if (g->smem_nodes < 0 || g->seg_rows_cap <= 0) {
    set_error("cdk_graph: bad shared-memory capacities");
    return CDK_INPUT;
  }
  return CDK_OK;
}

static size_t stage_smem(const cdk_graph *g) {
  return ((size_t)g->smem_nodes + (size_t)g->seg_rows_cap) * sizeof(double2);
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
    const int wpb = 8;
    prepare_kernel<<<(g->n_rblk + wpb - 1) / wpb, 32 * wpb, 0, st>>>(*g, theta, w.z[0], w.part);
    CDK_CHECK_LAUNCH("prepare_kernel");
  }
  const int m = (int)g->n_comm;
  comm_reduce_kernel<<<m > 0 ? m : 1, 32, 0, st>>>(*g, w.part, w.R[0], w.cnt, w.status);
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
