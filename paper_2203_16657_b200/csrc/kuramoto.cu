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
constexpr int GL = 8;   // lanes per row

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
  w.z[0] = (double2 *)take(n * sizeof(double2));
  w.z[1] = (double2 *)take(n * sizeof(double2));
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

// MODE 0: out = f(theta) (single RHS).  MODE 1..4: RK4 stage.  MODE 5: Euler step.
template <int MODE>
__global__ void __launch_bounds__(512, 2) kuramoto_stage_kernel(const StageArgs a) {
  extern __shared__ __align__(128) double2 zs[];
  __shared__ int s_last;
  const cdk_graph &g = a.g;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  const int grp = lane >> 3, t = lane & 7;
  const int segA = g.cta_seg[blockIdx.x], segB = g.cta_seg[blockIdx.x + 1];

  for (int s = segA; s < segB; ++s) {
    const int rb0 = g.seg_rblk[s], rb1 = g.seg_rblk[s + 1];
    const int c = g.rblk_comm[rb0];
    int64_t c0 = 0, cend = g.n_rows;
    if (c >= 0) {
      c0 = g.comm_off[c];
      cend = g.comm_off[c + 1];
    }
    const bool staged = (c >= 0) && (cend - c0) <= (int64_t)g.smem_nodes;
    __syncthreads();  // previous segment done with zs
    if (staged) {
      const int lam = (int)(cend - c0);
      for (int i = tid; i < lam; i += blockDim.x) zs[i] = ldg(a.z_in + c0 + i);
    }
    __syncthreads();
    const double2 R = (c >= 0) ? ldcg2(a.R_in + c) : make_double2(0.0, 0.0);

    for (int rb = rb0 + warp; rb < rb1; rb += nwarp) {
      const int64_t row0 = g.rblk_row0[rb];
      const int nr = (int)min((int64_t)RB, cend - row0);
      const int64_t ip = (lane < nr) ? ldg(g.intra_ptr + row0 + lane) : 0;
      const int64_t ipe = ldg(g.intra_ptr + row0 + nr);
      const int64_t xp = (lane < nr) ? ldg(g.inter_ptr + row0 + lane) : 0;
      const int64_t xpe = ldg(g.inter_ptr + row0 + nr);

      double accr = 0.0, acci = 0.0;  // lane L ends with row L's sparse sum
      const int npass = (nr + 3) >> 2;
      for (int q = 0; q < npass; ++q) {
        const int r = 4 * q + grp;  // this group's row in the rblock
        const int rn = (r + 1) & 31;
        const int64_t s0 = __shfl_sync(FULL, ip, r & 31);
        const int64_t e0n = __shfl_sync(FULL, ip, rn);
        const int64_t x0 = __shfl_sync(FULL, xp, r & 31);
        const int64_t x1n = __shfl_sync(FULL, xp, rn);
        double sr = 0.0, si = 0.0;
        if (r < nr) {
          const int64_t e0 = (r + 1 < nr) ? e0n : ipe;
          const int64_t x1 = (r + 1 < nr) ? x1n : xpe;
          for (int64_t p = s0 + 8 * t; p < e0; p += 8 * GL) {
            const uint4 w = ldg(reinterpret_cast<const uint4 *>(g.intra_col + p));
            const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const uint32_t u = (wv[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu;
              if (u != CDK_INTRA_PAD) {
                const double2 z = staged ? zs[u] : ldg(a.z_in + c0 + u);
                sr -= z.x;
                si -= z.y;
              }
            }
          }
          for (int64_t p = x0 + t; p < x1; p += GL) {
            const int32_t j = ldg(g.inter_col + p);
            const double2 z = ldg(a.z_in + j);
            sr += z.x;
            si += z.y;
          }
        }
        sr = warp_sum(sr, GL);
        si = warp_sum(si, GL);
        const double vr = __shfl_sync(FULL, sr, (lane & 3) * GL);
        const double vi = __shfl_sync(FULL, si, (lane & 3) * GL);
        if ((lane >> 2) == q) {
          accr = vr;
          acci = vi;
        }
      }

      // epilogue: lane L owns row row0 + L
      double2 znew = make_double2(0.0, 0.0);
      if (lane < nr) {
        const int64_t i = row0 + lane;
        const double2 zi = staged ? zs[i - c0] : ldg(a.z_in + i);
        const double kn = a.k_over_n;
        double k = ldg(a.omega + i) + kn * (R.y * zi.x - R.x * zi.y);
        k = k + kn * (acci * zi.x - accr * zi.y);
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
      if (MODE != 0) {
        const double pr = warp_sum(znew.x), pi = warp_sum(znew.y);
        if (lane == 0) a.part[rb] = make_double2(pr, pi);
      }
    }

    // community completion: the last CTA reduces the partials into R_out[c]
    if (MODE != 0 && c >= 0) {
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        const int mine = rb1 - rb0;
        const int total = g.comm_rblk_off[c + 1] - g.comm_rblk_off[c];
        const int old = atomicAdd(a.cnt + c, mine);
        s_last = (old + mine == total);
      }
      __syncthreads();
      if (s_last && warp == 0) {
        __threadfence();
        const double2 Rn = reduce_comm(a.part, g.comm_rblk_off[c], g.comm_rblk_off[c + 1], lane);
        if (lane == 0) {
          a.R_out[c] = Rn;
          a.cnt[c] = 0;
        }
      }
    }
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
  return CDK_OK;
}

static size_t stage_smem(const cdk_graph *g) { return (size_t)g->smem_nodes * sizeof(double2); }

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
