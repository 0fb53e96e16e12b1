// Cucker–Smale flocking (2-D) with the per-community polynomial expansion of
// the coupling (BASELINE config 4), CIA form, fused into RK4.
// Math and notation: paper_2203_16657_b200/cs.py.  Per stage:
//   1. cs_moments_kernel: M^f_{ij} = sum_{l in c} x_l^i y_l^j f_l (f = 1, vx, vy),
//      x, y = scaled centred positions, i + j <= 16 (153 monomials), one CTA
//      per community, fixed node order;
//   2. cs_contract_kernel: H^f = T_c M^f (153 x 153 per community);
//   3. cs_rows_kernel: per row (8-lane group) the bivariate evaluation
//      G^f(x_m, y_m) = sum H^f_{pq} x_m^p y_m^q split over lanes by p, the
//      exact sparse correction sum_j s_mj eta(|s_j - s_m|^2)(v_j - v_m) over
//      the missing (-1) and inter (+1) CSRs, the domain guard |p_m| <= 1 and
//      the RK4 stage update of (s, v).
// The reference kernel for the sparse part is pairs_cs (_kernels.py:297-314).
#include "common.cuh"

namespace cdk {

constexpr int CS_D2 = 16;
constexpr int CS_NMON = (CS_D2 + 1) * (CS_D2 + 2) / 2;  // 153
constexpr int CS_NOUT = 3 * CS_NMON;                     // 459

__constant__ unsigned char c_mono_i[CS_NMON];
__constant__ unsigned char c_mono_j[CS_NMON];
__constant__ short c_mono_row[CS_D2 + 2];  // first packed index of each i (i-major)

struct CsArgs {
  int64_t n_rows;
  int32_t n_comm;
  int32_t n_rblk;
  const int64_t *comm_off;
  const int64_t *rblk_row0;
  const int32_t *rblk_comm;
  const int64_t *miss_ptr;
  const int32_t *miss_col;
  const int64_t *inter_ptr;
  const int32_t *inter_col;
  const double2 *mu;
  const double *inv_L;
  const double *chat;       // [M][9]
  const int32_t *t_ptr;     // [154] shared contraction pattern (CSR by output monomial)
  const int32_t *t_col;     // input monomial | k << 8
  const double *t_coef;
  double *M;                // [M][mom_split][3][153] partial moments (node chunks)
  int32_t mom_split;        // CTAs per community in the moments pass
  int32_t max_comm;         // largest community (nodes)
  double *H;                // [M][3][153]
  const double2 *s_in, *v_in;  // stage state
  double2 *s_out, *v_out;
  double2 *s0, *v0;         // step-start state (RK4 base; written at stage 4)
  double2 *ks, *kv;         // RK4 accumulators
  double2 *out;             // MODE 0: v'
  double2 *sacc;            // [n] exact sparse correction of this stage (cs_sparse_kernel)
  cdk_run_status *status;   // reserved = domain violations
  double K, sigma2, beta, inv_n, h;
  int64_t step_rel;
};

// x^(-1/2) for a positive normal x: the hardware seed (rsqrt.approx.f64, ~2^-22)
// and one cubic step y (1 + e/2 + 3 e^2/8), e = 1 - x y^2 (error ~ e^3).  No
// special-case branch or slow-path call, which the library sqrt/rsqrt carry
// per evaluation (the sparse correction is issue-bound: ~100 instructions per
// entry, a third of them this function).
__device__ __forceinline__ double rsqrt_normal(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-(x * y), y, 1.0);
  return fma(y, e * fma(0.375, e, 0.5), y);
}

__device__ __forceinline__ double eta_exact(double d2, double K, double sigma2, double beta) {
  const double x = sigma2 + d2;
  if (beta == 0.25) {  // x^(-1/4) = sqrt(r), r = x^(-1/2): within 2 ulp of pow(x, -0.25)
    if (x > 1e-280 && x < 1e280) {
      const double r = rsqrt_normal(x);
      return K * (r * rsqrt_normal(r));
    }
    return K * rsqrt(sqrt(x));
  }
  return K / pow(x, beta);
}

// moments of node chunk q of community c: CTA (c, q) sums nodes
// [b + q * CS_MOM_NODES, ...) in node order.  Thread t owns the outputs
// (f = 0..2, i, j0..j0+3): a "quad" of consecutive y powers for all three
// functions.  Per node it reads x^i, four y powers and the three f values (8
// shared loads) for 12 FMAs + 3 multiplies; one thread per (f, i, quad) read 6
// for 5, and the kernel sat at 89 % of the L1/shared pipe.  Twelve
// independent chains per thread.  The contraction adds the chunks' partials
// in q order.
#ifndef CDK_CS_MOM_NODES
#define CDK_CS_MOM_NODES 256
#endif
constexpr int CS_MOM_NODES = CDK_CS_MOM_NODES;
constexpr int CS_NQUAD = 45;  // sum_i ceil((17 - i) / 4)
constexpr int CS_MOM_THREADS = 64;
__constant__ unsigned char c_quad_i[CS_NQUAD];
__constant__ unsigned char c_quad_j[CS_NQUAD];
__global__ void __launch_bounds__(CS_MOM_THREADS) cs_moments_kernel(const CsArgs a) {
  __shared__ double px[128][CS_D2 + 1];
  __shared__ double py[128][CS_D2 + 4];  // 3 zero pads: a quad may run past j = 16 - i
  __shared__ double pf[128][3];
  const int c = blockIdx.x, q = blockIdx.y;
  const int64_t cb = a.comm_off[c], ce = a.comm_off[c + 1];
  const int64_t b = cb + (int64_t)q * CS_MOM_NODES;
  const int64_t e = min(ce, b + CS_MOM_NODES);
  const double2 mu = a.mu[c];
  const double il = a.inv_L[c];
  const int t = threadIdx.x;
  const bool act = t < CS_NQUAD;
  const int i = act ? c_quad_i[t] : 0, j0 = act ? c_quad_j[t] : 0;
  double acc[3][4];
#pragma unroll
  for (int f = 0; f < 3; ++f)
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[f][k] = 0.0;
  for (int64_t base = b; base < e; base += 128) {
    const int cnt = (int)min((int64_t)128, e - base);
    __syncthreads();
    for (int n = t; n < cnt; n += blockDim.x) {
      const double2 sv = a.s_in[base + n];
      const double2 v = a.v_in[base + n];
      const double x = (sv.x - mu.x) * il, y = (sv.y - mu.y) * il;
      double xp = 1.0, yp = 1.0;
      for (int k = 0; k <= CS_D2; ++k) {
        px[n][k] = xp;
        py[n][k] = yp;
        xp *= x;
        yp *= y;
      }
      py[n][CS_D2 + 1] = py[n][CS_D2 + 2] = py[n][CS_D2 + 3] = 0.0;
      pf[n][0] = 1.0;
      pf[n][1] = v.x;
      pf[n][2] = v.y;
    }
    __syncthreads();
    if (act) {
      for (int n = 0; n < cnt; ++n) {
        const double xi = px[n][i];
        const double y0 = py[n][j0], y1 = py[n][j0 + 1], y2 = py[n][j0 + 2], y3 = py[n][j0 + 3];
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          const double xf = xi * pf[n][f];
          acc[f][0] += xf * y0;
          acc[f][1] += xf * y1;
          acc[f][2] += xf * y2;
          acc[f][3] += xf * y3;
        }
      }
    }
  }
  if (act) {
    const int nj = CS_D2 - i + 1;  // valid j of this i: 0..16-i
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      double *Mq = a.M + ((int64_t)c * a.mom_split + q) * CS_NOUT + f * CS_NMON + c_mono_row[i];
      Mq[j0] = acc[f][0];
      if (j0 + 1 < nj) Mq[j0 + 1] = acc[f][1];
      if (j0 + 2 < nj) Mq[j0 + 2] = acc[f][2];
      if (j0 + 3 < nj) Mq[j0 + 3] = acc[f][3];
    }
  }
}

// H^f_c = T_c M^f_c with T_c[r][s] = chat_c[k(r,s)] t_coef[r,s]: the shared
// 1365-entry pattern and 9 coefficients per community replace the dense
// 153 x 153 tensor per community (19 MB per stage of mostly zeros on config 4)
__global__ void __launch_bounds__(512) cs_contract_kernel(const CsArgs a) {
  __shared__ double Ms[CS_NOUT];
  __shared__ double ch[9];
  const int c = blockIdx.x;
  const int o = threadIdx.x;
  if (o < CS_NOUT) {
    const double *Mc = a.M + (int64_t)c * a.mom_split * CS_NOUT;
    double m = 0.0;
    for (int q = 0; q < a.mom_split; ++q) m += Mc[(int64_t)q * CS_NOUT + o];  // chunk order
    Ms[o] = m;
  }
  if (o < 9) ch[o] = a.chat[(int64_t)c * 9 + o];
  __syncthreads();
  if (o >= CS_NOUT) return;
  const int f = o / CS_NMON, r = o % CS_NMON;
  const double *Mf = Ms + f * CS_NMON;
  double s = 0.0;
  for (int e = __ldg(a.t_ptr + r); e < __ldg(a.t_ptr + r + 1); ++e) {
    const int sc = __ldg(a.t_col + e);
    s += (ch[sc >> 8] * __ldg(a.t_coef + e)) * Mf[sc & 0xFF];
  }
  a.H[(int64_t)c * CS_NOUT + o] = s;
}

// sparse-correction entries per lane in flight, and resident cs_rows CTAs per
// SM (register cap 80): measured on config 4, batch 2 x 3 CTAs 0.556 ms per
// step, batch 4 x 3 0.564, batch 4 x 2 (114 registers) 0.624, batch 1 0.729
constexpr int CS_BATCH = 2;
constexpr int CS_MINB = 3;
#ifndef CDK_CS_LPR
#define CDK_CS_LPR 4  // lanes per row of cs_rows (1, 2, 4, 8); measured 4 (+ unroll 2) best
#endif
constexpr int CS_LPR = CDK_CS_LPR;

// sum over entries p = p0, p0 + CS_LPR, ... < p1 of eta(|s_j - s_m|^2)(v_j - v_m)
// added onto (ax, ay) in entry order
__device__ __forceinline__ void cs_sparse_sum(const CsArgs &a, const int32_t *__restrict__ col,
                                              int64_t p0, int64_t p1, double2 sm, double2 vm,
                                              double &ax, double &ay) {
  for (int64_t p = p0; p < p1; p += CS_BATCH * CS_LPR) {
    int jb[CS_BATCH];
#pragma unroll
    for (int b = 0; b < CS_BATCH; ++b) {
      const int64_t q = p + (int64_t)b * CS_LPR;
      jb[b] = q < p1 ? __ldg(col + q) : -1;
    }
    double2 sj[CS_BATCH], vj[CS_BATCH];
#pragma unroll
    for (int b = 0; b < CS_BATCH; ++b) {
      const int j = jb[b] >= 0 ? jb[b] : 0;
      sj[b] = __ldg(a.s_in + j);
      vj[b] = __ldg(a.v_in + j);
    }
#pragma unroll
    for (int b = 0; b < CS_BATCH; ++b) {
      if (jb[b] >= 0) {
        const double dx = sj[b].x - sm.x, dy = sj[b].y - sm.y;
        const double w = eta_exact(dx * dx + dy * dy, a.K, a.sigma2, a.beta);
        ax += w * (vj[b].x - vm.x);
        ay += w * (vj[b].y - vm.y);
      }
    }
  }
}

// Exact sparse correction of every row (CS_LPR lanes per row, CS_BATCH
// columns per lane loaded first, then all their (s_j, v_j) gathers; fixed
// per-lane order + xor butterfly): its own launch, so the gather loop runs at
// the occupancy its ~40 registers allow instead of the bivariate evaluation's
// 80 (the gathers are latency-bound: long_scoreboard 56 % when fused).
__global__ void __launch_bounds__(256, 4) cs_sparse_kernel(const CsArgs a) {
  const int lane = threadIdx.x & 31, t = lane & (CS_LPR - 1);
  const unsigned gmask = CS_LPR == 32 ? 0xFFFFFFFFu
                                      : (((1u << CS_LPR) - 1u) << (lane & ~(CS_LPR - 1)));
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / CS_LPR;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / CS_LPR; i < a.n_rows;
       i += ngroups) {
    const double2 sm = a.s_in[i], vm = a.v_in[i];
    double ax = 0.0, ay = 0.0;
    cs_sparse_sum(a, a.miss_col, a.miss_ptr[i] + t, a.miss_ptr[i + 1], sm, vm, ax, ay);
    ax = -ax;
    ay = -ay;
    cs_sparse_sum(a, a.inter_col, a.inter_ptr[i] + t, a.inter_ptr[i + 1], sm, vm, ax, ay);
#pragma unroll
    for (int o = CS_LPR / 2; o > 0; o >>= 1) {
      ax += __shfl_xor_sync(gmask, ax, o);
      ay += __shfl_xor_sync(gmask, ay, o);
    }
    if (t == 0) a.sacc[i] = make_double2(ax, ay);
  }
}

// The same sums with the community's state staged in shared memory: a CTA
// owns CS_WIN_RB consecutive rblocks, stages (s, v) of the first one's
// community (<= CS_WIN_CAP nodes, 32 bytes each) with coalesced loads, and
// the missing-edge gathers of that community's rows become LDS.128 pairs
// (~0.33 cycles per 16 bytes per SM with random bank conflicts) instead of two
// L1/L2 sector gathers per entry (~1 cycle each).  Inter entries, pool rows
// and an rblock of another community (a CTA straddling a boundary) keep the
// global path.  Same per-lane entry order, same butterfly: bitwise equal to
// cs_sparse_kernel.
constexpr int CS_WIN_RB = 4;      // rblocks (<= 128 rows) per CTA, CS_LPR lanes per row
constexpr int CS_WIN_CAP = 3072;  // nodes: 96 KB of shared memory
__device__ __forceinline__ int ld_col(const int32_t *p) {
  int v;
  asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void cs_sparse_sum_win(const CsArgs &a, const int32_t *__restrict__ col,
                                                  int64_t p0, int64_t p1, double2 sm, double2 vm,
                                                  const double2 *__restrict__ sS,
                                                  const double2 *__restrict__ sV, int cb,
                                                  double &ax, double &ay) {
  // the next batch's columns load while this batch's gathers and eta run: the
  // column load's L2 latency was the kernel's top stall (24 % of the warp
  // samples on its first use).  Volatile asm keeps the loads where they are
  // written (the compiler sinks a plain __ldg back to its use).
  // 32-bit entry counter relative to the lane's first entry (the kernel
  // issues ~60 % of its slots: index arithmetic counts)
  const int32_t *__restrict__ cp = col + p0;
  const int cnt = (int)(p1 - p0);
  int jn[CS_BATCH];
#pragma unroll
  for (int b = 0; b < CS_BATCH; ++b) jn[b] = b * CS_LPR < cnt ? ld_col(cp + b * CS_LPR) : -1;
  for (int e = 0; e < cnt; e += CS_BATCH * CS_LPR) {
    int jb[CS_BATCH];
#pragma unroll
    for (int b = 0; b < CS_BATCH; ++b) {
      jb[b] = jn[b];
      const int q = e + (CS_BATCH + b) * CS_LPR;
      jn[b] = q < cnt ? ld_col(cp + q) : -1;
    }
    double2 sj[CS_BATCH], vj[CS_BATCH];
#pragma unroll
    for (int b = 0; b < CS_BATCH; ++b) {
      const int j = jb[b] >= 0 ? jb[b] - cb : 0;
      sj[b] = sS[j];
      vj[b] = sV[j];
    }
#pragma unroll
    for (int b = 0; b < CS_BATCH; ++b) {
      // pads evaluate node 0 of the window and add nothing (no divergent branch)
      const double dx = sj[b].x - sm.x, dy = sj[b].y - sm.y;
      const double w = jb[b] >= 0 ? eta_exact(dx * dx + dy * dy, a.K, a.sigma2, a.beta) : 0.0;
      ax += w * (vj[b].x - vm.x);
      ay += w * (vj[b].y - vm.y);
    }
  }
}

__global__ void __launch_bounds__(32 * CS_WIN_RB * CS_LPR, 2) cs_sparse_win_kernel(const CsArgs a) {
  extern __shared__ __align__(16) unsigned char cs_win_raw[];
  const int lane = threadIdx.x & 31, t = lane & (CS_LPR - 1);
  const unsigned gmask = CS_LPR == 32 ? 0xFFFFFFFFu
                                      : (((1u << CS_LPR) - 1u) << (lane & ~(CS_LPR - 1)));
  const int rb0 = blockIdx.x * CS_WIN_RB;
  const int c0 = a.rblk_comm[rb0];
  int64_t cb = 0, ce = 0;
  if (c0 >= 0) {
    cb = a.comm_off[c0];
    ce = a.comm_off[c0 + 1];
  }
  const int nc = (int)(ce - cb);
  double2 *sS = reinterpret_cast<double2 *>(cs_win_raw);
  double2 *sV = sS + nc;
  for (int k = threadIdx.x; k < nc; k += blockDim.x) {
    sS[k] = a.s_in[cb + k];
    sV[k] = a.v_in[cb + k];
  }
  __syncthreads();
  const int g = threadIdx.x / CS_LPR;  // row slot of the CTA: rblock g / 32, row g % 32
  const int rb = rb0 + (g >> 5);
  if (rb >= a.n_rblk) return;
  const int64_t i = a.rblk_row0[rb] + (g & 31);
  if (i >= a.rblk_row0[rb + 1]) return;  // whole CS_LPR-lane groups leave together
  const double2 sm = a.s_in[i], vm = a.v_in[i];
  double ax = 0.0, ay = 0.0;
  if (i >= cb && i < ce) {
    cs_sparse_sum_win(a, a.miss_col, a.miss_ptr[i] + t, a.miss_ptr[i + 1], sm, vm, sS, sV, (int)cb,
                      ax, ay);
  } else {
    cs_sparse_sum(a, a.miss_col, a.miss_ptr[i] + t, a.miss_ptr[i + 1], sm, vm, ax, ay);
  }
  ax = -ax;
  ay = -ay;
  cs_sparse_sum(a, a.inter_col, a.inter_ptr[i] + t, a.inter_ptr[i + 1], sm, vm, ax, ay);
#pragma unroll
  for (int o = CS_LPR / 2; o > 0; o >>= 1) {
    ax += __shfl_xor_sync(gmask, ax, o);
    ay += __shfl_xor_sync(gmask, ay, o);
  }
  if (t == 0) a.sacc[i] = make_double2(ax, ay);
}

// MODE 0: out = v'(s_in, v_in).  MODE 1..4: RK4 stage.  CTA b owns rows
// [CS_ROWS_PER_CTA b, ...) (CS_RLPR lanes per row); the contraction outputs H of the
// communities those rows belong to are staged in shared memory first (every
// row reads all 459 values of its community's H).
#ifndef CDK_CS_RLPR
#define CDK_CS_RLPR 1  // lanes per row of cs_rows' bivariate evaluation
#endif
// With one lane per row every lane of a warp reads the same H entry of its
// community (a broadcast: one wavefront per LDS instead of one per distinct
// p residue), 459 LDS per 32 rows instead of per 8.
constexpr int CS_RLPR = CDK_CS_RLPR;
constexpr int CS_ROWS_PER_CTA = 256 / CS_RLPR;
constexpr int CS_H_SLOTS = 4;  // communities staged per CTA (more: read from global)

// G^f(x, y) = sum_pq H^f_pq x^p y^q for f = 0, x, y: lane t of a row's
// CS_RLPR lanes takes p = t, t + CS_RLPR, ...; Horner in y, then one x^p term
template <typename HPtr>
__device__ __forceinline__ void cs_bivariate(HPtr Hc, double x, double y, int t, double &g0,
                                             double &gx, double &gy) {
  double xp = 1.0;
  for (int k = 0; k < t; ++k) xp *= x;
  double x8 = 1.0;  // x^CS_RLPR
  for (int k = 0; k < CS_RLPR; ++k) x8 *= x;
  for (int p = t; p <= CS_D2; p += CS_RLPR) {
    const int r0 = c_mono_row[p], nq = CS_D2 - p;
    double h0 = Hc[r0 + nq], hx = Hc[CS_NMON + r0 + nq], hy = Hc[2 * CS_NMON + r0 + nq];
    for (int q = nq - 1; q >= 0; --q) {
      h0 = fma(h0, y, Hc[r0 + q]);
      hx = fma(hx, y, Hc[CS_NMON + r0 + q]);
      hy = fma(hy, y, Hc[2 * CS_NMON + r0 + q]);
    }
    g0 = fma(xp, h0, g0);
    gx = fma(xp, hx, gx);
    gy = fma(xp, hy, gy);
    xp *= x8;
  }
}
template <int MODE>
__global__ void __launch_bounds__(256, CS_MINB) cs_rows_kernel(const CsArgs a) {
  __shared__ double Hs[CS_H_SLOTS][CS_NOUT];
  __shared__ int cfirst;
  const int lane = threadIdx.x & 31, t = lane & (CS_RLPR - 1);
  const unsigned gmask = CS_RLPR == 32 ? 0xFFFFFFFFu
                                      : (((1u << CS_RLPR) - 1u) << (lane & ~(CS_RLPR - 1)));
  const int64_t r0 = (int64_t)blockIdx.x * CS_ROWS_PER_CTA;
  const int64_t n_in = a.n_comm > 0 ? a.comm_off[a.n_comm] : 0;
  auto comm_of = [&](int64_t i) {  // binary search over comm_off
    int lo = 0, hi = a.n_comm;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (a.comm_off[mid] <= i) lo = mid; else hi = mid;
    }
    return lo;
  };
  if (threadIdx.x == 0) cfirst = (r0 < n_in) ? comm_of(r0) : -1;
  __syncthreads();
  const int c0 = cfirst;
  if (c0 >= 0) {
    for (int k = threadIdx.x; k < CS_H_SLOTS * CS_NOUT; k += blockDim.x) {
      const int cc = c0 + k / CS_NOUT;
      if (cc < a.n_comm) Hs[k / CS_NOUT][k % CS_NOUT] = __ldcg(a.H + (int64_t)cc * CS_NOUT + k % CS_NOUT);
    }
  }
  __syncthreads();
  const int64_t i = r0 + threadIdx.x / CS_RLPR;
  if (i < a.n_rows) {
    const int c = (i < n_in) ? comm_of(i) : -1;
    const double2 sm = a.s_in[i], vm = a.v_in[i];
    double g0 = 0.0, gx = 0.0, gy = 0.0;
    bool out_of_domain = false;
    if (c >= 0) {
      const double2 mu = a.mu[c];
      const double il = a.inv_L[c];
      const double x = (sm.x - mu.x) * il, y = (sm.y - mu.y) * il;
      out_of_domain = (x * x + y * y) > 1.0 + 1e-12;
      // two instantiations so the staged case reads with LDS (a pointer that
      // may be shared or global compiles to generic loads)
      if (c - c0 < CS_H_SLOTS) {
        cs_bivariate(Hs[c - c0], x, y, t, g0, gx, gy);
      } else {
        cs_bivariate(a.H + (int64_t)c * CS_NOUT, x, y, t, g0, gx, gy);
      }
    }
#pragma unroll
    for (int o = CS_RLPR / 2; o > 0; o >>= 1) {
      g0 += __shfl_xor_sync(gmask, g0, o);
      gx += __shfl_xor_sync(gmask, gx, o);
      gy += __shfl_xor_sync(gmask, gy, o);
    }
    if (t == 0) {
      const double2 sa = __ldcg(a.sacc + i);  // the row's exact sparse correction
      const double ax = sa.x, ay = sa.y;
      if (out_of_domain) atomicAdd(reinterpret_cast<unsigned long long *>(&a.status->reserved), 1ull);
      const double accx = (gx - vm.x * g0) + ax, accy = (gy - vm.y * g0) + ay;
      const double2 acc = make_double2(accx * a.inv_n, accy * a.inv_n);
      if (MODE == 0) {
        a.out[i] = acc;
      } else {
        const double2 s0 = a.s0[i], v0 = a.v0[i];
        double2 ks, kv;
        if (MODE == 1) {
          ks = vm;
          kv = acc;
        } else {
          const double2 ps = a.ks[i], pv = a.kv[i];
          const double w = (MODE == 4) ? 1.0 : 2.0;
          ks = make_double2(add_rn(ps.x, mul_rn(w, vm.x)), add_rn(ps.y, mul_rn(w, vm.y)));
          kv = make_double2(add_rn(pv.x, mul_rn(w, acc.x)), add_rn(pv.y, mul_rn(w, acc.y)));
        }
        if (MODE < 4) {
          a.ks[i] = ks;
          a.kv[i] = kv;
          a.s_out[i] = make_double2(add_rn(s0.x, mul_rn(a.h, vm.x)), add_rn(s0.y, mul_rn(a.h, vm.y)));
          a.v_out[i] = make_double2(add_rn(v0.x, mul_rn(a.h, acc.x)), add_rn(v0.y, mul_rn(a.h, acc.y)));
        } else {
          const double2 sn = make_double2(add_rn(s0.x, mul_rn(a.h, ks.x)), add_rn(s0.y, mul_rn(a.h, ks.y)));
          const double2 vn = make_double2(add_rn(v0.x, mul_rn(a.h, kv.x)), add_rn(v0.y, mul_rn(a.h, kv.y)));
          a.s_out[i] = sn;
          a.v_out[i] = vn;
          if (!isfinite(sn.x) || !isfinite(sn.y) || !isfinite(vn.x) || !isfinite(vn.y)) {
            atomicAdd(reinterpret_cast<unsigned long long *>(&a.status->nonfinite), 1ull);
            atomicMin(reinterpret_cast<long long *>(&a.status->first_bad_step),
                      (long long)(a.status->steps_done + a.step_rel + 1));
          }
        }
      }
    }
  }
}

__global__ void cs_reset_status_kernel(cdk_run_status *st) {
  st->nonfinite = 0;
  st->first_bad_step = INT64_MAX;
  st->steps_done = 0;
  st->reserved = 0;
}
__global__ void cs_advance_kernel(cdk_run_status *st, int64_t n) { st->steps_done += n; }

// CTAs per community in the moments pass (g->max_comm: the largest community)
static int cs_mom_split(const cdk_cs_graph *g) {
  const int64_t mx = g->max_comm > 0 ? g->max_comm : 1;
  return (int)((mx + CS_MOM_NODES - 1) / CS_MOM_NODES);
}

struct CsWs {
  double2 *s[2], *v[2], *ks, *kv, *sacc;
  double *M, *H;
  cdk_run_status *status;
};

static CsWs cs_carve(const cdk_cs_graph *g, void *base, size_t *total) {
  CsWs w{};
  size_t off = 0;
  char *b = reinterpret_cast<char *>(base);
  auto take = [&](size_t bytes) {
    void *p = b ? b + off : nullptr;
    off = (off + bytes + 255) / 256 * 256;
    return p;
  };
  const size_t n = (size_t)g->n_rows + 1, m = (size_t)g->n_comm + 1;
  for (int k = 0; k < 2; ++k) {
    w.s[k] = (double2 *)take(n * 16);
    w.v[k] = (double2 *)take(n * 16);
  }
  w.ks = (double2 *)take(n * 16);
  w.sacc = (double2 *)take(n * 16);
  w.kv = (double2 *)take(n * 16);
  w.M = (double *)take(m * (size_t)cs_mom_split(g) * CS_NOUT * 8);
  w.H = (double *)take(m * CS_NOUT * 8);
  w.status = (cdk_run_status *)take(sizeof(cdk_run_status));
  if (total) *total = off;
  return w;
}

static bool g_cs_tables = false;
static int cs_tables() {
  if (g_cs_tables) return CDK_OK;
  unsigned char mi[CS_NMON], mj[CS_NMON];
  short row[CS_D2 + 2];
  int k = 0;
  for (int i = 0; i <= CS_D2; ++i) {
    row[i] = (short)k;
    for (int j = 0; j <= CS_D2 - i; ++j, ++k) {
      mi[k] = (unsigned char)i;
      mj[k] = (unsigned char)j;
    }
  }
  row[CS_D2 + 1] = (short)k;
  unsigned char qi[CS_NQUAD], qj[CS_NQUAD];
  int nq = 0;
  for (int i = 0; i <= CS_D2; ++i)
    for (int j = 0; j <= CS_D2 - i; j += 4) {
      if (nq < CS_NQUAD) {
        qi[nq] = (unsigned char)i;
        qj[nq] = (unsigned char)j;
      }
      ++nq;
    }
  if (nq != CS_NQUAD) {
    set_error("cs quad table size");
    return CDK_INPUT;
  }
  cudaError_t e = cudaMemcpyToSymbol(c_mono_i, mi, sizeof(mi));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_quad_i, qi, sizeof(qi));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_quad_j, qj, sizeof(qj));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_mono_j, mj, sizeof(mj));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_mono_row, row, sizeof(row));
  if (e != cudaSuccess) return cuda_status(e, "cs constant tables");
  g_cs_tables = true;
  return CDK_OK;
}

static CsArgs cs_args(const cdk_cs_graph *g, const CsWs &w, double K, double sigma2, double beta,
                      double inv_n) {
  CsArgs a{};
  a.n_rows = g->n_rows;
  a.n_comm = (int32_t)g->n_comm;
  a.n_rblk = g->n_rblk;
  a.comm_off = g->comm_off;
  a.rblk_row0 = g->rblk_row0;
  a.rblk_comm = g->rblk_comm;
  a.miss_ptr = g->miss_ptr;
  a.miss_col = g->miss_col;
  a.inter_ptr = g->inter_ptr;
  a.inter_col = g->inter_col;
  a.mu = reinterpret_cast<const double2 *>(g->mu);
  a.inv_L = g->inv_L;
  a.chat = g->chat;
  a.t_ptr = g->t_ptr;
  a.t_col = g->t_col;
  a.t_coef = g->t_coef;
  a.M = w.M;
  a.sacc = w.sacc;
  a.mom_split = cs_mom_split(g);
  a.max_comm = g->max_comm;
  a.H = w.H;
  a.ks = w.ks;
  a.kv = w.kv;
  a.status = w.status;
  a.K = K;
  a.sigma2 = sigma2;
  a.beta = beta;
  a.inv_n = inv_n;
  return a;
}

static unsigned cs_row_grid(int64_t n) {
  const int64_t groups_per_block = 256 / CS_LPR;
  int64_t g = (n + groups_per_block - 1) / groups_per_block;
  if (g > 148 * 16) g = 148 * 16;
  return (unsigned)(g > 0 ? g : 1);
}

// The community part of a stage (moments -> contraction, ~400 small CTAs at 3
// warps per scheduler) and the exact sparse correction (every SM, gather
// bound) are independent until cs_rows: the first runs on an auxiliary
// stream forked from and joined back into the caller's with events, so the
// two overlap instead of queueing (config 4: 47 us of the 138 us stage).
template <int MODE>
static int cs_stage(CsArgs a, cudaStream_t st) {
  AuxFork *fk = a.n_comm > 0 ? aux_fork(st) : nullptr;
  cudaStream_t sc = fk ? fk->aux : st;  // stream of the community part
  if (a.n_comm > 0) {
    cs_moments_kernel<<<dim3(a.n_comm, a.mom_split), CS_MOM_THREADS, 0, sc>>>(a);
    CDK_CHECK_LAUNCH("cs_moments_kernel");
    cs_contract_kernel<<<a.n_comm, 512, 0, sc>>>(a);
    CDK_CHECK_LAUNCH("cs_contract_kernel");
  }
  if (a.max_comm > 0 && a.max_comm <= CS_WIN_CAP && a.n_rblk > 0) {
    static bool optin = false;
    const size_t smem = (size_t)a.max_comm * 32;
    if (!optin) {
      cudaError_t e = cudaFuncSetAttribute(cs_sparse_win_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           CS_WIN_CAP * 32);
      if (e != cudaSuccess) return cuda_status(e, "cs_sparse_win_kernel shared memory");
      optin = true;
    }
    cs_sparse_win_kernel<<<(unsigned)((a.n_rblk + CS_WIN_RB - 1) / CS_WIN_RB),
                           32 * CS_WIN_RB * CS_LPR, smem, st>>>(a);
    CDK_CHECK_LAUNCH("cs_sparse_win_kernel");
  } else {
    cs_sparse_kernel<<<cs_row_grid(a.n_rows), 256, 0, st>>>(a);
    CDK_CHECK_LAUNCH("cs_sparse_kernel");
  }
  if (fk && aux_join(fk, st) != CDK_OK) return CDK_CUDA;  // cs_rows reads H
  cs_rows_kernel<MODE><<<(unsigned)((a.n_rows + CS_ROWS_PER_CTA - 1) / CS_ROWS_PER_CTA), 256, 0,
                         st>>>(a);
  CDK_CHECK_LAUNCH("cs_rows_kernel");
  return CDK_OK;
}

static int cs_check(const cdk_cs_graph *g) {
  if (!g || g->n_rows < 0 || g->n_comm < 0) {
    set_error("cdk_cs_graph: invalid sizes");
    return CDK_INPUT;
  }
  return cs_tables();
}

}  // namespace cdk

using namespace cdk;

extern "C" size_t cdk_cs_workspace_bytes(const cdk_cs_graph *g) {
  size_t total = 0;
  cs_carve(g, nullptr, &total);
  return total;
}

extern "C" int cdk_cs_prepare(const cdk_cs_graph *g, void *workspace, void *stream) {
  int rc = cs_check(g);
  if (rc) return rc;
  CsWs w = cs_carve(g, workspace, nullptr);
  cs_reset_status_kernel<<<1, 1, 0, as_stream(stream)>>>(w.status);
  CDK_CHECK_LAUNCH("cs_reset_status_kernel");
  return CDK_OK;
}

extern "C" int cdk_cs_rhs(const cdk_cs_graph *g, const double *pos, const double *vel, double K,
                          double sigma2, double beta, double inv_n, double *out, void *workspace,
                          void *stream) {
  int rc = cs_check(g);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  CsWs w = cs_carve(g, workspace, nullptr);
  CsArgs a = cs_args(g, w, K, sigma2, beta, inv_n);
  a.s_in = reinterpret_cast<const double2 *>(pos);
  a.v_in = reinterpret_cast<const double2 *>(vel);
  a.out = reinterpret_cast<double2 *>(out);
  return cs_stage<0>(a, st);
}

extern "C" int cdk_cs_rk4(const cdk_cs_graph *g, double *pos, double *vel, double K,
                          double sigma2, double beta, double inv_n, double dt, int64_t n_steps,
                          void *workspace, void *stream) {
  int rc = cs_check(g);
  if (rc) return rc;
  if (n_steps < 0) return set_error("n_steps < 0"), CDK_INPUT;
  cudaStream_t st = as_stream(stream);
  CsWs w = cs_carve(g, workspace, nullptr);
  CsArgs a = cs_args(g, w, K, sigma2, beta, inv_n);
  double2 *s0 = reinterpret_cast<double2 *>(pos), *v0 = reinterpret_cast<double2 *>(vel);
  a.s0 = s0;
  a.v0 = v0;
  for (int64_t s = 0; s < n_steps; ++s) {
    a.step_rel = s;
    a.s_in = s0; a.v_in = v0; a.s_out = w.s[0]; a.v_out = w.v[0]; a.h = dt / 2.0;
    if ((rc = cs_stage<1>(a, st))) return rc;
    a.s_in = w.s[0]; a.v_in = w.v[0]; a.s_out = w.s[1]; a.v_out = w.v[1]; a.h = dt / 2.0;
    if ((rc = cs_stage<2>(a, st))) return rc;
    a.s_in = w.s[1]; a.v_in = w.v[1]; a.s_out = w.s[0]; a.v_out = w.v[0]; a.h = dt;
    if ((rc = cs_stage<3>(a, st))) return rc;
    a.s_in = w.s[0]; a.v_in = w.v[0]; a.s_out = s0; a.v_out = v0; a.h = dt / 6.0;
    if ((rc = cs_stage<4>(a, st))) return rc;
  }
  if (n_steps > 0) {
    cs_advance_kernel<<<1, 1, 0, st>>>(w.status, n_steps);
    CDK_CHECK_LAUNCH("cs_advance_kernel");
  }
  return CDK_OK;
}

extern "C" int cdk_cs_status(const cdk_cs_graph *g, const void *workspace, cdk_run_status *out,
                             void *stream) {
  int rc = cs_check(g);
  if (rc) return rc;
  CsWs w = cs_carve(g, const_cast<void *>(workspace), nullptr);
  cudaStream_t st = as_stream(stream);
  cudaError_t e = cudaMemcpyAsync(out, w.status, sizeof(cdk_run_status), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return cuda_status(e, "cdk_cs_status");
}
