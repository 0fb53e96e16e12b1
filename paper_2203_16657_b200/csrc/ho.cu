// Higher-order (triadic) Kuramoto on the 3-cliques of a community graph
// (BASELINE config 3), CIA form, fused into RK4.
//
//   theta'_i = omega_i + K1/N Im(A_i z conj z_i)
//                      + K2/N^2 Im(S_i conj z_i^2),
//   S_i = sum over ordered (j,k) with {i,j,k} a triangle of z_j z_k.
//
// For i in community c the in-community part of S_i is expanded over the
// missing-edge graph m (proper, no self loops, re-derived in
// oracle/ho.py):
//   S_in_i = Zi^2 - Z2i - 2 Y_i Zi + V_i - W_c + Y_i^2 + 2 U_i - T_i
//   Zi = Z_c - z_i, Z2i = Z2_c - z_i^2, Y_i = sum_j m_ij z_j, V_i = sum_j m_ij z_j^2,
//   W_c = sum_{j in c} z_j Y_j, U_i = sum_j m_ij z_j Y_j,
//   T_i = 2 sum over missing-graph triangles {i,j,k} of z_j z_k;
// triangles spanning communities (or the NONE pool) are listed explicitly.
// Per RHS (see the kernel comment below): row sums Y, V, X, T and P = z Y;
// canonical rblock partials of P; U; community sums and the epilogue.  All
// reductions fixed-order (bitwise deterministic).
#include <climits>

#include "common.cuh"

namespace cdk {

struct HoArgs {
  // graph (device)
  int64_t n_rows;
  int32_t n_rblk;
  int32_t n_comm;
  const int64_t *rblk_row0;      // [n_rblk+1]
  const int32_t *rblk_comm;      // [n_rblk]
  const int32_t *comm_rblk_off;  // [n_comm+1]
  const int64_t *miss_ptr;       // [n+1]
  const int32_t *miss_col;       // global columns (proper missing intra edges)
  const int64_t *inter_ptr;      // [n+1]
  const int32_t *inter_col;
  const int64_t *tri_ptr;        // [n+1] triangle pairs per row
  const int2 *tri_jk;            // (j,k); j < 0 marks an inter triangle (j = -j-1)
  double2 *T, *U;                // [n] triangle and U sums of this stage
  // state
  const double2 *z_in;
  double2 *z_out;
  double2 *Y, *V, *X, *P;        // per row (pass 1 -> pass 2)
  const double2 *pz_in, *pz2_in; // rblock partials of z, z^2 (previous stage)
  double2 *pz_out, *pz2_out;
  double2 *pP;                   // rblock partials of P (this stage)
  double *theta;
  const double *omega;
  double *ksum;
  double *out;
  cdk_run_status *status;
  double k1n, k2n2;              // K1/N, K2/N^2
  double h;
  int64_t step_rel;
};

__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// canonical rblock partial of v (lane = row within the rblock; absent rows 0)
__device__ __forceinline__ double2 rblock_partial(double2 v) {
  const double r8 = __shfl_down_sync(FULL, v.x, 8), i8 = __shfl_down_sync(FULL, v.y, 8);
  const double r16 = __shfl_down_sync(FULL, v.x, 16), i16 = __shfl_down_sync(FULL, v.y, 16);
  const double r24 = __shfl_down_sync(FULL, v.x, 24), i24 = __shfl_down_sync(FULL, v.y, 24);
  double pr = ((v.x + r8) + r16) + r24, pim = ((v.y + i8) + i16) + i24;
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    pr += __shfl_xor_sync(FULL, pr, o);
    pim += __shfl_xor_sync(FULL, pim, o);
  }
  return make_double2(pr, pim);
}

// canonical community sum (8-lane form; call with all 32 lanes, lanes >= 8 idle)
__device__ __forceinline__ double2 comm_sum(const double2 *part, int b0, int b1, int lane) {
  double sr = 0.0, si = 0.0;
  if (lane < 8) {
    for (int b = b0 + lane; b < b1; b += 8) {
      const double2 v = __ldcg(part + b);
      sr += v.x;
      si += v.y;
    }
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    sr += __shfl_xor_sync(FULL, sr, o);
    si += __shfl_xor_sync(FULL, si, o);
  }
  return make_double2(__shfl_sync(FULL, sr, 0), __shfl_sync(FULL, si, 0));
}

__device__ __forceinline__ void group_reduce(double2 &v, unsigned gmask) {
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(gmask, v.x, o);
    v.y += __shfl_xor_sync(gmask, v.y, o);
  }
}

// Per stage: every sum over a row's lists runs in 8-lane groups over the
// row's CSR runs (coalesced index reads, HO_BATCH entries in flight per
// lane, fixed per-lane order + xor butterfly) on a grid of all rows (full
// occupancy: rows hold ~50 missing edges and ~125 triangle pairs on config 3
// with a wide spread, and the lane-per-row passes of round 1 ran ~10 warps
// per SM, latency-bound); only what needs a whole rblock — the canonical
// partials and the epilogue — runs warp per rblock, lane = row.
//   ho_rowsum: Y, V (missing), X (inter), T (triangle pairs), P = z Y
//   ho_ppart:  canonical rblock partials of P
//   ho_usum:   U = sum over missing edges of P_j
//   ho_epi:    community sums Z, Z2, W from canonical partials + RK4 epilogue
// entries per lane in flight and resident ho_rowsum CTAs per SM (64-register
// cap): measured on config 3, batch 2 x 4 CTAs 0.252 ms per step, batch 4 x 4
// 0.255, batch 4 or 8 x 2 CTAs 0.284
constexpr int HO_BATCH = 2;
constexpr int HO_ROWSUM_MINB = 4;

__device__ __forceinline__ void group_reduce8(double2 &v, unsigned gmask) {
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(gmask, v.x, o);
    v.y += __shfl_xor_sync(gmask, v.y, o);
  }
}

__global__ void __launch_bounds__(256, HO_ROWSUM_MINB) ho_rowsum_kernel(const HoArgs a) {
  const int t = threadIdx.x & 7;
  const unsigned gmask = 0xFFu << (threadIdx.x & 24);
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  if (i >= a.n_rows) return;  // whole 8-lane groups exit together
  double2 y = make_double2(0.0, 0.0), v = y, x = y, tr = y;
  const int64_t m0 = a.miss_ptr[i], m1 = a.miss_ptr[i + 1];
  for (int64_t p = m0 + t; p < m1; p += 8 * HO_BATCH) {
    int jb[HO_BATCH];
#pragma unroll
    for (int b = 0; b < HO_BATCH; ++b) jb[b] = (p + 8 * b < m1) ? __ldg(a.miss_col + p + 8 * b) : -1;
    double2 zb[HO_BATCH];
#pragma unroll
    for (int b = 0; b < HO_BATCH; ++b) zb[b] = __ldg(a.z_in + (jb[b] >= 0 ? jb[b] : 0));
#pragma unroll
    for (int b = 0; b < HO_BATCH; ++b)
      if (jb[b] >= 0) {
        y = cadd(y, zb[b]);
        v = cadd(v, cmul(zb[b], zb[b]));
      }
  }
  const int64_t x0 = a.inter_ptr[i], x1 = a.inter_ptr[i + 1];
  for (int64_t p = x0 + t; p < x1; p += 8) x = cadd(x, __ldg(a.z_in + a.inter_col[p]));
  const int64_t q0 = a.tri_ptr[i], q1 = a.tri_ptr[i + 1];
  for (int64_t p = q0 + t; p < q1; p += 8 * HO_BATCH) {
    int2 jk[HO_BATCH];
#pragma unroll
    for (int b = 0; b < HO_BATCH; ++b)
      jk[b] = (p + 8 * b < q1) ? __ldg(a.tri_jk + p + 8 * b) : make_int2(INT_MIN, 0);
    double2 zj[HO_BATCH], zk[HO_BATCH];
#pragma unroll
    for (int b = 0; b < HO_BATCH; ++b) {
      const bool pad = jk[b].x == INT_MIN;
      const int j = pad ? 0 : (jk[b].x < 0 ? -jk[b].x - 1 : jk[b].x);
      zj[b] = __ldg(a.z_in + j);
      zk[b] = __ldg(a.z_in + (pad ? 0 : jk[b].y));
    }
#pragma unroll
    for (int b = 0; b < HO_BATCH; ++b)
      if (jk[b].x != INT_MIN) {
        const double2 w = cmul(zj[b], zk[b]);
        const double sg = jk[b].x < 0 ? 2.0 : -2.0;  // spanning +2, missing -2
        tr.x += sg * w.x;
        tr.y += sg * w.y;
      }
  }
  group_reduce8(y, gmask);
  group_reduce8(v, gmask);
  group_reduce8(x, gmask);
  group_reduce8(tr, gmask);
  if (t == 0) {
    a.Y[i] = y;
    a.V[i] = v;
    a.X[i] = x;
    a.T[i] = tr;
    a.P[i] = cmul(__ldg(a.z_in + i), y);
  }
}

__global__ void __launch_bounds__(256) ho_ppart_kernel(const HoArgs a) {
  const int lane = threadIdx.x & 31;
  const int rb = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (rb >= a.n_rblk) return;
  const int64_t row0 = a.rblk_row0[rb];
  const int nr = (int)(a.rblk_row0[rb + 1] - row0);
  const double2 pv = lane < nr ? __ldcg(a.P + row0 + lane) : make_double2(0.0, 0.0);
  const double2 part = rblock_partial(pv);
  if (lane == 0) a.pP[rb] = part;
}

__global__ void __launch_bounds__(256) ho_usum_kernel(const HoArgs a) {
  const int t = threadIdx.x & 7;
  const unsigned gmask = 0xFFu << (threadIdx.x & 24);
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  if (i >= a.n_rows) return;
  double2 u = make_double2(0.0, 0.0);
  const int64_t m0 = a.miss_ptr[i], m1 = a.miss_ptr[i + 1];
  for (int64_t p = m0 + t; p < m1; p += 8 * HO_BATCH) {
    int jb[HO_BATCH];
#pragma unroll
    for (int b = 0; b < HO_BATCH; ++b) jb[b] = (p + 8 * b < m1) ? __ldg(a.miss_col + p + 8 * b) : -1;
    double2 pb[HO_BATCH];
#pragma unroll
    for (int b = 0; b < HO_BATCH; ++b) pb[b] = __ldcg(a.P + (jb[b] >= 0 ? jb[b] : 0));
#pragma unroll
    for (int b = 0; b < HO_BATCH; ++b)
      if (jb[b] >= 0) u = cadd(u, pb[b]);
  }
  group_reduce8(u, gmask);
  if (t == 0) a.U[i] = u;
}

// community sums from canonical partials + the RK4 epilogue (lane = row)
template <int MODE>
__global__ void __launch_bounds__(256) ho_epi_kernel(const HoArgs a) {
  const int lane = threadIdx.x & 31;
  const int rb = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (rb >= a.n_rblk) return;
  {
    const int64_t row0 = a.rblk_row0[rb];
    const int nr = (int)(a.rblk_row0[rb + 1] - row0);
    const int c = a.rblk_comm[rb];
    double2 Zc = make_double2(0.0, 0.0), Z2c = Zc, Wc = Zc;
    if (c >= 0) {
      const int b0 = a.comm_rblk_off[c], b1 = a.comm_rblk_off[c + 1];
      Zc = comm_sum(a.pz_in, b0, b1, lane);
      Z2c = comm_sum(a.pz2_in, b0, b1, lane);
      Wc = comm_sum(a.pP, b0, b1, lane);
    }
    const double2 myU = lane < nr ? __ldcg(a.U + row0 + lane) : make_double2(0.0, 0.0);
    const double2 myT = lane < nr ? __ldcg(a.T + row0 + lane) : make_double2(0.0, 0.0);
    // epilogue: lane = row
    double2 zn = make_double2(0.0, 0.0), zn2 = zn;
    if (lane < nr) {
      const int64_t i = row0 + lane;
      const double2 zi = __ldg(a.z_in + i);
      const double2 Y = __ldcg(a.Y + i), V = __ldcg(a.V + i), X = __ldcg(a.X + i);
      double2 S = myT;
      double2 pair = make_double2(X.x - Y.x, X.y - Y.y);
      if (c >= 0) {
        pair = cadd(pair, Zc);
        const double2 Zi = make_double2(Zc.x - zi.x, Zc.y - zi.y);
        const double2 zi2 = cmul(zi, zi);
        const double2 Z2i = make_double2(Z2c.x - zi2.x, Z2c.y - zi2.y);
        const double2 ZiZi = cmul(Zi, Zi), YZ = cmul(Y, Zi), YY = cmul(Y, Y);
        S.x += ZiZi.x - Z2i.x - 2.0 * YZ.x + V.x - Wc.x + YY.x + 2.0 * myU.x;
        S.y += ZiZi.y - Z2i.y - 2.0 * YZ.y + V.y - Wc.y + YY.y + 2.0 * myU.y;
      }
      // Im(pair conj z) and Im(S conj z^2)
      const double2 zc2 = make_double2(zi.x * zi.x - zi.y * zi.y, -2.0 * zi.x * zi.y);
      double k = a.omega[i] + a.k1n * (pair.y * zi.x - pair.x * zi.y);
      k = k + a.k2n2 * (S.x * zc2.y + S.y * zc2.x);
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
        } else {
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
        zn = make_double2(cs, sn);
        zn2 = cmul(zn, zn);
        a.z_out[i] = zn;
      }
    }
    if (MODE != 0) {
      const double2 p1 = rblock_partial(zn), p2 = rblock_partial(zn2);
      if (lane == 0) {
        a.pz_out[rb] = p1;
        a.pz2_out[rb] = p2;
      }
    }
  }
}

// z = exp(i theta), rblock partials of z and z^2
__global__ void __launch_bounds__(256) ho_prepare_kernel(const HoArgs a, const double *theta,
                                                         double2 *z, double2 *pz, double2 *pz2) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int rb = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; rb < a.n_rblk; rb += warps) {
    const int64_t row0 = a.rblk_row0[rb];
    const int nr = (int)(a.rblk_row0[rb + 1] - row0);
    double2 zz = make_double2(0.0, 0.0), z2 = zz;
    if (lane < nr) {
      double sn, cs;
      sincos(theta[row0 + lane], &sn, &cs);
      zz = make_double2(cs, sn);
      z2 = cmul(zz, zz);
      z[row0 + lane] = zz;
    }
    const double2 p1 = rblock_partial(zz), p2 = rblock_partial(z2);
    if (lane == 0) {
      pz[rb] = p1;
      pz2[rb] = p2;
    }
  }
}

struct HoWs {
  double2 *z[2], *Y, *V, *X, *P, *T, *U, *pz[2], *pz2[2], *pP;
  double *ksum;
  cdk_run_status *status;
};

static HoWs ho_carve(int64_t n, int32_t n_rblk, void *base, size_t *total) {
  HoWs w{};
  size_t off = 0;
  char *b = reinterpret_cast<char *>(base);
  auto take = [&](size_t bytes) {
    void *p = b ? b + off : nullptr;
    off = (off + bytes + 255) / 256 * 256;
    return p;
  };
  const size_t nz = (size_t)n + 1, nb = (size_t)n_rblk + 1;
  w.z[0] = (double2 *)take(nz * 16);
  w.z[1] = (double2 *)take(nz * 16);
  w.Y = (double2 *)take(nz * 16);
  w.V = (double2 *)take(nz * 16);
  w.X = (double2 *)take(nz * 16);
  w.P = (double2 *)take(nz * 16);
  w.T = (double2 *)take(nz * 16);
  w.U = (double2 *)take(nz * 16);
  w.pz[0] = (double2 *)take(nb * 16);
  w.pz[1] = (double2 *)take(nb * 16);
  w.pz2[0] = (double2 *)take(nb * 16);
  w.pz2[1] = (double2 *)take(nb * 16);
  w.pP = (double2 *)take(nb * 16);
  w.ksum = (double *)take(nz * 8);
  w.status = (cdk_run_status *)take(sizeof(cdk_run_status));
  if (total) *total = off;
  return w;
}

__global__ void ho_reset_status_kernel(cdk_run_status *st) {
  st->nonfinite = 0;
  st->first_bad_step = INT64_MAX;
  st->steps_done = 0;
  st->reserved = 0;
}
__global__ void ho_advance_kernel(cdk_run_status *st, int64_t n) { st->steps_done += n; }

static int ho_check(const cdk_ho_graph *g) {
  if (!g || g->n_rows < 0 || g->n_rblk < 0 || g->n_comm < 0) {
    set_error("cdk_ho_graph: invalid sizes");
    return CDK_INPUT;
  }
  return CDK_OK;
}

static HoArgs ho_args(const cdk_ho_graph *g, const HoWs &w, double *theta, const double *omega,
                      double k1n, double k2n2) {
  HoArgs a{};
  a.n_rows = g->n_rows;
  a.n_rblk = g->n_rblk;
  a.n_comm = g->n_comm;
  a.rblk_row0 = g->rblk_row0;
  a.rblk_comm = g->rblk_comm;
  a.comm_rblk_off = g->comm_rblk_off;
  a.miss_ptr = g->miss_ptr;
  a.miss_col = g->miss_col;
  a.inter_ptr = g->inter_ptr;
  a.inter_col = g->inter_col;
  a.tri_ptr = g->tri_ptr;
  a.tri_jk = reinterpret_cast<const int2 *>(g->tri_jk);
  a.T = w.T;
  a.U = w.U;
  a.Y = w.Y;
  a.V = w.V;
  a.X = w.X;
  a.P = w.P;
  a.pP = w.pP;
  a.theta = theta;
  a.omega = omega;
  a.ksum = w.ksum;
  a.status = w.status;
  a.k1n = k1n;
  a.k2n2 = k2n2;
  return a;
}

static unsigned ho_grid(int32_t n_rblk) {
  const int wpb = 8;
  unsigned gsz = (unsigned)((n_rblk + wpb - 1) / wpb);
  return gsz ? gsz : 1u;
}

template <int MODE>
static int ho_stage(HoArgs a, int src, const HoWs &w, cudaStream_t st) {
  a.z_in = w.z[src];
  a.z_out = w.z[src ^ 1];
  a.pz_in = w.pz[src];
  a.pz2_in = w.pz2[src];
  a.pz_out = w.pz[src ^ 1];
  a.pz2_out = w.pz2[src ^ 1];
  const unsigned row_grid = (unsigned)((a.n_rows * 8 + 255) / 256);
  const unsigned rb_grid = (unsigned)(((int64_t)a.n_rblk * 32 + 255) / 256);
  if (a.n_rows > 0) {
    ho_rowsum_kernel<<<row_grid, 256, 0, st>>>(a);
    CDK_CHECK_LAUNCH("ho_rowsum_kernel");
  }
  // the rblock partials of P (a few warps per SM) and the U sums both read
  // the row sums' P and nothing of each other: side by side
  AuxFork *fk = (a.n_rblk > 0 && a.n_rows > 0) ? aux_fork(st) : nullptr;
  if (a.n_rblk > 0) {
    ho_ppart_kernel<<<rb_grid, 256, 0, fk ? fk->aux : st>>>(a);
    CDK_CHECK_LAUNCH("ho_ppart_kernel");
  }
  if (a.n_rows > 0) {
    ho_usum_kernel<<<row_grid, 256, 0, st>>>(a);
    CDK_CHECK_LAUNCH("ho_usum_kernel");
  }
  if (fk && aux_join(fk, st) != CDK_OK) return CDK_CUDA;
  if (a.n_rblk > 0) {
    ho_epi_kernel<MODE><<<rb_grid, 256, 0, st>>>(a);
    CDK_CHECK_LAUNCH("ho_epi_kernel");
  }
  return CDK_OK;
}

static int ho_prepare(const cdk_ho_graph *g, const HoArgs &a, const double *theta, const HoWs &w,
                      cudaStream_t st) {
  ho_prepare_kernel<<<ho_grid(g->n_rblk), 256, 0, st>>>(a, theta, w.z[0], w.pz[0], w.pz2[0]);
  CDK_CHECK_LAUNCH("ho_prepare_kernel");
  ho_reset_status_kernel<<<1, 1, 0, st>>>(w.status);
  CDK_CHECK_LAUNCH("ho_reset_status_kernel");
  return CDK_OK;
}

}  // namespace cdk

using namespace cdk;

extern "C" size_t cdk_ho_workspace_bytes(const cdk_ho_graph *g) {
  size_t total = 0;
  ho_carve(g->n_rows, g->n_rblk, nullptr, &total);
  return total;
}

extern "C" int cdk_ho_prepare(const cdk_ho_graph *g, const double *theta, void *workspace,
                              void *stream) {
  int rc = ho_check(g);
  if (rc) return rc;
  HoWs w = ho_carve(g->n_rows, g->n_rblk, workspace, nullptr);
  HoArgs a = ho_args(g, w, nullptr, nullptr, 0.0, 0.0);
  return ho_prepare(g, a, theta, w, as_stream(stream));
}

extern "C" int cdk_ho_rhs(const cdk_ho_graph *g, const double *theta, const double *omega,
                          double k1_over_n, double k2_over_n2, double *out, void *workspace,
                          void *stream) {
  int rc = ho_check(g);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  HoWs w = ho_carve(g->n_rows, g->n_rblk, workspace, nullptr);
  HoArgs a = ho_args(g, w, const_cast<double *>(theta), omega, k1_over_n, k2_over_n2);
  if ((rc = ho_prepare(g, a, theta, w, st))) return rc;
  a.out = out;
  return ho_stage<0>(a, 0, w, st);
}

extern "C" int cdk_ho_rk4(const cdk_ho_graph *g, double *theta, const double *omega,
                          double k1_over_n, double k2_over_n2, double dt, int64_t n_steps,
                          void *workspace, void *stream) {
  int rc = ho_check(g);
  if (rc) return rc;
  if (n_steps < 0) return set_error("n_steps < 0"), CDK_INPUT;
  cudaStream_t st = as_stream(stream);
  HoWs w = ho_carve(g->n_rows, g->n_rblk, workspace, nullptr);
  HoArgs a = ho_args(g, w, theta, omega, k1_over_n, k2_over_n2);
  for (int64_t s = 0; s < n_steps; ++s) {
    a.step_rel = s;
    a.h = dt / 2.0;
    if ((rc = ho_stage<1>(a, 0, w, st))) return rc;
    if ((rc = ho_stage<2>(a, 1, w, st))) return rc;
    a.h = dt;
    if ((rc = ho_stage<3>(a, 0, w, st))) return rc;
    a.h = dt / 6.0;
    if ((rc = ho_stage<4>(a, 1, w, st))) return rc;
  }
  if (n_steps > 0) {
    ho_advance_kernel<<<1, 1, 0, st>>>(w.status, n_steps);
    CDK_CHECK_LAUNCH("ho_advance_kernel");
  }
  return CDK_OK;
}

extern "C" int cdk_ho_status(const cdk_ho_graph *g, const void *workspace, cdk_run_status *out,
                             void *stream) {
  int rc = ho_check(g);
  if (rc) return rc;
  HoWs w = ho_carve(g->n_rows, g->n_rblk, const_cast<void *>(workspace), nullptr);
  cudaStream_t st = as_stream(stream);
  cudaError_t e = cudaMemcpyAsync(out, w.status, sizeof(cdk_run_status), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return cuda_status(e, "cdk_ho_status");
}
