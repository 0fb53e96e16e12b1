// Higher-harmonics Kuramoto (SPEC.md:440-446 higher_harmonics_rhs; SURVEY
// §8f rank 3), CIA form fused into RK4 — the p > 1 generalisation of the
// first-mode path in kuramoto.cu:
//
//   theta'_i = omega_i + (1/N) sum_l a_il h(theta_l - theta_i),
//   h(x) = sum_{a=0..p} d_cos[a] cos(a x) + d_sin[a] sin(a x)      (p <= 8)
//
// E1 (replaces order_params_blocks + dense_complex/dense_real,
// _kernels.py:34-73,124-204): per community c and mode a the observable
// R_ac = sum_{l in c} Z_a[l], Z_a = e^{i a theta}; the dense part of node i is
//   d_cos[0] lambda_c + sum_a d_cos[a] Re(R_ac conj Z_a[i]) + d_sin[a] Im(R_ac conj Z_a[i]).
// E2 (replaces pairs_trig with p harmonics, _kernels.py:246-283): the signed
// sums S_a[i] = sum_j s_ij Z_a[j] over the directed correction (missing intra
// -1, inter +1) give the same expression with R -> S plus d_cos[0] sum_j s_ij;
// the diagonal entry (i, i, -1) of every in-community node
// subtracts h(0) = sum_a d_cos[a].
// Per stage: one reduce launch (R_ac from the previous stage's canonical
// rblock partials, fixed order) and one stage launch (warp per rblock, lane =
// row: the row's corrections gather Z_a of its neighbours from L2, then the
// RK4 stage update, Z_a of the new phase by the rotation recurrence, the
// rblock partials).  All reductions fixed-order: bitwise deterministic.
#include "common.cuh"

namespace cdk {

constexpr int HH_MAXP = 8;

struct HhArgs {
  int64_t n_rows;
  int32_t n_rblk, n_comm, p;
  const int64_t *rblk_row0;
  const int32_t *rblk_comm;
  const int32_t *comm_rblk_off;
  const int64_t *comm_off;  // [n_comm+1] community row offsets (lambda_c)
  const int64_t *miss_ptr;
  const int32_t *miss_col;
  const int64_t *inter_ptr;
  const int32_t *inter_col;
  const double *d_cos, *d_sin;  // [p+1], coupling folded in
  const double2 *z_in;          // [p][n_rows]
  double2 *z_out;
  const double2 *part_in;       // [p][n_rblk]
  double2 *part_out;
  double2 *R;                   // [p][n_comm]
  double *theta;
  const double *omega;
  double *ksum;
  double *out;
  cdk_run_status *status;
  double inv_n, h;
  int64_t step_rel;
};

__device__ __forceinline__ double2 hh_partial(double2 v) {
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

// Z_a = e^{i a theta}, a = 1..p, by the rotation recurrence (the pairs_trig
// recurrence, _kernels.py:246-261), stored mode-major
__device__ __forceinline__ void hh_powers(double th, int p, double2 (&z)[HH_MAXP]) {
  double s1, c1;
  sincos(th, &s1, &c1);
  double ck = 1.0, sk = 0.0;
#pragma unroll
  for (int a = 0; a < HH_MAXP; ++a) {
    if (a < p) {
      const double nck = ck * c1 - sk * s1;
      const double nsk = sk * c1 + ck * s1;
      ck = nck;
      sk = nsk;
    }
    z[a] = make_double2(ck, sk);
  }
}

__global__ void __launch_bounds__(256) hh_prepare_kernel(const HhArgs a) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int rb = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; rb < a.n_rblk; rb += warps) {
    const int64_t row0 = a.rblk_row0[rb];
    const int nr = (int)(a.rblk_row0[rb + 1] - row0);
    double2 z[HH_MAXP];
    if (lane < nr) {
      hh_powers(a.theta[row0 + lane], a.p, z);
    } else {
#pragma unroll
      for (int q = 0; q < HH_MAXP; ++q) z[q] = make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int q = 0; q < HH_MAXP; ++q) {
      if (q < a.p) {
        if (lane < nr) a.z_out[q * a.n_rows + row0 + lane] = z[q];
        const double2 pv = hh_partial(z[q]);
        if (lane == 0) a.part_out[(int64_t)q * a.n_rblk + rb] = pv;
      }
    }
  }
}

// R_ac: 8 lanes per (community, mode), canonical order (reduce_comm8's)
__global__ void __launch_bounds__(256) hh_reduce_kernel(const HhArgs a) {
  const int t = threadIdx.x & 7;
  const unsigned gmask = 0xFFu << (threadIdx.x & 24);
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 3;
  if (g >= (int64_t)a.n_comm * a.p) return;
  const int c = (int)(g % a.n_comm), q = (int)(g / a.n_comm);
  const int b0 = a.comm_rblk_off[c], b1 = a.comm_rblk_off[c + 1];
  const double2 *part = a.part_in + (int64_t)q * a.n_rblk;
  double sr = 0.0, si = 0.0;
  for (int b = b0 + t; b < b1; b += 8) {
    const double2 v = __ldcg(part + b);
    sr += v.x;
    si += v.y;
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    sr += __shfl_xor_sync(gmask, sr, o);
    si += __shfl_xor_sync(gmask, si, o);
  }
  if (t == 0) a.R[(int64_t)q * a.n_comm + c] = make_double2(sr, si);
}

template <int MODE>
__global__ void __launch_bounds__(256) hh_stage_kernel(const HhArgs a) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int p = a.p;
  for (int rb = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; rb < a.n_rblk; rb += warps) {
    const int64_t row0 = a.rblk_row0[rb];
    const int nr = (int)(a.rblk_row0[rb + 1] - row0);
    const int c = a.rblk_comm[rb];
    double2 zn[HH_MAXP];
#pragma unroll
    for (int q = 0; q < HH_MAXP; ++q) zn[q] = make_double2(0.0, 0.0);
    if (lane < nr) {
      const int64_t i = row0 + lane;
      double2 S[HH_MAXP];
#pragma unroll
      for (int q = 0; q < HH_MAXP; ++q) S[q] = make_double2(0.0, 0.0);
      // signed sums over the row's corrections (missing intra: -1, inter: +1)
      const int64_t m0 = a.miss_ptr[i], m1 = a.miss_ptr[i + 1];
      const int64_t x0 = a.inter_ptr[i], x1 = a.inter_ptr[i + 1];
#pragma unroll 4
      for (int64_t e = m0; e < m1; ++e) {
        const int64_t j = a.miss_col[e];
#pragma unroll
        for (int q = 0; q < HH_MAXP; ++q)
          if (q < p) {
            const double2 v = __ldcg(a.z_in + q * a.n_rows + j);
            S[q].x -= v.x;
            S[q].y -= v.y;
          }
      }
#pragma unroll 4
      for (int64_t e = x0; e < x1; ++e) {
        const int64_t j = a.inter_col[e];
#pragma unroll
        for (int q = 0; q < HH_MAXP; ++q)
          if (q < p) {
            const double2 v = __ldcg(a.z_in + q * a.n_rows + j);
            S[q].x += v.x;
            S[q].y += v.y;
          }
      }
      const double s0 = (double)((x1 - x0) - (m1 - m0));
      // coupling sum: sparse part, then the community's dense part
      double acc = a.d_cos[0] * s0;
      double h0 = a.d_cos[0];
#pragma unroll
      for (int q = 0; q < HH_MAXP; ++q)
        if (q < p) {
          const double2 zi = __ldcg(a.z_in + q * a.n_rows + i);
          const double2 w = S[q];
          // Re/Im(w conj zi)
          acc += a.d_cos[q + 1] * (w.x * zi.x + w.y * zi.y) +
                 a.d_sin[q + 1] * (w.y * zi.x - w.x * zi.y);
          h0 += a.d_cos[q + 1];
        }
      if (c >= 0) {
        double dense = a.d_cos[0] * (double)(a.comm_off[c + 1] - a.comm_off[c]);
#pragma unroll
        for (int q = 0; q < HH_MAXP; ++q)
          if (q < p) {
            const double2 zi = __ldcg(a.z_in + q * a.n_rows + i);
            const double2 Rq = __ldcg(a.R + (int64_t)q * a.n_comm + c);
            dense += a.d_cos[q + 1] * (Rq.x * zi.x + Rq.y * zi.y) +
                     a.d_sin[q + 1] * (Rq.y * zi.x - Rq.x * zi.y);
          }
        acc = (dense + acc) - h0;  // the diagonal correction (i, i, -1)
      }
      const double k = a.omega[i] + a.inv_n * acc;
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
        hh_powers(thn, p, zn);
#pragma unroll
        for (int q = 0; q < HH_MAXP; ++q)
          if (q < p) a.z_out[q * a.n_rows + i] = zn[q];
      }
    }
    if (MODE != 0) {
#pragma unroll
      for (int q = 0; q < HH_MAXP; ++q)
        if (q < p) {
          const double2 pv = hh_partial(zn[q]);
          if (lane == 0) a.part_out[(int64_t)q * a.n_rblk + rb] = pv;
        }
    }
  }
}

__global__ void hh_reset_status_kernel(cdk_run_status *st) {
  st->nonfinite = 0;
  st->first_bad_step = INT64_MAX;
  st->steps_done = 0;
  st->reserved = 0;
}

__global__ void hh_advance_kernel(cdk_run_status *st, int64_t n) { st->steps_done += n; }

struct HhWs {
  double2 *z[2], *part[2], *R;
  double *ksum;
  cdk_run_status *status;
};

static size_t hh_align(size_t x) { return (x + 255) / 256 * 256; }

static HhWs hh_carve(const cdk_hh_graph *g, void *base, size_t *total) {
  HhWs w{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    void *p = base ? static_cast<char *>(base) + off : nullptr;
    off += hh_align(bytes ? bytes : 1);
    return p;
  };
  const size_t zb = sizeof(double2) * (size_t)g->p * (size_t)g->n_rows;
  const size_t pb = sizeof(double2) * (size_t)g->p * (size_t)(g->n_rblk > 0 ? g->n_rblk : 1);
  w.z[0] = static_cast<double2 *>(take(zb));
  w.z[1] = static_cast<double2 *>(take(zb));
  w.part[0] = static_cast<double2 *>(take(pb));
  w.part[1] = static_cast<double2 *>(take(pb));
  w.R = static_cast<double2 *>(take(sizeof(double2) * (size_t)g->p *
                                    (size_t)(g->n_comm > 0 ? g->n_comm : 1)));
  w.ksum = static_cast<double *>(take(sizeof(double) * (size_t)g->n_rows));
  w.status = static_cast<cdk_run_status *>(take(sizeof(cdk_run_status)));
  if (total) *total = off;
  return w;
}

static int hh_check(const cdk_hh_graph *g) {
  if (!g || g->n_rows < 0 || g->n_rblk < 0 || g->n_comm < 0) return set_error("hh: bad graph"), CDK_INPUT;
  if (g->p < 1 || g->p > HH_MAXP) return set_error("hh: need 1 <= p <= 8"), CDK_INPUT;
  return CDK_OK;
}

static HhArgs hh_args(const cdk_hh_graph *g, const HhWs &w, double *theta, const double *omega,
                      double inv_n) {
  HhArgs a{};
  a.n_rows = g->n_rows;
  a.n_rblk = g->n_rblk;
  a.n_comm = g->n_comm;
  a.p = g->p;
  a.rblk_row0 = g->rblk_row0;
  a.rblk_comm = g->rblk_comm;
  a.comm_rblk_off = g->comm_rblk_off;
  a.comm_off = g->comm_off;
  a.miss_ptr = g->miss_ptr;
  a.miss_col = g->miss_col;
  a.inter_ptr = g->inter_ptr;
  a.inter_col = g->inter_col;
  a.d_cos = g->d_cos;
  a.d_sin = g->d_sin;
  a.R = w.R;
  a.theta = theta;
  a.omega = omega;
  a.ksum = w.ksum;
  a.status = w.status;
  a.inv_n = inv_n;
  return a;
}

static unsigned hh_grid(int64_t warps_needed) {
  const int64_t g = (warps_needed + 7) / 8;
  return (unsigned)(g > 0 ? g : 1);
}

template <int MODE>
static int hh_stage(HhArgs a, int src, const HhWs &w, cudaStream_t st) {
  a.z_in = w.z[src];
  a.z_out = w.z[src ^ 1];
  a.part_in = w.part[src];
  a.part_out = w.part[src ^ 1];
  if (a.n_comm > 0) {
    const int64_t groups = (int64_t)a.n_comm * a.p;
    hh_reduce_kernel<<<(unsigned)((groups * 8 + 255) / 256), 256, 0, st>>>(a);
    CDK_CHECK_LAUNCH("hh_reduce_kernel");
  }
  hh_stage_kernel<MODE><<<hh_grid(a.n_rblk), 256, 0, st>>>(a);
  CDK_CHECK_LAUNCH("hh_stage_kernel");
  return CDK_OK;
}

static int hh_prepare(HhArgs a, const HhWs &w, cudaStream_t st) {
  a.z_out = w.z[0];
  a.part_out = w.part[0];
  hh_prepare_kernel<<<hh_grid(a.n_rblk), 256, 0, st>>>(a);
  CDK_CHECK_LAUNCH("hh_prepare_kernel");
  hh_reset_status_kernel<<<1, 1, 0, st>>>(w.status);
  CDK_CHECK_LAUNCH("hh_reset_status_kernel");
  return CDK_OK;
}

}  // namespace cdk

using namespace cdk;

extern "C" size_t cdk_hh_workspace_bytes(const cdk_hh_graph *g) {
  size_t total = 0;
  hh_carve(g, nullptr, &total);
  return total;
}

extern "C" int cdk_hh_prepare(const cdk_hh_graph *g, const double *theta, void *workspace,
                              void *stream) {
  int rc = hh_check(g);
  if (rc) return rc;
  HhWs w = hh_carve(g, workspace, nullptr);
  HhArgs a = hh_args(g, w, const_cast<double *>(theta), nullptr, 0.0);
  return hh_prepare(a, w, as_stream(stream));
}

extern "C" int cdk_hh_rhs(const cdk_hh_graph *g, const double *theta, const double *omega,
                          double inv_n, double *out, void *workspace, void *stream) {
  int rc = hh_check(g);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  HhWs w = hh_carve(g, workspace, nullptr);
  HhArgs a = hh_args(g, w, const_cast<double *>(theta), omega, inv_n);
  if ((rc = hh_prepare(a, w, st))) return rc;
  a.out = out;
  return hh_stage<0>(a, 0, w, st);
}

extern "C" int cdk_hh_rk4(const cdk_hh_graph *g, double *theta, const double *omega,
                          double inv_n, double dt, int64_t n_steps, void *workspace,
                          void *stream) {
  int rc = hh_check(g);
  if (rc) return rc;
  if (n_steps < 0) return set_error("n_steps < 0"), CDK_INPUT;
  cudaStream_t st = as_stream(stream);
  HhWs w = hh_carve(g, workspace, nullptr);
  HhArgs a = hh_args(g, w, theta, omega, inv_n);
  for (int64_t s = 0; s < n_steps; ++s) {
    a.step_rel = s;
    a.h = dt / 2.0;
    if ((rc = hh_stage<1>(a, 0, w, st))) return rc;
    if ((rc = hh_stage<2>(a, 1, w, st))) return rc;
    a.h = dt;
    if ((rc = hh_stage<3>(a, 0, w, st))) return rc;
    a.h = dt / 6.0;
    if ((rc = hh_stage<4>(a, 1, w, st))) return rc;
  }
  if (n_steps > 0) {
    hh_advance_kernel<<<1, 1, 0, st>>>(w.status, n_steps);
    CDK_CHECK_LAUNCH("hh_advance_kernel");
  }
  return CDK_OK;
}

extern "C" int cdk_hh_status(const cdk_hh_graph *g, const void *workspace, cdk_run_status *out,
                             void *stream) {
  int rc = hh_check(g);
  if (rc) return rc;
  HhWs w = hh_carve(g, const_cast<void *>(workspace), nullptr);
  cudaStream_t st = as_stream(stream);
  cudaError_t e = cudaMemcpyAsync(out, w.status, sizeof(cdk_run_status), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return cuda_status(e, "hh status");
}
