// Kernel-level twins of the reference dispatchers (commdyn/_kernels.py), same
// array contracts, for literal drop-in and per-kernel parity testing.  The
// trajectory hot path does NOT use these (it runs the fused kernels in
// kuramoto.cu); they exist so every reference dispatcher on the path has a
// device counterpart.
#include <algorithm>

#include "common.cuh"

namespace cdk {

constexpr int TW_MAXP = 16;  // order/moment twins support p <= 16
constexpr int TW_THREADS = 256;

// block-wide fixed-order sum (warp butterflies, then warp 0 over warp totals)
__device__ double block_sum(double v, double *sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (warp == 0) {
    r = (lane < nw) ? sh[lane] : 0.0;
    r = warp_sum(r);
  }
  __syncthreads();
  if (threadIdx.x == 0) sh[32] = r;
  __syncthreads();
  return sh[32];
}

__device__ __forceinline__ int find_comm(const int64_t *offsets, int64_t m_comm, int64_t node) {
  int64_t lo = 0, hi = m_comm;  // offsets[lo] <= node < offsets[hi]
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (ldg(offsets + mid) <= node) lo = mid; else hi = mid;
  }
  return (int)lo;
}

// _kernels.py:34-51
__global__ void order_params_kernel(const double *x, const int64_t *offsets, int p,
                                    double pi_over_l, double norm, double2 *r) {
  __shared__ double sh[33];
  const int c = blockIdx.x;
  const int64_t b = offsets[c], e = offsets[c + 1];
  double ar[TW_MAXP], ai[TW_MAXP];
#pragma unroll
  for (int a = 0; a < TW_MAXP; ++a) ar[a] = ai[a] = 0.0;
  for (int64_t m = b + threadIdx.x; m < e; m += blockDim.x) {
    double s, co;
    sincos(pi_over_l * x[m], &s, &co);
    double pr = 1.0, pim = 0.0;
#pragma unroll
    for (int a = 0; a < TW_MAXP; ++a) {
      if (a < p) {
        const double nr = pr * co - pim * s;
        const double ni = pr * s + pim * co;
        pr = nr;
        pim = ni;
        ar[a] += pr;
        ai[a] += pim;
      }
    }
  }
  const int w = 2 * p + 1;
  for (int a = 0; a < p; ++a) {
    const double sr = block_sum(ar[a], sh);
    const double si = block_sum(ai[a], sh);
    if (threadIdx.x == 0) {
      r[(int64_t)c * w + p + 1 + a] = make_double2(sr / norm, si / norm);
      r[(int64_t)c * w + p - 1 - a] = make_double2(sr / norm, -(si / norm));
    }
  }
  if (threadIdx.x == 0) r[(int64_t)c * w + p] = make_double2((double)(e - b) / norm, 0.0);
}

// _kernels.py:124-149
__global__ void dense_complex_kernel(const double *x, const int64_t *offsets, int64_t m_comm,
                                     const double2 *tbl, int p, double pi_over_l, double *out,
                                     unsigned long long *guard) {
  const int64_t n_in = offsets[m_comm];
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= n_in) return;
  const int c = find_comm(offsets, m_comm, m);
  const double2 *tc = tbl + (int64_t)c * (2 * p + 1);
  double wi, wr;
  sincos(pi_over_l * x[m], &wi, &wr);
  double accr = tc[2 * p].x, acci = tc[2 * p].y;
  for (int j = 2 * p - 1; j >= 0; --j) {
    const double nr = accr * wr - acci * wi + tc[j].x;
    const double ni = accr * wi + acci * wr + tc[j].y;
    accr = nr;
    acci = ni;
  }
  double sr = 1.0, si = 0.0;  // wbar^p
  for (int k = 0; k < p; ++k) {
    const double nr = sr * wr + si * wi;
    const double ni = si * wr - sr * wi;
    sr = nr;
    si = ni;
  }
  const double vr = accr * sr - acci * si;
  const double vi = fabs(accr * si + acci * sr);
  out[m] += vr;
  if (vi > 1e-9 * (1.0 + fabs(vr))) atomicAdd(guard, 1ull);
  atomicMax(reinterpret_cast<unsigned long long *>(guard + 1),
            (unsigned long long)__double_as_longlong(vi));
}

// _kernels.py:172-187
__global__ void dense_real_kernel(const double *x, const int64_t *offsets, int64_t m_comm,
                                  const double *tcos, const double *tsin, int p, double pi_over_l,
                                  double *out) {
  const int64_t n_in = offsets[m_comm];
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= n_in) return;
  const int c = find_comm(offsets, m_comm, m);
  double s1, c1;
  sincos(pi_over_l * x[m], &s1, &c1);
  double ck = 1.0, sk = 0.0, val = tcos[(int64_t)c * (p + 1)];
  for (int b = 1; b <= p; ++b) {
    const double nck = ck * c1 - sk * s1;
    const double nsk = sk * c1 + ck * s1;
    ck = nck;
    sk = nsk;
    val += tcos[(int64_t)c * (p + 1) + b] * ck + tsin[(int64_t)c * (p + 1) + b] * sk;
  }
  out[m] += val;
}

// _kernels.py:246-283 (scatter to both ends, fp64 atomics)
__global__ void pairs_trig_kernel(const int64_t *iu, const int64_t *iv, int64_t n_pairs,
                                  const double *x, double inv_n, const double *d_cos,
                                  const double *d_sin, int p, double pi_over_l, const double *sgn,
                                  double *out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n_pairs) return;
  const int64_t u = iu[e], v = iv[e];
  const double s = sgn[e] * inv_n;
  double s1, c1;
  sincos(pi_over_l * (x[v] - x[u]), &s1, &c1);
  double ck = 1.0, sk = 0.0, hp = d_cos[0], hm = d_cos[0];
  for (int a = 1; a <= p; ++a) {
    const double nck = ck * c1 - sk * s1;
    const double nsk = sk * c1 + ck * s1;
    ck = nck;
    sk = nsk;
    hp += d_cos[a] * ck + d_sin[a] * sk;
    hm += d_cos[a] * ck - d_sin[a] * sk;
  }
  atomicAdd(out + u, s * hp);
  if (u != v) atomicAdd(out + v, s * hm);
}

// _kernels.py:297-314
__global__ void pairs_cs_kernel(const int64_t *iu, const int64_t *iv, int64_t n_pairs,
                                const double *pos, const double *vel, int ndim, double inv_n,
                                double amp, double sigma2, double beta, const double *sgn,
                                double *out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n_pairs) return;
  const int64_t u = iu[e], v = iv[e];
  if (u == v) return;
  double d2 = 0.0;
  for (int d = 0; d < ndim; ++d) {
    const double dd = pos[v * ndim + d] - pos[u * ndim + d];
    d2 += dd * dd;
  }
  const double eta = amp / pow(sigma2 + d2, beta);
  const double s = sgn[e] * inv_n * eta;
  for (int d = 0; d < ndim; ++d) {
    const double dv = vel[v * ndim + d] - vel[u * ndim + d];
    atomicAdd(out + u * ndim + d, s * dv);
    atomicAdd(out + v * ndim + d, -(s * dv));
  }
}

// _kernels.py:81-93
__global__ void moments_kernel(const double *x, const int64_t *offsets, int p, double x0,
                               double norm, double *w) {
  __shared__ double sh[33];
  const int c = blockIdx.x;
  const int64_t b = offsets[c], e = offsets[c + 1];
  double acc[TW_MAXP + 1];
#pragma unroll
  for (int a = 0; a <= TW_MAXP; ++a) acc[a] = 0.0;
  for (int64_t m = b + threadIdx.x; m < e; m += blockDim.x) {
    const double t = x[m] - x0;
    double tp = 1.0;
    acc[0] += 1.0;
#pragma unroll
    for (int a = 1; a <= TW_MAXP; ++a) {
      if (a <= p) {
        tp = tp * t;
        acc[a] += tp;
      }
    }
  }
  for (int a = 0; a <= p; ++a) {
    const double sa = block_sum(acc[a], sh);
    if (threadIdx.x == 0) w[(int64_t)c * (p + 1) + a] = sa / norm;
  }
}

// _kernels.py:207-217
__global__ void dense_poly_kernel(const double *x, const int64_t *offsets, int64_t m_comm,
                                  const double *tbl, int p, double scale, double shift,
                                  double *out) {
  const int64_t n_in = offsets[m_comm];
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= n_in) return;
  const int c = find_comm(offsets, m_comm, m);
  const double *tc = tbl + (int64_t)c * (p + 1);
  const double t = scale * x[m] + shift;
  double val = tc[p];
  for (int b = p - 1; b >= 0; --b) val = val * t + tc[b];
  out[m] += val;
}

// _kernels.py:264-271,286-294 (poly coupling over pairs; Horner as
// _poly_eval_nb; scatter to both ends with fp64 atomics like pairs_trig)
__global__ void pairs_poly_kernel(const int64_t *iu, const int64_t *iv, int64_t n_pairs,
                                  const double *x, double inv_n, const double *coef, int p,
                                  double x0, const double *sgn, double *out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n_pairs) return;
  const int64_t u = iu[e], v = iv[e];
  const double s = sgn[e] * inv_n;
  const double d = x[v] - x[u];
  // no FMA contraction (the reference's numba body rounds every * and +)
  double t = d - x0, val = coef[p];
  for (int a = p - 1; a >= 0; --a) val = __dadd_rn(__dmul_rn(val, t), coef[a]);
  atomicAdd(out + u, s * val);
  if (u != v) {
    t = -d - x0;
    val = coef[p];
    for (int a = p - 1; a >= 0; --a) val = __dadd_rn(__dmul_rn(val, t), coef[a]);
    atomicAdd(out + v, s * val);
  }
}

// _kernels.py:398-410: out[m] = (1/lam^3) sum_{i1,i2,i3} sin(l1 th1 + l2 th2 +
// l3 th3 + l4 th_m).  One thread per m walks (i1, i2, i3) in the reference's
// order, so every out[m] sums its terms in the same sequence; theta staged in
// shared memory (lam <= 4096).
constexpr int HO_NAIVE_MAX = 4096;
__global__ void ho_naive_block_kernel(const double *theta, int lam, double l1, double l2,
                                      double l3, double l4, double *out) {
  __shared__ double th[HO_NAIVE_MAX];
  for (int i = threadIdx.x; i < lam; i += blockDim.x) th[i] = theta[i];
  __syncthreads();
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= lam) return;
  const double am = l4 * th[m];
  double acc = 0.0;
  for (int i1 = 0; i1 < lam; ++i1) {
    const double a1 = l1 * th[i1];
    for (int i2 = 0; i2 < lam; ++i2) {
      const double a12 = __dadd_rn(a1, __dmul_rn(l2, th[i2]));
      for (int i3 = 0; i3 < lam; ++i3) acc += sin(__dadd_rn(a12, __dmul_rn(l3, th[i3])) + am);
    }
  }
  const double l3d = (double)lam * (double)lam * (double)lam;
  out[m] = acc / l3d;
}

// _kernels.py:436-456: window sums F_m = inv_n sum_{l=m-k..m+k} ph[l mod n]
// with the O(1) update, re-anchored by a direct sum every anchor_every steps.
// Anchored segments are independent, so one thread per segment reproduces the
// reference's arithmetic exactly (same additions in the same order).
__global__ void nn_recurrence_kernel(const double2 *ph, int64_t n, int64_t k, double inv_n,
                                     int64_t anchor_every, double2 *f) {
  const int64_t seg = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t start = seg * anchor_every;
  if (start >= n) return;
  const int64_t stop = min(start + anchor_every, n);
  auto at = [&](int64_t l) { int64_t r = l % n; return ph[r < 0 ? r + n : r]; };
  double wr = 0.0, wi = 0.0;
  for (int64_t l = start - k; l <= start + k; ++l) {
    const double2 q = at(l);
    wr += q.x;
    wi += q.y;
  }
  f[start] = make_double2(wr * inv_n, wi * inv_n);
  for (int64_t m = start + 1; m < stop; ++m) {
    const double2 a = at(m - 1 - k), b = at(m + k);
    wr = (wr - a.x) + b.x;
    wi = (wi - a.y) + b.y;
    f[m] = make_double2(wr * inv_n, wi * inv_n);
  }
}

// _kernels.py:485-509: f[m] = sum_l spins[l] for every m (int64, exact).
__global__ void spin_sum_kernel(const int64_t *spins, int64_t n, unsigned long long *total) {
  long long acc = 0;
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n;
       l += (int64_t)gridDim.x * blockDim.x)
    acc += spins[l];
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(total, (unsigned long long)acc);  // two's complement
}

__global__ void spin_fill_kernel(const unsigned long long *total, int64_t n, int64_t *f) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m < n) f[m] = (int64_t)*total;
}

// Direct-sum triadic term of the higher-order Kuramoto model (SPEC.md:463-470
// naive mode): every 3-clique {a, b, c} of the graph adds
// coef * sin(theta_b + theta_c - 2 theta_a) to out[a] (and the two rotations),
// coef = 2 K2 / N^2 (ordered (j, k) pairs).  fp64 atomics.
__global__ void triangles_sin_kernel(const int64_t *tri, int64_t n_tri, const double *theta,
                                     double coef, double *out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_tri) return;
  const int64_t a = tri[3 * t], b = tri[3 * t + 1], c = tri[3 * t + 2];
  const double ta = theta[a], tb = theta[b], tc = theta[c];
  atomicAdd(out + a, coef * sin((tb + tc) - 2.0 * ta));
  atomicAdd(out + b, coef * sin((ta + tc) - 2.0 * tb));
  atomicAdd(out + c, coef * sin((ta + tb) - 2.0 * tc));
}

// Appendix B.1 rank-one coupling: r = inv_n sum_l beta_l
// e^{i x_l} (fixed-order two-level sum: per-block partials, then block order),
// out_m = alpha_m r e^{-i x_m} (complex, interleaved).
__global__ void rank_one_partial_kernel(const double *beta, const double *x, int64_t n,
                                        double2 *part) {
  __shared__ double sh[33];
  double sr = 0.0, si = 0.0;
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n;
       l += (int64_t)gridDim.x * blockDim.x) {
    double s, c;
    sincos(x[l], &s, &c);
    sr += beta[l] * c;
    si += beta[l] * s;
  }
  const double br = block_sum(sr, sh);
  const double bi = block_sum(si, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = make_double2(br, bi);
}

__global__ void rank_one_apply_kernel(const double *alpha, const double *x, int64_t n,
                                      const double2 *part, int n_part, double inv_n,
                                      double2 *out) {
  __shared__ double2 r_sh;
  if (threadIdx.x == 0) {
    double rr = 0.0, ri = 0.0;
    for (int q = 0; q < n_part; ++q) {  // block order
      rr += part[q].x;
      ri += part[q].y;
    }
    r_sh = make_double2(rr * inv_n, ri * inv_n);
  }
  __syncthreads();
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= n) return;
  double s, c;
  sincos(x[m], &s, &c);
  const double2 r = r_sh;
  // alpha r e^{-ix}
  out[m] = make_double2(alpha[m] * (r.x * c + r.y * s), alpha[m] * (r.y * c - r.x * s));
}

static inline unsigned grid_for(int64_t n) {
  return (unsigned)((n + TW_THREADS - 1) / TW_THREADS);
}

static int need_offsets_host(const int64_t *offsets_dev, int64_t m_comm, int64_t *n_in,
                             cudaStream_t st) {
  // n_in = offsets[m_comm] is read on the device by every per-node twin; only
  // an emptiness check is needed on the host to avoid zero-size grids.
  cudaError_t e = cudaMemcpyAsync(n_in, offsets_dev + m_comm, sizeof(int64_t),
                                  cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return cuda_status(e, "read offsets[-1]");
}

}  // namespace cdk

using namespace cdk;

extern "C" int cdk_order_params_blocks(const double *x, const int64_t *offsets, int64_t m_comm,
                                       int p, double pi_over_l, double norm, double *r,
                                       void *stream) {
  if (p < 0 || p > TW_MAXP || m_comm < 0) {
    set_error("order_params_blocks: need 0 <= p <= 16");
    return CDK_INPUT;
  }
  if (m_comm == 0) return CDK_OK;
  order_params_kernel<<<(unsigned)m_comm, TW_THREADS, 0, as_stream(stream)>>>(
      x, offsets, p, pi_over_l, norm, reinterpret_cast<double2 *>(r));
  CDK_CHECK_LAUNCH("order_params_kernel");
  return CDK_OK;
}

extern "C" int cdk_dense_complex(const double *x, const int64_t *offsets, int64_t m_comm,
                                 const double *tbl, int p, double pi_over_l, double *out,
                                 void *guard, void *stream) {
  if (p < 0 || m_comm < 0) return set_error("dense_complex: bad p"), CDK_INPUT;
  if (m_comm == 0) return CDK_OK;
  cudaStream_t st = as_stream(stream);
  int64_t n_in = 0;
  int rc = need_offsets_host(offsets, m_comm, &n_in, st);
  if (rc || n_in == 0) return rc;
  dense_complex_kernel<<<grid_for(n_in), TW_THREADS, 0, st>>>(
      x, offsets, m_comm, reinterpret_cast<const double2 *>(tbl), p, pi_over_l, out,
      reinterpret_cast<unsigned long long *>(guard));
  CDK_CHECK_LAUNCH("dense_complex_kernel");
  return CDK_OK;
}

extern "C" int cdk_dense_real(const double *x, const int64_t *offsets, int64_t m_comm,
                              const double *tbl_cos, const double *tbl_sin, int p,
                              double pi_over_l, double *out, void *stream) {
  if (p < 0 || m_comm < 0) return set_error("dense_real: bad p"), CDK_INPUT;
  if (m_comm == 0) return CDK_OK;
  cudaStream_t st = as_stream(stream);
  int64_t n_in = 0;
  int rc = need_offsets_host(offsets, m_comm, &n_in, st);
  if (rc || n_in == 0) return rc;
  dense_real_kernel<<<grid_for(n_in), TW_THREADS, 0, st>>>(x, offsets, m_comm, tbl_cos, tbl_sin,
                                                            p, pi_over_l, out);
  CDK_CHECK_LAUNCH("dense_real_kernel");
  return CDK_OK;
}

extern "C" int cdk_pairs_trig(const int64_t *iu, const int64_t *iv, int64_t n_pairs,
                              const double *x, double inv_n, const double *d_cos,
                              const double *d_sin, int p, double pi_over_l, const double *sgn,
                              double *out, void *stream) {
  if (p < 0 || n_pairs < 0) return set_error("pairs_trig: bad sizes"), CDK_INPUT;
  if (n_pairs == 0) return CDK_OK;
  pairs_trig_kernel<<<grid_for(n_pairs), TW_THREADS, 0, as_stream(stream)>>>(
      iu, iv, n_pairs, x, inv_n, d_cos, d_sin, p, pi_over_l, sgn, out);
  CDK_CHECK_LAUNCH("pairs_trig_kernel");
  return CDK_OK;
}

extern "C" int cdk_pairs_cs(const int64_t *iu, const int64_t *iv, int64_t n_pairs,
                            const double *pos, const double *vel, int ndim, double inv_n,
                            double amp, double sigma2, double beta, const double *sgn,
                            double *out, void *stream) {
  if (ndim < 1 || n_pairs < 0) return set_error("pairs_cs: bad sizes"), CDK_INPUT;
  if (n_pairs == 0) return CDK_OK;
  pairs_cs_kernel<<<grid_for(n_pairs), TW_THREADS, 0, as_stream(stream)>>>(
      iu, iv, n_pairs, pos, vel, ndim, inv_n, amp, sigma2, beta, sgn, out);
  CDK_CHECK_LAUNCH("pairs_cs_kernel");
  return CDK_OK;
}

extern "C" int cdk_moments_blocks(const double *x, const int64_t *offsets, int64_t m_comm, int p,
                                  double x0, double norm, double *w, void *stream) {
  if (p < 0 || p > TW_MAXP || m_comm < 0) {
    set_error("moments_blocks: need 0 <= p <= 16");
    return CDK_INPUT;
  }
  if (m_comm == 0) return CDK_OK;
  moments_kernel<<<(unsigned)m_comm, TW_THREADS, 0, as_stream(stream)>>>(x, offsets, p, x0, norm,
                                                                          w);
  CDK_CHECK_LAUNCH("moments_kernel");
  return CDK_OK;
}

extern "C" int cdk_dense_poly(const double *x, const int64_t *offsets, int64_t m_comm,
                              const double *tbl, int p, double scale, double shift, double *out,
                              void *stream) {
  if (p < 0 || m_comm < 0) return set_error("dense_poly: bad p"), CDK_INPUT;
  if (m_comm == 0) return CDK_OK;
  cudaStream_t st = as_stream(stream);
  int64_t n_in = 0;
  int rc = need_offsets_host(offsets, m_comm, &n_in, st);
  if (rc || n_in == 0) return rc;
  dense_poly_kernel<<<grid_for(n_in), TW_THREADS, 0, st>>>(x, offsets, m_comm, tbl, p, scale,
                                                            shift, out);
  CDK_CHECK_LAUNCH("dense_poly_kernel");
  return CDK_OK;
}

extern "C" int cdk_pairs_poly(const int64_t *iu, const int64_t *iv, int64_t n_pairs,
                              const double *x, double inv_n, const double *coef, int p,
                              double x0, const double *sgn, double *out, void *stream) {
  if (p < 0 || n_pairs < 0) return set_error("pairs_poly: bad sizes"), CDK_INPUT;
  if (n_pairs == 0) return CDK_OK;
  pairs_poly_kernel<<<grid_for(n_pairs), TW_THREADS, 0, as_stream(stream)>>>(
      iu, iv, n_pairs, x, inv_n, coef, p, x0, sgn, out);
  CDK_CHECK_LAUNCH("pairs_poly_kernel");
  return CDK_OK;
}

extern "C" int cdk_ho_naive_block(const double *theta, int64_t lam, double l1, double l2,
                                  double l3, double l4, double *out, void *stream) {
  if (lam < 0 || lam > HO_NAIVE_MAX) {
    set_error("ho_naive_block: need 0 <= lam <= 4096");
    return CDK_INPUT;
  }
  if (lam == 0) return CDK_OK;
  constexpr int T = 128;
  ho_naive_block_kernel<<<(unsigned)((lam + T - 1) / T), T, 0, as_stream(stream)>>>(
      theta, (int)lam, l1, l2, l3, l4, out);
  CDK_CHECK_LAUNCH("ho_naive_block_kernel");
  return CDK_OK;
}

extern "C" int cdk_nn_recurrence(const double *ph, int64_t n, int64_t k, double inv_n,
                                 int64_t anchor_every, double *f, void *stream) {
  if (n < 0 || k < 0 || anchor_every < 1) {
    set_error("nn_recurrence: need n >= 0, k >= 0, anchor_every >= 1");
    return CDK_INPUT;
  }
  if (n == 0) return CDK_OK;
  const int64_t segs = (n + anchor_every - 1) / anchor_every;
  constexpr int T = 64;
  nn_recurrence_kernel<<<(unsigned)((segs + T - 1) / T), T, 0, as_stream(stream)>>>(
      reinterpret_cast<const double2 *>(ph), n, k, inv_n, anchor_every,
      reinterpret_cast<double2 *>(f));
  CDK_CHECK_LAUNCH("nn_recurrence_kernel");
  return CDK_OK;
}

extern "C" int cdk_spin_field_sums(const int64_t *spins, int64_t n, int64_t *f,
                                   void *scratch, void *stream) {
  if (n < 0) return set_error("spin_field_sums: bad n"), CDK_INPUT;
  if (n == 0) return CDK_OK;
  cudaStream_t st = as_stream(stream);
  auto *total = reinterpret_cast<unsigned long long *>(scratch);
  cudaError_t e = cudaMemsetAsync(total, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return cuda_status(e, "spin_field_sums memset");
  const unsigned g = (unsigned)std::min<int64_t>(grid_for(n), 148 * 8);
  spin_sum_kernel<<<g, TW_THREADS, 0, st>>>(spins, n, total);
  CDK_CHECK_LAUNCH("spin_sum_kernel");
  spin_fill_kernel<<<grid_for(n), TW_THREADS, 0, st>>>(total, n, f);
  CDK_CHECK_LAUNCH("spin_fill_kernel");
  return CDK_OK;
}

extern "C" int cdk_triangles_sin(const int64_t *tri, int64_t n_tri, const double *theta,
                                 double coef, double *out, void *stream) {
  if (n_tri < 0) return set_error("triangles_sin: bad n_tri"), CDK_INPUT;
  if (n_tri == 0) return CDK_OK;
  triangles_sin_kernel<<<grid_for(n_tri), TW_THREADS, 0, as_stream(stream)>>>(tri, n_tri, theta,
                                                                               coef, out);
  CDK_CHECK_LAUNCH("triangles_sin_kernel");
  return CDK_OK;
}

extern "C" int cdk_rank_one(const double *alpha, const double *beta, const double *x, int64_t n,
                            double inv_n, double *out, void *scratch, void *stream) {
  if (n < 0) return set_error("rank_one: bad n"), CDK_INPUT;
  if (n == 0) return CDK_OK;
  cudaStream_t st = as_stream(stream);
  constexpr int NPART = 148;  // scratch: NPART double2
  auto *part = reinterpret_cast<double2 *>(scratch);
  rank_one_partial_kernel<<<NPART, TW_THREADS, 0, st>>>(beta, x, n, part);
  CDK_CHECK_LAUNCH("rank_one_partial_kernel");
  rank_one_apply_kernel<<<grid_for(n), TW_THREADS, 0, st>>>(
      alpha, x, n, part, NPART, inv_n, reinterpret_cast<double2 *>(out));
  CDK_CHECK_LAUNCH("rank_one_apply_kernel");
  return CDK_OK;
}
