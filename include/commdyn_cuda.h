/*
 * commdyn_cuda.h — C ABI of libcommdyn_cuda.so, the B200 (sm_100a) drop-in for
 * the Community Integration Algorithm hot path of the reference package
 * `commdyn` (arXiv 2203.16657).
 *
 * Conventions (all entry points):
 *   - every array argument is a DEVICE pointer unless marked [host];
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream);
 *     work is stream-ordered, nothing synchronises unless stated;
 *   - complex arrays are interleaved (re, im) float64, i.e. numpy complex128;
 *   - return value is a status: CDK_OK, CDK_INPUT (bad shape/argument),
 *     CDK_CUDA (CUDA runtime error; cdk_last_error() has the text).  Numeric
 *     guards (blow-up, imaginary residue) are REPORTED through output counters
 *     (as the reference's dense_complex reports (n_viol, max_imag)); the Python
 *     layer maps them onto commdyn/errors.py classes.
 *   - the caller allocates every buffer (reference ownership convention,
 *     SURVEY §8b); kernels accumulate into `out`, they never zero it.
 *   - no exceptions cross the ABI; no hidden global state beyond per-process
 *     function attributes and the last-error string.
 */
#ifndef COMMDYN_CUDA_H
#define COMMDYN_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define CDK_API __attribute__((visibility("default")))
#else
#define CDK_API
#endif

#define CDK_OK 0
#define CDK_NUMERIC 1
#define CDK_INPUT 2
#define CDK_CUDA 3

#define CDK_ABI_VERSION 17
#define CDK_INTRA_PAD 0xFFFFu /* padding entry in intra_col */

/* ------------------------------------------------------------------------ */
/* Kernel-level twins of the reference dispatchers (commdyn/_kernels.py).   */
/* Same array contracts; `pi_over_l` = pi / half_width as the dispatchers   */
/* compute it.  Reductions are fixed-order (deterministic); the pair        */
/* kernels scatter with fp64 atomics (SPEC.md:408 parallel mode, 1e-12).    */
/* ------------------------------------------------------------------------ */

/* replaces order_params_blocks, _kernels.py:68-73 (numba body :34-51).
 * x f64[>= offsets[m_comm]], offsets i64[m_comm+1] -> r c128[m_comm][2p+1]. */
CDK_API int cdk_order_params_blocks(const double *x, const int64_t *offsets, int64_t m_comm, int p,
                            double pi_over_l, double norm, double *r, void *stream);

/* replaces dense_complex, _kernels.py:165-169 (:124-149).  out += ...;
 * guard[0] (int64) += violations, guard[1] (f64 bits) = max(|imag|). */
CDK_API int cdk_dense_complex(const double *x, const int64_t *offsets, int64_t m_comm, const double *tbl,
                      int p, double pi_over_l, double *out, void *guard, void *stream);

/* replaces dense_real, _kernels.py:199-204 (:172-187). */
CDK_API int cdk_dense_real(const double *x, const int64_t *offsets, int64_t m_comm,
                   const double *tbl_cos, const double *tbl_sin, int p, double pi_over_l,
                   double *out, void *stream);

/* replaces pairs_trig, _kernels.py:353-362 (:246-261, :274-283). */
CDK_API int cdk_pairs_trig(const int64_t *iu, const int64_t *iv, int64_t n_pairs, const double *x,
                   double inv_n, const double *d_cos, const double *d_sin, int p,
                   double pi_over_l, const double *sgn, double *out, void *stream);

/* replaces pairs_cs, _kernels.py:372-376 (:297-314).  pos/vel/out f64[n][ndim]. */
CDK_API int cdk_pairs_cs(const int64_t *iu, const int64_t *iv, int64_t n_pairs, const double *pos,
                 const double *vel, int ndim, double inv_n, double amp, double sigma2,
                 double beta, const double *sgn, double *out, void *stream);

/* replaces moments_blocks, _kernels.py:109-113 (:81-93).  w f64[m_comm][p+1]. */
CDK_API int cdk_moments_blocks(const double *x, const int64_t *offsets, int64_t m_comm, int p, double x0,
                       double norm, double *w, void *stream);

/* replaces dense_poly, _kernels.py:231-235 (:207-217). */
CDK_API int cdk_dense_poly(const double *x, const int64_t *offsets, int64_t m_comm, const double *tbl,
                   int p, double scale, double shift, double *out, void *stream);

/* replaces pairs_poly, _kernels.py:365-369 (:264-271, :286-294).  coef f64[p+1]. */
CDK_API int cdk_pairs_poly(const int64_t *iu, const int64_t *iv, int64_t n_pairs, const double *x,
                   double inv_n, const double *coef, int p, double x0, const double *sgn,
                   double *out, void *stream);

/* replaces ho_naive_block, _kernels.py:424-428 (:398-410).  theta, out f64[lam],
 * lam <= 4096 (the literal O(lam^4) oracle; one thread per m). */
CDK_API int cdk_ho_naive_block(const double *theta, int64_t lam, double l1, double l2, double l3,
                       double l4, double *out, void *stream);

/* replaces nn_recurrence, _kernels.py:472-477 (:436-456).  ph, f c128[n]; one
 * thread per anchored segment, same additions in the same order. */
CDK_API int cdk_nn_recurrence(const double *ph, int64_t n, int64_t k, double inv_n,
                      int64_t anchor_every, double *f, void *stream);

/* replaces spin_field_sums, _kernels.py:505-509 (:485-502).  spins, f int64[n];
 * scratch: 8 device bytes. */
CDK_API int cdk_spin_field_sums(const int64_t *spins, int64_t n, int64_t *f, void *scratch,
                        void *stream);

/* Appendix B.1 rank-one coupling (no reference kernel):
 * r = inv_n sum_l beta_l e^{i x_l}, out (complex, interleaved) = alpha_m r e^{-i x_m};
 * scratch: 148 double2 (fixed-order two-level reduction). */
CDK_API int cdk_rank_one(const double *alpha, const double *beta, const double *x, int64_t n,
                 double inv_n, double *out, void *scratch, void *stream);

/* Direct-sum (naive-mode) triadic term of the higher-order Kuramoto model,
 * SPEC.md:463-470 eval_rhs_naive: tri int64[n_tri][3] (the graph's 3-cliques),
 * out[a] += coef sin(theta_b + theta_c - 2 theta_a) and rotations. */
CDK_API int cdk_triangles_sin(const int64_t *tri, int64_t n_tri, const double *theta, double coef,
                      double *out, void *stream);

/* ------------------------------------------------------------------------ */
/* Fused CIA path: Kuramoto RHS (E1 + E2) inside RK4 stages.                */
/* ------------------------------------------------------------------------ */

/* Device form of a Decomposition as a directed CSR without
 * the diagonal, rows in permuted (community-contiguous) order, plus the
 * static work schedule built by the host planner (paper_2203_16657_b200/plan.py).
 *   rows [comm_off[c], comm_off[c+1]) form community c; rows >= comm_off[M]
 *   are the NONE pool (sparse contributions only, SPEC.md evaluator:205).
 *   intra entries (sign -1): uint16 column RELATIVE TO THE ROW'S SEGMENT BASE
 *   (seg_base), each row's run padded to a multiple of 8 with CDK_INTRA_PAD
 *   and ordered by cdk_host_bank_order; inter entries (sign +1, also every
 *   entry of a NONE-pool row): global column (int32).
 *   rblock  = <= 32 consecutive rows of one community (or of the pool);
 *   segment = a run of whole rblocks owned by one CTA, <= seg_rows_cap rows,
 *             whose intra neighbours all lie in the node window
 *             seg_win[2s]..seg_win[2s+1] (staged in shared memory by one bulk
 *             async copy) or, for a community larger than the window
 *             capacity (and the NONE pool), in global memory (w0 == w1).
 * Padding contract (bulk copies move 16-byte units): intra_ptr / inter_ptr
 * readable up to index n_rows + 3, theta / omega up to n_rows + 1. */
#define CDK_SEG_INTER_PHASE 256

typedef struct cdk_graph {
  int64_t n_rows;
  int64_t n_comm;
  const int64_t *comm_off;      /* [n_comm+1] */
  const int64_t *intra_ptr;     /* [n_rows+1 (+3 pad)], multiples of 8 */
  const uint16_t *intra_col;    /* [intra_ptr[n_rows]] */
  const int64_t *inter_ptr;     /* [n_rows+1 (+3 pad)] */
  const int32_t *inter_col;     /* [inter_ptr[n_rows]] */
  int32_t n_rblk;
  int32_t n_seg;
  int32_t n_cta;
  int32_t cta_threads;          /* 1024 */
  int32_t smem_nodes;           /* window capacity (nodes, multiple of 8) */
  int32_t seg_rows_cap;         /* max rows per segment (multiple of 8) */
  const int64_t *rblk_row0;     /* [n_rblk+1]: rblock b = rows [rblk_row0[b], rblk_row0[b+1]) */
  const int32_t *rblk_comm;     /* [n_rblk], -1 = NONE pool */
  const int32_t *comm_rblk_off; /* [n_comm+1] */
  const int32_t *seg_rblk;      /* [n_seg+1] rblock boundaries of segments */
  const int64_t *seg_win;       /* [2*n_seg] staged node window [w0, w1) */
  const int64_t *seg_base;      /* [n_seg] base of the segment's intra columns */
  const int32_t *cta_seg;       /* [n_cta+1] segment boundaries per CTA */
  const int32_t *seg_lpr;       /* [n_seg] lanes per row of the segment's gathers (4|8|16|32),
                                   | CDK_SEG_INTER_PHASE: inter entries in a separate phase */
  /* Communities wider than the window (smem_nodes) but at most 4 windows
   * wide are staged in passes of smem_nodes nodes: each row's intra run is
   * then up to 4 sub-runs (one per pass, each padded to 8, columns of pass p
   * in [p*smem_nodes, (p+1)*smem_nodes) after rebasing) and intra_split[row]
   * packs the sub-run starts in 8-entry chunks from the row start (bits
   * 0-15: pass 1, 16-31: pass 2, 32-47: pass 3).  NULL if no such community. */
  const uint64_t *intra_split;  /* [n_rows] or NULL */
  /* Large graphs (z above the L2 share): inter entries are swept per CTA in
   * inter_blocks column blocks of inter_block_nodes nodes (all rows for
   * block 0, then block 1, ...), so the random z gathers of the whole GPU hit
   * one L2-resident block at a time; inter_split[row] packs the block
   * sub-run starts like intra_split (entries from the row start).  0 = off. */
  int32_t inter_blocks;         /* 0 (off) or 1..4 (1: no column split) */
  int32_t inter_block_nodes;
  const uint64_t *inter_split;  /* [n_rows] (inter_blocks >= 2) or NULL (cdk_inter_split) */
  /* Staged inter indices: segments whose inter run (seg_xr[2s]..seg_xr[2s+1],
   * 4-entry aligned) fits xs_cap int32 entries have it bulk-copied into
   * shared memory with the window, so the row pipeline reads inter columns
   * from shared memory and issues the z gathers two rows ahead.  0 = off. */
  int32_t xs_cap;               /* multiple of 16 */
  int32_t reserved0;            /* 0 */
  const int64_t *seg_xr;        /* [2*n_seg] inter_ptr at the segment's first/last row, or NULL */
  /* Lane-per-row sliced layout ("ELL"; cdk_host_ell_intra).  When ell_off is
   * set the stage kernels run one warp per rblock, lane = row: the rblock's
   * intra chunks are ell_col[(ell_off[b] + 32 c + lane) * 8 .. +8) for
   * c < (ell_off[b+1] - ell_off[b]) / 32 (columns relative to seg_base, as
   * intra_col; staged pads point at zero slots smem_nodes + g), its inter
   * columns xell_col[xell_off[b] + 32 k + lane] for k < (xell_off[b+1] -
   * xell_off[b]) / 32 (global, -1 = none).  cta_threads must then equal
   * cdk_kuramoto_ell_threads(); requires inter_blocks == 0 and no
   * intra_split (communities wider than the window gather from global). */
  const int64_t *ell_off;       /* [n_rblk+1] uint4 units, or NULL */
  const uint16_t *ell_col;
  const int64_t *xell_off;      /* [n_rblk+1] int32 units */
  const int32_t *xell_col;
  /* ELL work units: warps of segment s claim units seg_unit[s] ..
   * seg_unit[s+1]-1 in order (longest first); unit u is rblock ell_units[u]. */
  const int32_t *ell_units;     /* [n_units] */
  const int32_t *seg_unit;      /* [n_seg+1] */
  /* packed ELL unit metadata (or NULL): unit u = int32[8] at ell_meta + 8u:
   * {first chunk (uint4 units), xell start, first row, rblock; chunks, inter
   * entries per lane, rows, ci} with ci the rblock's community minus the
   * segment's first (255: pool) */
  const int32_t *ell_meta;
} cdk_graph;

/* device-side run status (lives inside the workspace) */
typedef struct cdk_run_status {
  int64_t nonfinite;      /* number of node-steps that produced a non-finite phase */
  int64_t first_bad_step; /* first step (1-based, counted from the last prepare) or INT64_MAX */
  int64_t steps_done;     /* steps advanced since the last prepare */
  int64_t reserved;
} cdk_run_status;

/* ------------------------------------------------------------------------ */
/* Fused multi-GPU exchange (community-sharded runs): each rank's */
/* stage epilogue stores its new z rows straight into every peer's z buffer  */
/* over NVLink (P2P stores), then the ranks meet at a system-scope counter   */
/* barrier — replacing the per-stage NCCL all-gather.                        */
/* ------------------------------------------------------------------------ */
typedef struct cdk_peers {
  int32_t n_ranks;             /* 1 = no peers */
  int32_t rank;
  void *const *z0;             /* [n_ranks] device array: every rank's z[0] (own included) */
  void *const *z1;             /* [n_ranks] device array: every rank's z[1] */
  unsigned int *const *bar;    /* [n_ranks] device array: every rank's peer-barrier counter */
  unsigned int bar_base;       /* this rank's counter value before the call (host-tracked) */
  int32_t wait;                /* 1: wait at the barrier; 0: signal only (single-device tests) */
} cdk_peers;

/* cdk_kuramoto_rk4 / cdk_kuramoto_rk4_stage with the fused exchange; the
 * counter advances by n_ranks per stage (bar_base += 4*n_steps*n_ranks) */
CDK_API int cdk_kuramoto_rk4_peers(const cdk_graph *g, double *theta, const double *omega,
                                   double k_over_n, double dt, int64_t n_steps, void *workspace,
                                   const cdk_peers *peers, void *stream);
CDK_API int cdk_kuramoto_rk4_stage_peers(const cdk_graph *g, double *theta, const double *omega,
                                         double k_over_n, double dt, int stage, void *workspace,
                                         const cdk_peers *peers, void *stream);
/* CUDA IPC helpers for the peer tables: export a device pointer (64-byte
 * handle of its allocation + byte offset), import it in another process */
CDK_API int cdk_ipc_export(const void *ptr, void *handle64, uint64_t *offset);
CDK_API int cdk_ipc_import(const void *handle64, uint64_t offset, void **ptr);
CDK_API int cdk_ipc_close(void *ptr, uint64_t offset);

/* threads per CTA of the stage kernels (cdk_graph.cta_threads must match) */
CDK_API int cdk_kuramoto_stage_threads(void);
/* resident stage CTAs per SM the library was built for (the planner launches
 * SMs x this many persistent CTAs and sizes their shared memory to match) */
CDK_API int cdk_kuramoto_stage_ctas_per_sm(void);
/* threads per CTA of the ELL stage kernels (graphs with ell_off set) */
CDK_API int cdk_kuramoto_ell_threads(void);
/* resident ELL CTAs per SM the library was built for */
CDK_API int cdk_kuramoto_ell_ctas_per_sm(void);
/* node capacity of the ELL kernels' shared-memory window (zero slots follow) */
CDK_API int cdk_kuramoto_ell_window_nodes(void);

/* planner calibration (ELL graphs): one RK4 stage-1 launch writing each CTA's
 * cycle count to cycles[n_cta] (device); only the workspace's stage buffers
 * change (run cdk_kuramoto_prepare before a trajectory) */
CDK_API int cdk_kuramoto_stage_cycles(const cdk_graph *g, double *theta, const double *omega,
                                      double k_over_n, double dt, void *workspace,
                                      unsigned long long *cycles, void *stream);

/* bytes of device workspace the fused Kuramoto path needs for graph g */
CDK_API size_t cdk_kuramoto_workspace_bytes(const cdk_graph *g);

/* z = exp(i theta), community sums R, counters and status reset.
 * Must precede cdk_kuramoto_rk4 whenever theta was changed outside it. */
CDK_API int cdk_kuramoto_prepare(const cdk_graph *g, const double *theta, void *workspace, void *stream);

/* One CIA right-hand side (eval_rhs_cia + kuramoto_rhs):
 *   out[i] = omega[i] + k_over_n * Im( (R_c(i) + sum_j s_ij z_j) * conj(z_i) )
 * with k_over_n = K / N (h = K sin, global 1/N).  Runs prepare internally.
 * theta / omega: see the padding contract of cdk_graph. */
CDK_API int cdk_kuramoto_rhs(const cdk_graph *g, const double *theta, const double *omega,
                     double k_over_n, double *out, void *workspace, void *stream);

/* n_steps classical RK4 steps, phases wrapped to (-pi, pi] after
 * each full step.  theta is updated in place; the workspace
 * stays consistent so calls chain without another prepare.  4 kernel launches
 * per step; graph-capturable. */
CDK_API int cdk_kuramoto_rk4(const cdk_graph *g, double *theta, const double *omega, double k_over_n,
                     double dt, int64_t n_steps, void *workspace, void *stream);

/* exactly one RK4 stage kernel (stage 1..4) of the step cdk_kuramoto_rk4 runs;
 * four calls in order == one step without the status bookkeeping.  Used by the
 * bench to time the stage kernel alone. */
CDK_API int cdk_kuramoto_rk4_stage(const cdk_graph *g, double *theta, const double *omega,
                                   double k_over_n, double dt, int stage, void *workspace,
                                   void *stream);

/* byte offsets inside the workspace of [z0, z1, ksum, part0, part1, status]
 * (offsets: [host] int64[7]: z0 z1 ksum part0 part1 status peer_bar); z_s buffers hold exp(i theta) of the stage state,
 * stage k (1..4) reads z[(k-1)&1] and writes z[k&1].  Used by multi-rank
 * drivers to exchange each rank's freshly written rows after a stage. */
CDK_API int cdk_kuramoto_workspace_layout(const cdk_graph *g, int64_t *offsets);

/* add n_steps to the workspace step counter (for drivers calling
 * cdk_kuramoto_rk4_stage directly; keeps BlowUp step numbers right). */
CDK_API int cdk_kuramoto_advance(const cdk_graph *g, void *workspace, int64_t n_steps,
                                 void *stream);

/* n_steps explicit Euler steps, same wrap/blow-up semantics. */
CDK_API int cdk_kuramoto_euler(const cdk_graph *g, double *theta, const double *omega, double k_over_n,
                       double dt, int64_t n_steps, void *workspace, void *stream);

/* copy the workspace's run status to [host] *out (synchronises `stream`). */
CDK_API int cdk_kuramoto_status(const cdk_graph *g, const void *workspace, cdk_run_status *out,
                        void *stream);

/* ------------------------------------------------------------------------ */
/* Higher-order (triadic) Kuramoto on 3-cliques (BASELINE config 3)          */
/*   theta'_i = omega_i + K1/N sum_j a_ij sin(theta_j - theta_i)             */
/*            + K2/N^2 sum_{ordered (j,k): {i,j,k} triangle}                 */
/*                      sin(theta_j + theta_k - 2 theta_i)                   */
/* CIA form: in-community triangles by inclusion-exclusion over the missing  */
/* graph (two CSR passes + missing-graph triangles), spanning triangles      */
/* listed explicitly.  No reference kernel exists for this model (the       */
/* reference's ho_naive_block, _kernels.py:398-428, is the all-to-all block  */
/* sum; it pins the dense part in the tests).                                */
/* ------------------------------------------------------------------------ */
typedef struct cdk_ho_graph {
  int64_t n_rows;
  int32_t n_rblk;
  int32_t n_comm;
  const int64_t *rblk_row0;      /* [n_rblk+1] */
  const int32_t *rblk_comm;      /* [n_rblk], -1 = NONE pool */
  const int32_t *comm_rblk_off;  /* [n_comm+1] */
  const int64_t *miss_ptr;       /* [n_rows+1] proper missing intra edges */
  const int32_t *miss_col;       /* global columns */
  const int64_t *inter_ptr;      /* [n_rows+1] */
  const int32_t *inter_col;      /* global columns */
  const int64_t *tri_ptr;        /* [n_rows+1] triangle pairs per row */
  const int32_t *tri_jk;         /* int32 pairs (j,k); j < 0: spanning triangle, j = -j-1 */
} cdk_ho_graph;

CDK_API size_t cdk_ho_workspace_bytes(const cdk_ho_graph *g);
CDK_API int cdk_ho_prepare(const cdk_ho_graph *g, const double *theta, void *workspace,
                           void *stream);
CDK_API int cdk_ho_rhs(const cdk_ho_graph *g, const double *theta, const double *omega,
                       double k1_over_n, double k2_over_n2, double *out, void *workspace,
                       void *stream);
CDK_API int cdk_ho_rk4(const cdk_ho_graph *g, double *theta, const double *omega,
                       double k1_over_n, double k2_over_n2, double dt, int64_t n_steps,
                       void *workspace, void *stream);
CDK_API int cdk_ho_status(const cdk_ho_graph *g, const void *workspace, cdk_run_status *out,
                          void *stream);

/* ------------------------------------------------------------------------ */
/* Higher-harmonics Kuramoto: coupling  */
/*   h(x) = sum_{a=0..p} d_cos[a] cos(a x) + d_sin[a] sin(a x), p <= 8,      */
/* CIA with 2p+1 Fourier modes in E1 (replaces order_params_blocks +         */
/* dense_complex/dense_real with p harmonics, _kernels.py:34-73,124-204) and  */
/* the exact h on the sparse correction (replaces pairs_trig,                 */
/* _kernels.py:246-283,353-362), fused into RK4 (reduce + stage per stage).   */
/* ------------------------------------------------------------------------ */
typedef struct cdk_hh_graph {
  int64_t n_rows;
  int32_t n_rblk;
  int32_t n_comm;
  int32_t p;                     /* harmonics, 1..8 */
  int32_t reserved;
  const int64_t *rblk_row0;      /* [n_rblk+1] */
  const int32_t *rblk_comm;      /* [n_rblk], -1 = NONE pool */
  const int32_t *comm_rblk_off;  /* [n_comm+1] */
  const int64_t *comm_off;       /* [n_comm+1] community row offsets */
  const int64_t *miss_ptr;       /* [n_rows+1] proper missing intra edges (sign -1) */
  const int32_t *miss_col;
  const int64_t *inter_ptr;      /* [n_rows+1] inter / pool edges (sign +1) */
  const int32_t *inter_col;
  const double *d_cos;           /* [p+1] (coupling constant folded in) */
  const double *d_sin;           /* [p+1] */
} cdk_hh_graph;

CDK_API size_t cdk_hh_workspace_bytes(const cdk_hh_graph *g);
CDK_API int cdk_hh_prepare(const cdk_hh_graph *g, const double *theta, void *workspace,
                           void *stream);
CDK_API int cdk_hh_rhs(const cdk_hh_graph *g, const double *theta, const double *omega,
                       double inv_n, double *out, void *workspace, void *stream);
CDK_API int cdk_hh_rk4(const cdk_hh_graph *g, double *theta, const double *omega, double inv_n,
                       double dt, int64_t n_steps, void *workspace, void *stream);
CDK_API int cdk_hh_status(const cdk_hh_graph *g, const void *workspace, cdk_run_status *out,
                          void *stream);

/* ------------------------------------------------------------------------ */
/* Cucker-Smale flocking, 2-D (BASELINE config 4)                            */
/*   s' = v,  v'_m = inv_n sum_l a_ml eta(|s_l - s_m|^2)(v_l - v_m),         */
/*   eta(y) = K / (sigma2 + y)^beta.                                          */
/* CIA with a per-community degree-8 polynomial of eta in the scaled squared */
/* distance (host P2 fit, paper_2203_16657_b200/cs.py): bivariate moments up */
/* to degree 16, contraction T_c (153 x 153), bivariate evaluation per node, */
/* EXACT sparse correction (replaces pairs_cs, _kernels.py:297-314, on S).   */
/* ------------------------------------------------------------------------ */
typedef struct cdk_cs_graph {
  int64_t n_rows;
  int64_t n_comm;
  int32_t n_rblk;
  int32_t max_comm;             /* largest community (moments pass: CTAs per community) */
  const int64_t *comm_off;      /* [n_comm+1] */
  const int64_t *rblk_row0;     /* [n_rblk+1] */
  const int32_t *rblk_comm;     /* [n_rblk] */
  const int64_t *miss_ptr;      /* [n_rows+1] missing intra edges (sign -1) */
  const int32_t *miss_col;
  const int64_t *inter_ptr;     /* [n_rows+1] inter / NONE-pool edges (sign +1) */
  const int32_t *inter_col;
  const double *mu;             /* [n_comm][2] community centres */
  const double *inv_L;          /* [n_comm] 1 / scale */
  /* contraction T_c[r][s] = chat_c[k(r,s)] * t_coef: one shared sparse
   * pattern (1365 nonzeros of 153 x 153, CSR by r) + 9 fit coefficients per
   * community (the dense per-community tensors are never formed on the device) */
  const double *chat;           /* [n_comm][9] P2 fit coefficients */
  const int32_t *t_ptr;         /* [154] */
  const int32_t *t_col;         /* s | k << 8 */
  const double *t_coef;         /* binomial coefficient x sign */
} cdk_cs_graph;

CDK_API size_t cdk_cs_workspace_bytes(const cdk_cs_graph *g);
/* reset the run status (domain-violation and blow-up counters) */
CDK_API int cdk_cs_prepare(const cdk_cs_graph *g, void *workspace, void *stream);
/* out (double[n][2]) = v' at (pos, vel) (double[n][2]); status.reserved counts
 * nodes outside the expansion domain (DomainViolationError). */
CDK_API int cdk_cs_rhs(const cdk_cs_graph *g, const double *pos, const double *vel, double K,
                       double sigma2, double beta, double inv_n, double *out, void *workspace,
                       void *stream);
/* n_steps RK4 steps of (pos, vel) in place */
CDK_API int cdk_cs_rk4(const cdk_cs_graph *g, double *pos, double *vel, double K, double sigma2,
                       double beta, double inv_n, double dt, int64_t n_steps, void *workspace,
                       void *stream);
CDK_API int cdk_cs_status(const cdk_cs_graph *g, const void *workspace, cdk_run_status *out,
                          void *stream);

/* ------------------------------------------------------------------------ */
/* Device-side deterministic generator (BASELINE config 5) */
/* Produces the stage kernel's CSR directly on the device (counter-based     */
/* hashes: identical on any GPU count, any row regenerable).                 */
/* ------------------------------------------------------------------------ */
typedef struct cdk_gen_params {
  uint64_t seed;
  int64_t n_rows;
  int64_t n_comm;
  const int64_t *comm_off;   /* [n_comm+1] device */
  const double *node_cdf;    /* [n_rows] device, cumulative endpoint weights, last = 1 */
  int64_t n_inter_edges;     /* sampled inter edges (before drops / dedupe) */
  uint32_t miss_thr;         /* intra pair missing iff hash < miss_thr (q * 2^32) */
  uint32_t pass_nodes;       /* window capacity of the stage kernel (cdk_graph.smem_nodes):
                                rows of communities wider than it get per-pass sub-runs */
  int64_t row_lo, row_hi;    /* rows generated: [row_lo, row_hi) (a rank's shard; other
                                rows stay empty, columns stay global) */
} cdk_gen_params;

/* intra: per-row padded run lengths (int64[n_rows], sub-runs per pass each
 * padded to 8), raw missing-partner counts (int64[n_rows]) and the packed
 * sub-run starts (uint64[n_rows], see cdk_graph.intra_split); then, with ptr =
 * the prefix sum of the padded lengths, the uint16 community-local columns */
CDK_API int cdk_gen_intra_count(const cdk_gen_params *p, int64_t *padded, int64_t *raw,
                                uint64_t *split, void *stream);
CDK_API int cdk_gen_intra_fill(const cdk_gen_params *p, const int64_t *ptr,
                               const uint64_t *split, uint16_t *col, void *stream);
/* inter: counts (atomic int64[n_rows], zeroed by the caller), scatter via a
 * cursor (= row starts), per-row sort + dedupe (writes unique counts), compact */
CDK_API int cdk_gen_inter_count(const cdk_gen_params *p, int64_t *cnt, void *stream);
CDK_API int cdk_gen_inter_fill(const cdk_gen_params *p, int64_t *cursor, int32_t *col,
                               void *stream);
CDK_API int cdk_gen_inter_sort(int64_t n_rows, const int64_t *ptr, int32_t *col, int64_t *uniq,
                               void *stream);
CDK_API int cdk_gen_inter_compact(int64_t n_rows, const int64_t *ptr_raw, const int64_t *ptr_new,
                                  const int32_t *col_raw, int32_t *col_new, void *stream);
/* add delta[row] to every non-padding intra column (segment-window rebasing) */
CDK_API int cdk_gen_rebase(int64_t n_rows, const int64_t *ptr, const int32_t *delta,
                           uint16_t *col, void *stream);
/* device twin of cdk_host_bank_order, out of place (src != dst): every row's
 * intra run, or each pass sub-run when split != NULL, reordered for
 * bank-conflict-free window gathers */
CDK_API int cdk_bank_order(int64_t n_rows, const int64_t *ptr, const uint64_t *split,
                           const uint16_t *src, uint16_t *dst, int pad_bank, void *stream);
/* cdk_graph.inter_split of a row-sorted inter CSR (device arrays): block q
 * sub-run = columns in [q*block_nodes, (q+1)*block_nodes); rows longer than
 * 65535 entries are rejected */
CDK_API int cdk_inter_split(int64_t n_rows, const int64_t *ptr, const int32_t *col, int blocks,
                            int block_nodes, uint64_t *split, void *stream);

/* ------------------------------------------------------------------------ */
/* host-side planning (no device needed)                                    */
/* ------------------------------------------------------------------------ */

/* [host] reorder each row's intra run (ptr[r]..ptr[r+1], multiples of 8) so
 * the 16-byte shared-memory gathers of one 8-lane row group hit distinct bank
 * groups (column mod 8); pads (pad_value) count as bank pad_bank. */
CDK_API int cdk_host_bank_order(uint16_t *cols, const int64_t *ptr, int64_t n_rows,
                                int32_t pad_value, int32_t pad_bank);

/* [host] ELL intra layout (cdk_graph.ell_off/ell_col): per rblock, the rows'
 * runs (ptr/cols as intra_ptr/intra_col, pads skipped) scheduled so each
 * quarter-warp step hits 8 distinct bank groups.  staged[b] != 0: pads point
 * at zero slot zero_slot + bank group; else CDK_INTRA_PAD.  Bank group of a
 * column v of rblock b: (v + bank_shift[b]) mod 8 (NULL: 0).  ell == NULL:
 * writes ell_off only (sizes); then call again with ell sized
 * 8 * ell_off[n_rblk] uint16. */
CDK_API int cdk_host_ell_intra(const int64_t *rblk_row0, int32_t n_rblk, const int64_t *ptr,
                               const uint16_t *cols, const uint8_t *staged,
                               const uint8_t *bank_shift, int32_t zero_slot, int64_t *ell_off,
                               uint16_t *ell);

/* [host] triangles {i<j<k} of a symmetric CSR (sorted global columns, no
 * self loops); writes <= cap int32 triples to out (NULL ok), returns the count
 * (-1 on bad input).  Used to enumerate the missing-edge-graph triangles of
 * the higher-order (triadic) model. */
CDK_API int64_t cdk_host_triangles(const int64_t *ptr, const int32_t *cols, int64_t n,
                                   int32_t *out, int64_t cap);

/* ------------------------------------------------------------------------ */
/* misc                                                                      */
/* ------------------------------------------------------------------------ */
CDK_API int cdk_abi_version(void);
CDK_API const char *cdk_last_error(void);
/* number of kernel launches issued by this library since load (for the bench's gpu_launches) */
CDK_API int64_t cdk_launch_count(void);
/* profiling builds (-DCDK_PROFILE) only: per-CTA phase cycles of the latest
 * stage launch go to prof (device, 4 * n_cta uint64); no-op otherwise */
CDK_API void cdk_debug_set_profile_buffer(void *prof);
/* max dynamic shared memory per block (opt-in) on the current device */
CDK_API int cdk_max_smem_optin(void);

#ifdef __cplusplus
}
#endif
#endif /* COMMDYN_CUDA_H */
