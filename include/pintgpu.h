/*
 * pintgpu.h -- C ABI of the B200-native batched-Phi MGRIT hot path.
 *
 * The reference (arxiv 1912.03106, package `pintmg`, pure Python) has one
 * plug-in boundary on this path: the problem object the MGRIT engine calls,
 *
 *   problem.step(u_prev, t_prev, t_next, spatial_level, guess, smooth)
 *       -> (BlockState, StepDiagnostics)         problems.py:1-17, :138-146
 *   problem.spatial.restrict_state / prolong_error      spatial.py:64-84
 *   problem.initial_state / loss_weights / n_scalars    problems.py:73-108
 *
 * called from MgritSolver._step (mgrit.py:361-366) and the sweeps around it
 * (mgrit.py:368-598).  Each entry point below replaces one of those calls,
 * batched over the C-intervals of a level (one column per interval):
 *
 *   pg_phi_batch      <- problem.step                  problems.py:138-146
 *                        (nonlinear: problems.py:201-244)
 *   pg_restrict       <- spatial.restrict_state        spatial.py:64-71
 *   pg_prolong_add    <- spatial.prolong_error + c_store += e
 *                                                      spatial.py:73-84,
 *                                                      mgrit.py:562-571
 *   pg_c_residual     <- res = step(u_{c-1}) - u_c (+g_c); |res|^2; joule
 *                                                      mgrit.py:416-420,
 *                                                      :585-596,
 *                                                      problems.py:53-56
 *   pg_fas_rhs        <- rhs = kept - step_c(kept_{j-1}) + R(res)
 *                                                      mgrit.py:421-426
 *
 * Conventions: every array argument is a DEVICE pointer, states are
 * row-major [B][n] fp64 (one contiguous state per column), every call is
 * asynchronous and ordered on `stream` (a cudaStream_t passed as void*), and
 * outputs never alias inputs unless stated.  Return codes are PG_OK or a
 * PG_E* value; pg_last_error() gives the message.  There is no CPU path: a
 * context cannot be created without a CUDA device.
 */
#ifndef PINTGPU_H
#define PINTGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PG_OK       0
#define PG_EINVAL   1   /* bad argument (ValueError on the Python side)   */
#define PG_ECUDA    2   /* CUDA runtime failure                            */
#define PG_ENEWTON  3   /* NewtonConvergenceError, errors.py:4-10          */
#define PG_ENOCONV  4   /* inner PCG hit max_iters above tolerance         */

typedef struct pg_ctx pg_ctx;

/* One spatial grid (reference: one entry of SpatialHierarchy.sizes).
 * CSR of the union pattern of the sigma-mass M and the stiffness K (for a
 * nonlinear level K holds only the linear, non-iron elements).  All arrays
 * here are HOST pointers; pg_add_level copies them to the device. */
typedef struct pg_level_desc {
    int32_t n;                  /* unknowns (interior nodes)               */
    int32_t nnz;
    const int32_t* row_ptr;     /* [n+1]                                   */
    const int32_t* col_idx;     /* [nnz], sorted per row, diagonal present */
    const double*  m_val;       /* [nnz]  M_sigma                          */
    const double*  k_val;       /* [nnz]  K_nu (linear part)               */
    int32_t n_src;              /* source phases                           */
    const double*  shapes;      /* [n_src][n] load vectors                 */
    const double*  weights;     /* [n] Joule-loss weights (lumped M_sigma) */
    /* structured-grid geometry for the transfer kernels: side = N_g - 1 */
    int32_t side;
    /* nonlinear iron elements (n_elem = 0 for linear levels) */
    int32_t n_elem;
    const int32_t* elem_dof;    /* [n_elem][3], -1 = Dirichlet vertex      */
    const double*  elem_geo;    /* [n_elem][7]: b0 b1 b2 c0 c1 c2 area     */
    const int32_t* node_elem_ptr; /* [n+1] node -> incident iron elements  */
    const int32_t* node_elem;   /* [..] elem * 4 + local vertex            */
    /* nonlinear levels, inner = PG_INNER_CHOLESKY: stiffness of the
     * linearised operator (iron at nu(|B| = 0)) on the CSR pattern; its
     * banded-Cholesky factor preconditions the Newton systems. Nullable. */
    const double*  k_pre_val;   /* [nnz]                                   */
} pg_level_desc;

/* Inner-solver and material options (NewtonOptions, problems.py:39-50;
 * BrauerCurve, problems.py:149-168, scaled by nu0 for the 2D model). */
#define PG_INNER_PCG       0   /* batched Jacobi-PCG                       */
#define PG_INNER_CHOLESKY  1   /* banded Cholesky per distinct dt (the
                                  reference's cholesky_banded path)        */

typedef struct pg_solver_opts {
    int32_t inner;              /* PG_INNER_PCG | PG_INNER_CHOLESKY (linear) */
    double  rtol;               /* PCG: |r| <= rtol |b| per column         */
    int32_t max_iters;          /* PCG iteration cap                       */
    int32_t check_every;        /* host convergence poll interval (iters)  */
    double  newton_tol;         /* |F| <= tol * max(|rhs|, 1e-300)         */
    int32_t newton_max_iters;
    double  damping;
    int32_t max_halvings;
    double  nu0, k1, k2, k3;    /* nu = nu0 (k1 exp(k2 s^2) + k3) on iron  */
    double  dt_merge_rtol;      /* banded Cholesky: reuse the factor of an
                                   existing 1/dt within this relative
                                   distance (0 = the reference's bitwise
                                   (level, float(dt)) cache key)           */
    int32_t strips;             /* banded Cholesky on structured grids of
                                   255^2 and more, batches that fill the GPU:
                                   1 = strip solve (strips + separator Schur
                                   complement: the same direct solve with
                                   ~2.7x fewer flops, agrees with the
                                   natural-order solve to rounding), 0 = the
                                   natural-order band solve only (the
                                   reference's dpbtrs ordering)            */
} pg_solver_opts;

/* Per-call statistics (host struct). */
typedef struct pg_phi_stats {
    int64_t columns;            /* columns solved                          */
    int64_t column_iters;       /* sum over columns of PCG iterations      */
    int64_t batch_iters;        /* max over columns (batched iterations)   */
    int64_t newton_iters;       /* sum over columns of Newton iterations   */
    int64_t failed;             /* columns that hit max_iters              */
    int64_t launches;           /* kernels launched by the call            */
} pg_phi_stats;

int  pg_create(pg_ctx** out, int device);
void pg_destroy(pg_ctx* ctx);
const char* pg_last_error(pg_ctx* ctx);

/* Returns the new level index (0, 1, ... in call order) or -1. */
int  pg_add_level(pg_ctx* ctx, const pg_level_desc* desc);
int  pg_set_options(pg_ctx* ctx, const pg_solver_opts* opts);

/* Batched implicit-Euler step.  Column b solves
 *   (inv_dt[b] M + K(u)) u_out[b] = inv_dt[b] M u_prev[b] + sum_s src[b][s] shape_s
 * starting from guess[b] (NULL = u_prev), then adds g[g_idx[b]] when g is
 * non-NULL and g_idx[b] >= 0.  inv_dt: [B]; src: [B][n_src]; g: [*][n];
 * g_idx: [B] int32.  u_out must not alias u_prev or guess.
 * Linear levels: banded Cholesky (PG_INNER_CHOLESKY) or Jacobi-PCG.  Levels
 * with iron elements: damped Newton (problems.py:201-244), inner solve CG
 * preconditioned by the banded-Cholesky factor of the linearised operator
 * (PG_INNER_CHOLESKY, needs k_pre_val) or Jacobi-PCG; on failure returns
 * PG_ENEWTON and pg_newton_failure() reports column and iteration count. */
int  pg_phi_batch(pg_ctx* ctx, int level, int B,
                  const double* u_prev, const double* guess,
                  const double* inv_dt, const double* src,
                  double* u_out, const double* g, const int32_t* g_idx,
                  void* stream);

/* Same, with an optional HOST copy of inv_dt (identical values): the banded-
 * Cholesky path then needs no device->host read to pick its per-dt factors,
 * and caches the column grouping per distinct inv_dt pattern. */
int  pg_phi_batch_h(pg_ctx* ctx, int level, int B,
                    const double* u_prev, const double* guess,
                    const double* inv_dt, const double* inv_dt_host, const double* src,
                    double* u_out, const double* g, const int32_t* g_idx,
                    void* stream);

/* Statistics of the most recent pg_phi_batch (synchronises the stream). */
/* Banded-Cholesky levels: factor every not-yet-cached 1/dt of the list in
 * one launch (one CTA per factor).  The engine calls it at setup with all
 * 1/dt of the levels on this grid, so factorisations run in parallel instead
 * of one launch per first-use.  No-op for Jacobi-PCG. */
int  pg_prefactor(pg_ctx* ctx, int level, int n, const double* inv_dt_host, void* stream);

int  pg_last_stats(pg_ctx* ctx, pg_phi_stats* out);
/* Cumulative statistics since the context was created / reset. */
int  pg_total_stats(pg_ctx* ctx, pg_phi_stats* out, int reset);
int  pg_newton_failure(pg_ctx* ctx, int* column, int* iterations);

/* out[b] = R(in[b]); fine level -> fine+1.  mode 0 = injection,
 * 1 = full weighting. */
int  pg_restrict(pg_ctx* ctx, int fine_level, int B, const double* in,
                 double* out, int mode, void* stream);

/* coarse level -> coarse-1:  out[out_idx[b]] = beta * out[out_idx[b]] + P(in[b])
 * (beta = 1: correction add, beta = 0: injection of values).  mode 0 =
 * bilinear, 1 = P1 nodal.  out_idx may be NULL (identity). */
int  pg_prolong_add(pg_ctx* ctx, int coarse_level, int B, const double* in,
                    double* out, const int32_t* out_idx, double beta,
                    int mode, void* stream);

/* res[b] = prop[b] - c[c_idx[b]] (+ g[g_idx[b]]);  sumsq[b] = |res[b]|^2;
 * if last_f != NULL: loss[b] = sum_i w_i ((c_i - last_f_i) * inv_dt[b])^2.
 * res may be NULL (norm/loss only).  c_idx / g_idx may be NULL (identity /
 * no g).  */
int  pg_c_residual(pg_ctx* ctx, int level, int B, const double* prop,
                   const double* c, const int32_t* c_idx,
                   const double* g, const int32_t* g_idx,
                   double* res, double* sumsq,
                   const double* last_f, const double* inv_dt, double* loss,
                   void* stream);

/* Coarse FAS right-hand side on level `coarse` (fine = coarse-1 when
 * coarsen != 0, same grid otherwise):
 *   rhs[b] = kept[b] - cprop[b] + R(res[b]).  */
int  pg_fas_rhs(pg_ctx* ctx, int coarse, int coarsen, int B,
                const double* kept, const double* cprop, const double* res,
                double* rhs, int mode, void* stream);

/* Row algebra of the level stores the engine keeps on the device (rows of n
 * doubles; replaces the reference's BlockState add / subtract / copy loops,
 * state.py:44-72, as used by mgrit.py:447-450, :483-490, :545-571):
 *   out[ro(b)] = a[ra(b)]                       (c == NULL)
 *   out[ro(b)] = a[ra(b)] + sign * c[rc(b)]     (sign = +1 or -1)
 * for b = 0..B-1, row selectors r(b) = idx ? idx[b] : start + b * step
 * (idx: device int32 [B] or NULL).  out may alias a or c row for row. */
int  pg_rows_axpby(pg_ctx* ctx, int n, int B,
                   const double* a, const int32_t* a_idx, int a_start, int a_step,
                   const double* c, const int32_t* c_idx, int c_start, int c_step, int sign,
                   double* out, const int32_t* o_idx, int o_start, int o_step, void* stream);

/* Number of kernels this context has launched (for the bench). */
int64_t pg_launch_count(pg_ctx* ctx);

/* Kernel-level timing (CUDA events around every launch of the hot kernels:
 * [0] k_sdir, [1] k_supd (streamed PCG, read back at the convergence
 * polls), [2] k_band_solve (forward + backward banded solves).
 * alg_bytes: algorithmic HBM bytes (32 n per column for k_sdir, 48 n for
 * k_supd; Y in/out + distinct factors for the band solves); alg_flops:
 * 4 np (W + 32) per column for the band solves. */
typedef struct pg_kernel_profile {
    char    name[16];
    double  total_ms;
    int64_t launches;
    double  alg_bytes;
    double  alg_flops;
    int64_t column_iters;
} pg_kernel_profile;
/* Profiling (dev / bench): with profiling on every kernel of a Phi call is
 * bracketed by CUDA events on the launching stream (and the call syncs).
 * pg_profile_read fills up to n of the PG_PROFILE_KINDS entries, in order:
 * k_sdir, k_supd (Jacobi-PCG), k_band_solve (= chains + SPIKE recombination),
 * band_chain_fwd, band_chain_bwd (column groups of 8 / 16), band_rhs,
 * spike_border, spike_fix (strip calls: the separator coupling + GEMM),
 * band_scatter (strip calls: the gathers and the scatter), chain32_fwd,
 * chain32_bwd (the chains of GPU-filling batches: k_band_rb<32, ...>, or
 * k_band_wcol on the 8-strip systems; the 16-strip chains of smaller batches
 * count as band_chain_*);
 * alg_flops / alg_bytes are the algorithmic work (the
 * reference's dpbtrs: 2 n w flops per direction and column). */
#define PG_PROFILE_KINDS 11
int  pg_profile(pg_ctx* ctx, int on);
int  pg_profile_read(pg_ctx* ctx, pg_kernel_profile* out, int n, int reset);

#ifdef __cplusplus
}
#endif
#endif /* PINTGPU_H */
