/*
 * phipm.h — C ABI of libphipm.so, a B200 (sm_100a) implementation of the hot path of
 * J. Niesen & W. M. Wright, "Algorithm 919: A Krylov subspace algorithm for evaluating the
 * phi-functions appearing in exponential integrators" (arXiv:0907.4631; PAPER.md).
 *
 * phipm evaluates  w(t) = phi_0(tA) u_0 + sum_{k=1..p} t^k phi_k(tA) u_k   (Eq. lincomb2,
 * PAPER.md P:485-489), i.e. the solution at t of u' = A u + sum_{j<p} s^j/j! u_{j+1}, u(0) = u_0
 * (Eq. phide), for a large sparse A given as CSR or as a 3/5/7-point stencil, by the
 * adaptive Krylov time stepping of Algorithms 3-4.
 *
 * Conventions for every entry point:
 *   - Pointers documented "device" must be CUDA device pointers of the current device (e.g. from
 *     torch); "host" pointers are ordinary CPU memory.  The library never frees, keeps or
 *     retains caller memory after a call returns.
 *   - All fp64.  Vectors are contiguous, length n.  Small dense matrices are column-major.
 *   - All GPU work is enqueued on the stream given to phipm_create (a cudaStream_t passed as
 *     void*; NULL = legacy default stream).  Calls are host-blocking: they return after the
 *     result is complete (the controller reads a few scalars back every attempt).
 *   - Errors are returned as status codes (PHIPM_*); nothing aborts or throws across the ABI.
 *     phipm_strerror() gives a message; phipm_last_error() a detailed one for the context.
 *   - One context per host thread; a context runs one call at a time.
 */
#ifndef PHIPM_H
#define PHIPM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define PHIPM_OK          0  /* success */
#define PHIPM_EINVAL      1  /* bad argument: null pointer, n <= 0, p < 0 or p > p_max, tol <= 0, t < 0,
                                m_init not in [1, m_max], n > n_max, malformed descriptor */
#define PHIPM_ENOMEM      2  /* device or pinned allocation failed */
#define PHIPM_ECUDA       3  /* CUDA launch / runtime error (message in phipm_last_error) */
#define PHIPM_ESTEP       4  /* step size underflow (tau < 1e-15 t) or > 100 attempts in one step;
                                w holds u(t_reached), stats->t_reached < t */
#define PHIPM_ENONFINITE  5  /* NaN/Inf in beta, H, exp(Hhat) or the error estimate */
#define PHIPM_ESINGULAR   6  /* singular Pade denominator in the small exponential */

typedef struct phipm_ctx phipm_ctx;

/* Sparse matrix in CSR form, DEVICE arrays.  row_ptr[n+1], col[nnz] (int32, strictly ascending
 * within a row, in [0,n)), val[nnz].  nnz = row_ptr[n] - row_ptr[0] < 2^31. */
typedef struct {
    int64_t n, nnz;
    const int32_t *row_ptr;
    const int32_t *col;
    const double *val;
} phipm_csr;

/* Constant-coefficient stencil on an nx*ny*nz grid with zero Dirichlet data (neighbours outside
 * the grid are 0).  Row r = i + nx*(j + ny*k).  dim in {1,2,3}: dim=1 uses c_center,c_xm,c_xp
 * (ny = nz = 1); dim=2 adds c_ym,c_yp (nz = 1); dim=3 adds c_zm,c_zp.  Unused coefficients are
 * ignored.  (A 3-point 1-D, 5-point 2-D or 7-point 3-D operator; BASELINE.json configs c1-c4.)
 * points = 9 (dim = 2 only, e.g. the 9-point Laplacian of the paper's gr_30_30,
 * P:1224-1232) adds the four corner neighbours c_xmym (i-1, j-1), c_xpym (i+1, j-1), c_xmyp
 * (i-1, j+1), c_xpyp (i+1, j+1); any other value of points selects the 2 dim + 1 point form. */
typedef struct {
    int dim, nx, ny, nz;
    double c_center, c_xm, c_xp, c_ym, c_yp, c_zm, c_zp;
    double c_xmym, c_xpym, c_xmyp, c_xpyp;
    int points;
} phipm_stencil;

/* Orthogonalisation of the Arnoldi step (ignored for symmetric = 1, which runs Lanczos, Alg. 2) */
#define PHIPM_ORTH_CGS   0   /* one classical Gram-Schmidt pass (equal to Alg. 1's MGS in exact
                                arithmetic; the default) */
#define PHIPM_ORTH_CGS2  1   /* CGS with one full re-orthogonalisation pass every step */

/* Method for exp(Hhat) (Eq. 8: scaling and squaring).  Both reach unit-
 * roundoff backward error; the oracle always uses Pade-13. */
#define PHIPM_EXPM_TAYLOR  0 /* degree 8/12/16 Taylor by Paterson-Stockmeyer, all products on the
                                fp64 tensor cores, squarings from ||A^k||^(1/k) (the default) */
#define PHIPM_EXPM_PADE13  1 /* the paper's [13/13] Pade, theta_13 = 5.37, with a pivoted
                                Gauss-Jordan solve (V - U) X = (V + U) */
#define PHIPM_EXPM_CHEBYSHEV 2 /* symmetric H only (Lanczos; "compute the phi-
                                function of H_m directly ... exploit the fact that H_m is symmetric"):
                                phi_p(tau T)e1 and phi_{p+1}(tau T)e1 by one Chebyshev expansion on the
                                Gershgorin interval of tau T, no augmented matrix.
                                Arnoldi solves with this method use TAYLOR; an interval too wide for
                                512 Chebyshev points (10.5 sqrt(r) + 32 > 512, r the half-width) falls
                                back to TAYLOR for that attempt.  phipm_phi_pair reads the lower
                                band of H and assumes H symmetric tridiagonal. */

/* Options.  Defaults (phipm_default_opts): tol 1e-7, m_init 10 (Alg. 3),
 * m_max 100, symmetric 0, fixed_m 0, eq6_variant 0, orth CGS, profile 0, expm_method Taylor. */
typedef struct {
    double tol;          /* Tol of Eq. (taunew) P:588-593 (absolute 2-norm error per unit time) */
    int m_init;          /* initial Krylov dimension m (Alg. 3) */
    int m_max;           /* cap on m (and on m <= n) */
    int symmetric;       /* 1: Lanczos (A symmetric), 0: Arnoldi */
    int fixed_m;         /* 1: "phip" mode: m fixed to m_init, only tau adapts */
    int eq6_variant;     /* 0: Eq. (6) as printed; 1: log(eps/eps_old)/log(tau/tau_old) - 1 (R13) */
    int orth;            /* PHIPM_ORTH_* */
    int profile;         /* 1: time every kernel class with CUDA events (phipm_get_profile);
                            2: also record every launch (phipm_get_trace) */
    int expm_method;     /* PHIPM_EXPM_* */
} phipm_opts;

/* Statistics (the paper's stats(1..4), plus the Krylov dimension). */
typedef struct {
    int32_t nsteps;      /* accepted time steps */
    int32_t nreject;     /* rejected attempts */
    int32_t nspmv;       /* products of A with a vector actually executed */
    int32_t nexpm;       /* small matrix exponentials */
    int32_t m_last;      /* m of the last accepted attempt */
    int32_t m_peak;      /* largest m attempted */
    double t_reached;    /* time reached (== t on success) */
} phipm_stats;

/* Per-kernel-class device time (CUDA events on the context stream) and algorithmic bytes, summed
 * over the calls made since the last phipm_reset_profile; valid when opts.profile = 1. */
typedef struct {
    double ms_spmv_dot;    /* fused SpMV (+ w-recurrence epilogue / Gram-Schmidt dot products) */
    double ms_orth;        /* fused orthogonalisation update + norm (and re-orth passes) */
    double ms_expm;        /* single-CTA augmented exponential + error estimate */
    double ms_combine;     /* w / u assembly (Eq. step) */
    double ms_other;       /* norms, copies */
    double bytes_spmv_dot; /* algorithmic bytes */
    double bytes_orth;
    double bytes_combine;
    int64_t launches;      /* kernels launched */
    int64_t n_spmv_dot, n_orth, n_expm, n_combine;
    double bytes_other;    /* algorithmic bytes of the setup passes (CSR analysis: 12 nnz + 4(n+1)) */
} phipm_profile;

/* One traced kernel launch (opts.profile = 2). */
typedef struct {
    int32_t cls;           /* 0 spmv_dot, 1 orth, 2 expm, 3 combine, 4 other */
    int32_t ncols;         /* dot columns (spmv) or streamed vectors (axpy); K for expm */
    double bytes;          /* algorithmic bytes */
    double us;             /* device time (CUDA events) */
} phipm_trace_rec;

/* One attempt of the controller (Alg. 3's inner loop), recorded by every solve of the context:
 * the step start t_k, the attempt's tau and m, the Krylov dimension mu used, omega and eps of
 * Eq. (taunew) / (errest), beta = ||w_p||_2, ||H_mu||_1, accepted (omega <= 1.2) and the branch the
 * controller took (1: tau changed, 2: m changed).  The fields are those of a test trajectory record. */
typedef struct {
    double t_k, tau, omega, eps, normH1, beta;
    int32_t m, mu, accepted, branch;
} phipm_attempt;

/* Attempts of the context's last solve: copies min(max, count) records to out (HOST) and sets
 * *count to the number the solve made (only the first 65536 are kept). */
int phipm_get_attempts(const phipm_ctx *ctx, phipm_attempt *out, int max, int *count);

/* Measurement stamps (environment PHIPM_EXPM_CLOCKS=1 at phipm_create, else zeros): copies 16 words to
 * out16 (HOST): the phase cycles of the last exponential kernel, or of the last device-driven small
 * solve (setup, w-recurrence + seed, extensions, exponential, controller, combine in words 0..5). */
int phipm_get_clocks(const phipm_ctx *ctx, long long *out16);

/* Which kernel path ran the last Krylov extension enqueued on this context (a solve's last extension, or
 * phipm_krylov_*): for tests and measurement scripts that must know a path was taken, not fallen back from.
 * A device-driven small solve (PHIPM_OPT_DEVSOLVE) runs its extensions inside its own kernel and leaves
 * the value unchanged. */
#define PHIPM_PATH_NONE          0   /* no extension yet */
#define PHIPM_PATH_TWO_KERNEL    1   /* fused SpMV + dots, then update + norm, per step (stream.cuh) */
#define PHIPM_PATH_SINGLE_CTA    2   /* n <= 8192: one single-CTA kernel (small.cuh) */
#define PHIPM_PATH_CLUSTER       3   /* Lanczos on one thread-block cluster (persist_cl.cuh) */
#define PHIPM_PATH_PERSIST_SMEM  4   /* persistent cooperative kernel, y in shared memory (persist.cuh) */
#define PHIPM_PATH_PERSIST_TMEM  5   /* persistent Lanczos, y / v~ in tensor memory (persist_tm.cuh) */
#define PHIPM_PATH_BRICK         6   /* persistent Lanczos on TMA-staged 3-D bricks (persist_brick.cuh) */
int phipm_krylov_path(const phipm_ctx *ctx);
/* The same for the last w-recurrence (Eq. wrecurrence) of a solve: PHIPM_PATH_BRICK (wrec_brick_kernel),
 * PHIPM_PATH_PERSIST_SMEM (wrec_persist_kernel, contiguous row ranges) or PHIPM_PATH_NONE (p streaming SpMV
 * launches, single-CTA kernels, or none yet). */
int phipm_wrec_path(const phipm_ctx *ctx);

/* Host logic of the brick kernels (no GPU needed): the decomposition of an nx x ny x nz grid into bricks of whole
 * x-lines on at most `ctas` CTAs with `smem_bytes` of dynamic shared memory each (persist_brick.cuh:
 * brick_geometry).  out10 (HOST) = {py, pz, ylen, zlen, nseg, ncol, ngrp, ppg, lstride, pstride}: py x pz
 * bricks of ylen lines x zlen planes; a line is nseg 64-point warp segments; the CTA's 32 warps form ncol =
 * nseg ylen columns x ngrp z groups of ppg <= 8 planes; shared line / plane strides in doubles.
 * Returns PHIPM_OK, -1 if the grid has no such decomposition (odd nx, nx > 252, too many rows), or
 * PHIPM_EINVAL. */
int phipm_brick_plan(int nx, int ny, int nz, int ctas, int64_t smem_bytes, int *out10);

void phipm_default_opts(phipm_opts *opts);

/* Method used by the kernel-level entry points phipm_expm and phipm_phi_pair (solves take
 * opts.expm_method).  PHIPM_EINVAL for an unknown method. */
int phipm_set_expm_method(phipm_ctx *ctx, int method);

/* Kernel-path selection, per context (measurement and A/B experiments; the defaults are the
 * measured-best paths of DESIGN.md §6 and every path is parity-tested).  Values:
 *   PHIPM_OPT_PERSIST          0 off, 1 auto (default: Lanczos stencil extensions of any size,
 *                              Arnoldi stencil extensions with n <= 2^19), 2 always (stencils)
 *   PHIPM_OPT_TMEM             1 (default) Lanczos persistent kernel keeps y / v~ in tensor memory
 *                              at n >= 303K; 0 shared-memory variant
 *   PHIPM_OPT_WREC             1 (default) w-recurrence of stencils as one cooperative kernel
 *   PHIPM_OPT_LAG              1 (default) lagged normalisation of the streaming Arnoldi step
 *   PHIPM_OPT_PDL              1 (default) programmatic dependent launch between kernels
 *   PHIPM_OPT_SPIN             1 (default) host spins on mapped pinned memory for the attempt
 *                              result; 0 stream synchronisation
 *   PHIPM_OPT_RPT              0 (default) auto, or 2/4/8 rows per thread of the streaming kernels
 *   PHIPM_OPT_CSR_ELL          1 (default) vectorised uniform-row CSR path
 *   PHIPM_OPT_CSR_RING         1 (default) x in a shared-memory ring for banded uniform-row CSR
 *   PHIPM_OPT_CSR_WINDOW       0 (default) per-tile x windows for general CSR
 *   PHIPM_OPT_SMALL_LZ         1 (default) multi-row single-CTA Lanczos for n <= 8192
 *   PHIPM_OPT_PERSIST_MINROWS  0 (default: half a tile) minimum rows per CTA of the persistent kernel
 *   PHIPM_OPT_CSR_PREFETCH     x-ring CSR path: rows ahead whose val / col the TMA engine prefetches
 *                              into L2 (cp.async.bulk.prefetch.L2), 0 = off; default 384
 *   PHIPM_OPT_COL_PREFETCH     1: streaming kernels prefetch the next group of Krylov columns / epilogue
 *                              vectors of the tile into L2 (TMA engine); default 0
 *   PHIPM_OPT_FUSE_ANORM       1 (default): on the banded uniform-row CSR path, ||A||_inf (a1 setup) is
 *                              computed by the first w-recurrence SpMV, which reads val anyway, and the
 *                              analysis pass reads only row_ptr and col; 0: the analysis pass reads val
 *   PHIPM_OPT_CSR_OFF16        1: uniform-row CSR whose band fits int16 -- the analysis pass also writes
 *                              col - row as int16 (context workspace, 2 B per nonzero) and the x-ring
 *                              SpMVs stream those instead of the int32 columns (10 instead of 12 B per
 *                              nonzero); 0 (default, measured faster: the SpMV time did not drop)
 *   PHIPM_OPT_CLUSTER_LZ       Lanczos extensions of stencils with n <= 65536 on one thread-block
 *                              cluster (vectors in the cluster's shared memory, DSMEM reductions and
 *                              halos): 0 off, 1 auto (default: n > 8192), a forced cluster size
 *                              2/4/8/16, or -1 for a single CTA (any n the slice fits)
 *   PHIPM_OPT_SPEC             1 (default): when a Krylov extension runs on few SMs (n <= 8192, or the
 *                              cluster Lanczos kernel), the extension to min((4m+2)/3, m_max) columns
 *                              that Algorithm 3's m-branch can ask for next runs on a second stream
 *                              while the exponential of the attempt runs; 0 off
 *   PHIPM_OPT_DEVSOLVE         1 (default): a symmetric problem with n <= 8192 and the Taylor exponential
 *                              is solved by ONE single-CTA kernel that also runs the controller (no host
 *                              round trip per attempt; opts.profile disables it); 0 off
 *   PHIPM_OPT_GRAPH            1: the two-kernel extension (Arnoldi with n > 2^19, CSR) is captured once as a
 *                              CUDA graph and replayed from a per-context cache; 0 (default) stream launches
 *                              with programmatic dependent launch
 *   PHIPM_OPT_DEFER            1 (default): in the two-kernel extension the fused SpMV + dots kernel ends
 *                              after writing its per-CTA partials; every CTA of the update kernel that
 *                              follows sums them itself (same fixed order, bit-identical totals) and derives
 *                              H(:, j), g, sigma_j; 0: the SpMV's last CTA reduces and finalizes (ticket)
 *   PHIPM_OPT_BRICK            Lanczos extensions of 3-D 7-point stencils on 3-D bricks staged by tensor-map
 *                              TMA (one box copy per brick plane, zero fill outside the grid, z-marching
 *                              warps; y / v~ in tensor memory): 0 off, 1 auto (default: n > 65536 and
 *                              x-lines that fill >= 3/4 of their 64-point warp segments), 2 whenever a
 *                              brick decomposition of the grid exists (nx even, <= 252)
 *   PHIPM_OPT_BRICK_HALO       1: the brick Lanczos kernel keeps the brick's interior in shared memory from step
 *                              to step, copies only the halo (two planes, two lines per plane) and writes
 *                              v~_{j+1} to global memory with tensor stores (shared -> global, one per plane);
 *                              0 (default, measured faster: c4 3500 vs 3320 solves/s): every plane of the brick
 *                              is staged through the tensor map each step and the threads store v~_{j+1}
 *   PHIPM_OPT_SIDE_MAXABS      1 (default): ||u_0||_inf of a solve (Eq. tau_0's b_inf, a1 setup) is reduced on the
 *                              context's second stream with its own scratch, concurrently with the first
 *                              w-recurrence and Krylov extension, which do not depend on it; 0: on the solve's
 *                              stream ahead of them
 *   PHIPM_OPT_PRECOMBINE       1 (n > 8192, not with the Chebyshev method or opts.profile): the exponential's
 *                              epilogue evaluates Algorithm 3's acceptance test (omega <= 1.2, the host's
 *                              expression) and the step's combine kernel is enqueued behind it before the host
 *                              has seen the result, guarded by that decision; 0 (default): the host launches
 *                              the combine.  Bit-identical results; measured: c4 3595 vs 3614 solves/s (no
 *                              gain), c2 2376 vs 3053 (the guarded grid, launched early by PDL, occupies the
 *                              SMs the speculative extension on the second stream needs)
 * phipm_set_option returns PHIPM_EINVAL for an unknown option or an out-of-range value. */
#define PHIPM_OPT_PERSIST          0
#define PHIPM_OPT_TMEM             1
#define PHIPM_OPT_WREC             2
#define PHIPM_OPT_LAG              3
#define PHIPM_OPT_PDL              4
#define PHIPM_OPT_SPIN             5
#define PHIPM_OPT_RPT              6
#define PHIPM_OPT_CSR_ELL          7
#define PHIPM_OPT_CSR_RING         8
#define PHIPM_OPT_CSR_WINDOW       9
#define PHIPM_OPT_SMALL_LZ        10
#define PHIPM_OPT_PERSIST_MINROWS 11
#define PHIPM_OPT_CSR_PREFETCH    12
#define PHIPM_OPT_COL_PREFETCH    13
#define PHIPM_OPT_FUSE_ANORM      14
#define PHIPM_OPT_CSR_OFF16       15
#define PHIPM_OPT_CLUSTER_LZ      16
#define PHIPM_OPT_SPEC            17
#define PHIPM_OPT_DEVSOLVE        18
#define PHIPM_OPT_GRAPH           19
#define PHIPM_OPT_DEFER           20
#define PHIPM_OPT_BRICK           21
#define PHIPM_OPT_BRICK_HALO      22
#define PHIPM_OPT_SIDE_MAXABS     23
#define PHIPM_OPT_PRECOMBINE      24
#define PHIPM_OPT_COUNT           25
int phipm_set_option(phipm_ctx *ctx, int option, int value);
int phipm_get_option(const phipm_ctx *ctx, int option, int *value);

/* Create a context that can solve problems with n <= n_max, m_max <= m_max, p <= p_max.
 * Allocates the device workspace (Krylov basis (m_max+1) x n_max, w vectors, small matrices,
 * reduction scratch) and a pinned result block.  stream: cudaStream_t or NULL. */
int phipm_create(phipm_ctx **ctx, int64_t n_max, int m_max, int p_max, void *stream);
void phipm_destroy(phipm_ctx *ctx);
const char *phipm_strerror(int status);
const char *phipm_last_error(const phipm_ctx *ctx);
int phipm_get_profile(const phipm_ctx *ctx, phipm_profile *out);
void phipm_reset_profile(phipm_ctx *ctx);
/* Copy up to max traced launches (oldest first) into out; *count = number recorded since the
 * last phipm_reset_profile (the buffer keeps the first 65536). */
int phipm_get_trace(const phipm_ctx *ctx, phipm_trace_rec *out, int max, int *count);

/* w = phi_0(tA)u_0 + sum_k t^k phi_k(tA) u_k.  u: HOST array of p+1 DEVICE pointers, each length
 * A->n; w: DEVICE, length n (may alias u[0] only).  opts NULL = defaults.  stats may be NULL.
 * t = 0 -> w = u_0.  All u_k = 0 -> w = 0.  t < 0 -> PHIPM_EINVAL (negate A and use
 * (-1)^k u_k instead). */
int phipm_solve_csr(phipm_ctx *ctx, double t, const phipm_csr *A, int p, const double *const *u,
                    const phipm_opts *opts, double *w, phipm_stats *stats);
int phipm_solve_stencil(phipm_ctx *ctx, double t, const phipm_stencil *S, int p,
                        const double *const *u, const phipm_opts *opts, double *w,
                        phipm_stats *stats);

/* Same computation with HOST buffers: A's arrays (host_csr), u_k and w are HOST pointers (pinned
 * memory copies fastest).  The call copies inputs to the context's device workspace, solves, and
 * copies w back; n <= n_max and nnz <= nnz_max of phipm_reserve_host_csr. */
int phipm_reserve_host_csr(phipm_ctx *ctx, int64_t nnz_max);
int phipm_solve_csr_host(phipm_ctx *ctx, double t, const phipm_csr *host_A, int p,
                         const double *const *host_u, const phipm_opts *opts, double *host_w,
                         phipm_stats *stats);
int phipm_solve_stencil_host(phipm_ctx *ctx, double t, const phipm_stencil *S, int p,
                             const double *const *host_u, const phipm_opts *opts, double *host_w,
                             phipm_stats *stats);

/* Batch of nb INDEPENDENT solves (e.g. the stages of an exponential integrator), run
 * concurrently on one GPU: solve b uses context ctx[b] (its own workspace and stream) and one
 * native host thread, so the host-side controllers of different problems overlap.  Problem b:
 * operator A[b] / S[b], time t[b], p[b], input vectors u[b][0..p[b]] (DEVICE), output w[b]
 * (DEVICE), opts (shared, NULL = defaults), stats[b] (may be NULL).  The contexts must be distinct.
 * Returns PHIPM_OK if every solve succeeded, else the first non-zero status; status[b] (may be
 * NULL) receives each problem's own status. */
int phipm_solve_csr_batch(phipm_ctx *const *ctx, int nb, const double *t, const phipm_csr *A, const int *p,
                          const double *const *const *u, const phipm_opts *opts, double *const *w,
                          phipm_stats *stats, int *status);
int phipm_solve_stencil_batch(phipm_ctx *const *ctx, int nb, const double *t, const phipm_stencil *S,
                              const int *p, const double *const *const *u, const phipm_opts *opts,
                              double *const *w, phipm_stats *stats, int *status);

/* Block solve of nb <= 8 problems sharing the CSR operator A, t, p and the options (
 * the many phipm evaluations with one operator of PAPER.md P:164-185 / P:1353-1358): problem b has
 * inputs u[b][0..p] (DEVICE) and output w[b] (DEVICE, distinct), workspace ctx[b] (distinct
 * contexts on one device).  One controller (Alg. 3/4) drives the block on the largest error estimate
 * (omega = max_b omega_b: every problem meets Tol when a block step is accepted), so all problems take
 * the same steps and Krylov dimensions; each Krylov step multiplies the nb basis vectors by A in ONE
 * pass over val/col (SpMM), then runs every problem's own Gram-Schmidt / Lanczos kernels.  All work
 * is ordered on ctx[0]'s stream (after the work already enqueued on the others); stats[b] (may be
 * NULL) per problem, their attempt records carry the block's omega.  opts.profile applies to ctx[0]'s
 * launches only.  The Chebyshev expm method is not used here (Taylor instead). */
int phipm_solve_csr_block(phipm_ctx *const *ctx, int nb, double t, const phipm_csr *A, int p,
                          const double *const *const *u, const phipm_opts *opts, double *const *w,
                          phipm_stats *stats);

/* Matrix Market ingestion (HOST, no GPU needed): "%%MatrixMarket matrix coordinate {real|integer|pattern}
 * {general|symmetric|skew-symmetric}", square, 1-based indices.  Result: CSR with columns ascending
 * in each row, symmetric / skew-symmetric storage expanded.
 * Call with row_ptr = col = val = NULL to get n and nnz; then again with caller-allocated HOST
 * arrays row_ptr[n+1], col[nnz], val[nnz].  PHIPM_EINVAL on a missing file, an unsupported or
 * malformed header, a non-square matrix, out-of-range indices, a duplicate entry (also one
 * created by expanding symmetric storage that already holds both triangles) or
 * nnz >= 2^31. */
int phipm_mm_read(const char *path, int64_t *n, int64_t *nnz, int32_t *row_ptr, int32_t *col, double *val);

/* ---- kernel-level entry points (parity tests; all DEVICE pointers unless stated) ---- */

/* structural nonzeros of the stencil's CSR form (N_A of Eq. 4); -1 on a bad descriptor */
int64_t phipm_stencil_nnz(const phipm_stencil *S);
/* CSR of the stencil (row order as above; entries of a row in ascending column order:
 * z-, y-, x-, centre, x+, y+, z+); row_ptr[n+1], col[nnz], val[nnz] device, caller-allocated */
int phipm_csr_from_stencil(phipm_ctx *ctx, const phipm_stencil *S, int32_t *row_ptr, int32_t *col,
                           double *val);
/* y = A x */
int phipm_spmv_csr(phipm_ctx *ctx, const phipm_csr *A, const double *x, double *y);
int phipm_spmv_stencil(phipm_ctx *ctx, const phipm_stencil *S, const double *x, double *y);
/* *result (HOST) = x^T y, deterministic grid reduction */
int phipm_dot(phipm_ctx *ctx, int64_t n, const double *x, const double *y, double *result);
/* *result (HOST) = ||A||_inf */
/* ||A||_inf of a stencil operator (HOST arithmetic, no GPU): the closed form over the grid's boundary
 * classes, each row summed in ascending column order (bit-exact with the CSR form's sequential sum);
 * -1 on a bad descriptor. */
double phipm_inf_norm_stencil(const phipm_stencil *S);
int phipm_inf_norm_csr(phipm_ctx *ctx, const phipm_csr *A, double *result);
/* E = exp(A), K x K column-major (Pade-13 scaling and squaring), K <= m_max + p_max + 1 */
int phipm_expm(phipm_ctx *ctx, int K, const double *A, double *E);
/* phi_p(tau H) e1 and phi_{p+1}(tau H) e1 from one augmented exponential (Eq. hathm), H mu x mu
 * with leading dimension ldh (device); phip, phip1 device length mu; *normH1 (HOST) = ||H||_1 */
int phipm_phi_pair(phipm_ctx *ctx, int mu, const double *H, int ldh, double tau, int p,
                   double *phip, double *phip1, double *normH1);
/* Krylov basis from seed v (Alg. 1 via CGS per opts->orth, or Alg. 2 if symmetric): V device
 * n x (m+1) column-major (ld n, normalised columns), H device (m+1) x m column-major; *k (HOST)
 * columns of H built, *brk (HOST) 1 on breakdown, *beta (HOST) = ||v||.  V = H = NULL builds the
 * basis in the context workspace without exporting it (the Arnoldi-step microbenchmark). */
int phipm_krylov_csr(phipm_ctx *ctx, const phipm_csr *A, const double *v, int m,
                     const phipm_opts *opts, double *V, double *H, int *k, int *brk, double *beta);
int phipm_krylov_stencil(phipm_ctx *ctx, const phipm_stencil *S, const double *v, int m,
                         const phipm_opts *opts, double *V, double *H, int *k, int *brk,
                         double *beta);

#ifdef __cplusplus
}
#endif

#endif /* PHIPM_H */
