// solve_small.cuh — the whole phipm solve (Algorithm 3) of a small symmetric problem
// (n <= SMALL_N, Lanczos, Taylor exponential) in ONE single-CTA kernel: the device-side controller.
//
// On the host-driven path every attempt costs a host round trip (the result block is read from mapped
// memory, Algorithm 4 runs on the host, the next kernels are launched) and every step three more
// launches (combine, w-recurrence, extension).  At c1's size (n = 1000, 14 steps, 20 attempts) those
// gaps are a large part of the solve, and one SM does all the work anyway.  Here one CTA of 512
// threads runs, in order and with the arithmetic of the host-driven path's kernels:
//   the w-recurrence w_j = A w_{j-1} + sum_l t_k^l/l! u_{j+l} and the seed (Eq. wrecurrence, P:536-540;
//     spmv_small_kernel's row sums and epilogue order, FIN_SEED),
//   the Lanczos extensions (Alg. 2; krylov_small_lanczos_kernel's step),
//   the augmented exponential and error estimate (expm_body of expm.cuh, shared memory when it fits),
//   the controller (ctl.cuh: the same source as the host loop's, on thread 0, broadcast through shared
//     memory),
//   the combine (Eq. step; axpy_small_kernel's item order).
// The host reads the stats, the status and the attempt records once, after the kernel.
#pragma once

#include "ctl.cuh"
#include "expm.cuh"
#include "kernels.cuh"
#include "small.cuh"

namespace phipm {

constexpr int SS_NT = EXPM_NT;                 // 512: the exponential's thread count
constexpr int SS_MAXU = 8;                     // u_0 .. u_p, p <= 6

// status codes (mapped to PHIPM_* by the host)
enum SsStatus : int { SS_OK = 0, SS_ABORT = 1, SS_NONFINITE = 2, SS_SINGULAR = 3, SS_STEP = 4 };

// same layout as phipm_attempt (include/phipm.h)
struct SsAttempt {
    double t_k, tau, omega, eps, normH1, beta;
    int32_t m, mu, accepted, branch;
};

struct SsOut {
    int status;
    int nsteps, nreject, nspmv, nexpm, m_last, m_peak, nattempts;
    double t_reached;
};

struct SmallSolveArgs {
    double t_end, tol, normA, bthr;
    int p, m_init;
    Problem P;                      // controller problem (m_max = min(m_max, n))
    const double *u[SS_MAXU];
    double *w;                      // output (caller's)
    double *ucur;                   // running solution u_k (workspace)
    double *W;                      // w_1 .. w_{p-1} (columns of ldv)
    double *scratch;                // expm global fallback (6 Kp^2)
    double *comb, *combd;
    AttemptResult *res;             // device-global attempt result
    SsAttempt *att;
    int att_cap;
    SsOut *out;
    int esm_cap;                    // doubles of dynamic shared memory for the exponential's buffers
    long long *clk;                 // optional phase cycles (thread 0): setup, w-recurrence + seed,
                                    // extensions, exponential, controller, combine
};

#define SS_CLK(i)                                                      \
    if (a.clk && threadIdx.x == 0) {                                   \
        const long long c_ = clock64();                                \
        ss_acc[i] += c_ - ss_prev;                                     \
        ss_prev = c_;                                                  \
    }

// block sum of one value per thread (total in every thread): warp trees, then a log2(16)-level tree
// over the 16 warp totals (lane l holds warp l mod 16's); `red` alternates between two arrays so one
// barrier per sum suffices
__device__ __forceinline__ double ss_sum(double v, double *red)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = red[lane & (SS_NT / 32 - 1)];
#pragma unroll
    for (int o = SS_NT / 64; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

// NaN-propagating block max of |x| over rows (maxabs_kernel's rule)
__device__ __forceinline__ double ss_maxabs(const double *x, int n, double *red)
{
    double m = 0.0;
    for (int r = threadIdx.x; r < n; r += SS_NT) {
        const double v = x[r];
        m = (v != v) ? v : fmax(m, fabs(v));
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) {
        const double q = __shfl_xor_sync(0xffffffffu, m, o);
        m = (q != q) ? q : fmax(m, q);
    }
    if (lane == 0) red[warp] = m;
    __syncthreads();
    double s = red[lane & (SS_NT / 32 - 1)];
    for (int o = SS_NT / 64; o > 0; o >>= 1) {
        const double q = __shfl_xor_sync(0xffffffffu, s, o);
        s = (q != q) ? q : fmax(s, q);
    }
    __syncthreads();
    return s;
}

// shared decision block (thread 0 writes, everyone reads after a barrier)
struct SsShared {
    double tau, tk, tau_used;
    int m, k, enq, brk, mu, corr, accepted, done, status, step0, last;
};

template <class Op, int R>
__global__ void __launch_bounds__(SS_NT, 1) small_solve_kernel(Op op, SmallSolveArgs a, Work wk)
{
    extern __shared__ __align__(16) double ssm[];
    __shared__ double red[3][SS_NT / 32];
    __shared__ SsShared sh;
    __shared__ double s_coef[MAXD + MAXZ + 2];
    __shared__ const double *s_src[MAXD + MAXZ + 2];
    const int t = threadIdx.x;
    const int n = (int)op.n;
    const int p = a.p;
    double *vs = ssm;                                        // v~_j of the Lanczos step
    double *esm = ssm + ((n + 15) & ~15);                    // the exponential's buffers
    long long ss_acc[6] = {0, 0, 0, 0, 0, 0};
    long long ss_prev = clock64();
    pdl_wait();

    // ---- setup: b_inf of Eq. (tau_0) (||u_0||_inf, else the first nonzero ||u_k||_inf, R7) ----
    double b_inf = ss_maxabs(a.u[0], n, red[0]);
    for (int k = 1; k <= p && b_inf == 0.0; k++) b_inf = ss_maxabs(a.u[k], n, red[0]);
    if (b_inf == 0.0) {                                       // all inputs zero: w = 0
        for (int r = t; r < n; r += SS_NT) a.w[r] = 0.0;
        if (t == 0) {
            *a.out = SsOut{};
            a.out->t_reached = a.t_end;
        }
        return;
    }
    if (!(b_inf - b_inf == 0.0)) {
        if (t == 0) {
            *a.out = SsOut{};
            a.out->status = SS_NONFINITE;
        }
        return;
    }
    SsOut S{};                                               // (thread 0's copy is the one written out)
    CtlMem mem;
    int attempts = 0;
    if (t == 0) {
        const int m_init = ctl_imin(a.m_init, a.P.m_max);
        const double mbar = 0.5 * ((double)a.m_init + (double)a.P.m_max);
        double tau = (a.normA == 0.0) ? a.t_end : fmin(a.t_end, tau0(a.normA, b_inf, a.tol, mbar));
        if (!(tau > 0.0)) tau = a.t_end;
        sh.tau = tau;
        sh.tk = 0.0;
        sh.m = m_init;
        sh.step0 = 1;
        sh.done = 0;
        sh.status = SS_OK;
        S.m_peak = m_init;
    }
    __syncthreads();
    SS_CLK(0)

    while (true) {
        // ---------------- a new step at t_k: w-recurrence and seed ----------------
        if (t == 0) {
            if (sh.tau > a.t_end - sh.tk) sh.tau = a.t_end - sh.tk;
            sh.k = 0;
            sh.enq = 0;
            sh.brk = 0;
            S.nspmv += p;
            mem = CtlMem();
            attempts = 0;
        }
        __syncthreads();
        const double tk = sh.tk;
        const double *x0 = sh.step0 ? a.u[0] : a.ucur;
        {
            double ysq = 0.0;
            if (p == 0) {
                for (int r = t; r < n; r += SS_NT) {            // V[:,0] = w_0 (axpy_small: 1.0 * x)
                    const double v = fma(1.0, x0[r], 0.0);
                    wk.V[r] = v;
                    ysq = fma(v, v, ysq);
                }
            }
            for (int j = 1; j <= p; j++) {
                const double *x = (j == 1) ? x0 : a.W + (int64_t)(j - 1) * wk.ldv;
                double *y = (j == p) ? wk.V : a.W + (int64_t)j * wk.ldv;
                double zc[SS_MAXU];
                const double *zp[SS_MAXU];
                int nz = 0;
                double coef = 1.0;
                for (int l = 0; l <= p - j; l++) {           // terms t_k^l / l! u_{j+l} (exact zeros skipped)
                    if (l > 0) coef = coef * tk / (double)l;
                    if (l > 0 && coef == 0.0) continue;
                    zc[nz] = coef;
                    zp[nz] = a.u[j + l];
                    nz++;
                }
                for (int r = t; r < n; r += SS_NT) {
                    double v = row_apply(op, x, r) * 1.0;
                    for (int l = 0; l < nz; l++) v = fma(zc[l] * 1.0, zp[l][r], v);
                    y[r] = v;
                    if (j == p) ysq = fma(v, v, ysq);
                }
                __syncthreads();
            }
            const double tot = ss_sum(ysq, red[1]);
            if (t == 0) {                                     // FIN_SEED
                const double b = sqrt(tot);
                wk.st->beta = b;
                wk.sigma[0] = 1.0 / b;
                wk.st->brk = (b > 0.0 && ctl_finite(b)) ? -1 : 0;
                wk.st->nonfinite = ctl_finite(b) ? 0 : 1;
                wk.st->lz = 0.0;
            }
            __syncthreads();
            SS_CLK(1)
        }
        // ---------------- attempts ----------------
        while (true) {
            // extension of the basis to m columns (Alg. 2 steps enq .. m-1)
            const int m = sh.m;
            const int k0 = max(sh.k, sh.enq);
            if (k0 < m && !sh.brk) {
                double sj = wk.sigma[k0];
                double lz = wk.st->lz;
                int brk = wk.st->brk;
                double zv[R];
#pragma unroll
                for (int i = 0; i < R; i++) {
                    const int r = t + SS_NT * i;
                    zv[i] = 0.0;
                    if (r < n) {
                        vs[r] = wk.V[(int64_t)k0 * wk.ldv + r];
                        if (k0 > 0) zv[i] = wk.V[(int64_t)(k0 - 1) * wk.ldv + r];
                    }
                }
                __syncthreads();
                for (int j = k0; j < m && brk < 0; j++) {
                    double y[R], xv[R];
                    double dl = 0.0;
#pragma unroll
                    for (int i = 0; i < R; i++) {
                        const int r = t + SS_NT * i;
                        y[i] = 0.0;
                        xv[i] = 0.0;
                        if (r < n) {
                            y[i] = sj * row_apply(op, vs, r);
                            xv[i] = vs[r];
                            if (j > 0) y[i] = fma(-lz, zv[i], y[i]);
                        }
                        dl = fma(xv[i], y[i], dl);
                    }
                    const double d = ss_sum(dl, red[0]);
                    const double al = sj * d;                 // t_jj = sigma_j v~_j^T y
                    const double g = al * sj;
                    double wl = 0.0;
#pragma unroll
                    for (int i = 0; i < R; i++) {
                        const int r = t + SS_NT * i;
                        if (r < n) {
                            const double w = fma(-g, xv[i], y[i]);   // v~_{j+1} = y - g v~_j
                            wk.V[(int64_t)(j + 1) * wk.ldv + r] = w;
                            vs[r] = w;                        // every thread has read vs (sum above)
                            wl = fma(w, w, wl);
                        }
                        zv[i] = xv[i];
                    }
                    const double tot = ss_sum(wl, red[1]);
                    const double h = sqrt(tot);
                    const double sn = 1.0 / h;
                    const double lzn = h * sj;
                    int b = -1;
                    if (!ctl_finite(h)) b = j + 1;
                    else if (h <= a.bthr) b = j + 1;
                    if (t == 0) {
                        wk.H[j + (size_t)j * wk.ldh] = al;
                        wk.g[0] = g;
                        wk.H[(j + 1) + (size_t)j * wk.ldh] = h;
                        if (j + 1 < wk.hcols) wk.H[j + (size_t)(j + 1) * wk.ldh] = h;
                        wk.st->lz = lzn;
                        wk.sigma[j + 1] = sn;
                        if (!ctl_finite(h)) wk.st->nonfinite = 1;
                        if (b >= 0) wk.st->brk = b;
                    }
                    sj = sn;
                    lz = lzn;
                    brk = b;
                }
                __syncthreads();
                if (t == 0) sh.enq = m;
                SS_CLK(2)
            }
            // the augmented exponential and the error estimate (expm_kernel's body, mode 0)
            {
                ExpmArgs ea;
                memset(&ea, 0, sizeof(ea));
                ea.mode = 0;
                ea.method = 0;                                // PHIPM_EXPM_TAYLOR
                ea.tridiag = 1;
                ea.m = m;
                ea.p = p;
                ea.tau = sh.tau;
                ea.H = wk.H;
                ea.ldh = wk.ldh;
                ea.sigma = wk.sigma;
                ea.st = wk.st;
                ea.comb = a.comb;
                ea.combd = a.combd;
                ea.scratch = a.scratch;
                ea.res = a.res;
                ea.seq = attempts + 1;
                const int Kp = (m + p + 1 + 7) & ~7;
                const bool fits = 6 * expm_ld(Kp) * Kp <= a.esm_cap;
                ea.use_smem = fits ? 1 : 0;
                if (fits) expm_body<true, false>(ea, esm);
                else expm_body<false, false>(ea, esm);
                __syncthreads();
                SS_CLK(3)
            }
            // the controller (Algorithm 4, then Algorithm 3's choice and clamps) on thread 0
            if (t == 0) {
                attempts++;
                __threadfence_block();                    // (this thread published it in expm_body)
                const AttemptResult R_ = *a.res;
                S.nexpm++;
                int kb;
                if (R_.brk >= 0) {
                    kb = ctl_imax(sh.k, R_.brk);
                    sh.brk = 1;
                } else {
                    kb = ctl_imax(sh.k, m);
                }
                if (R_.brk >= 0 && R_.brk < sh.k) kb = sh.k;
                S.nspmv += kb - sh.k;
                sh.k = kb;
                const double tau = sh.tau;
                const double omega = a.t_end * R_.eps / (tau * a.tol);
                if (R_.status == 3) sh.status = SS_ABORT;
                else if (R_.status == 5) sh.status = SS_NONFINITE;
                else if (R_.status == 6) sh.status = SS_SINGULAR;
                else if (!ctl_finite(omega)) sh.status = SS_NONFINITE;
                if (sh.status == SS_OK) {
                    sh.mu = R_.mu;
                    sh.corr = (R_.h != 0.0 && !(R_.brk >= 0 && R_.brk <= R_.mu)) ? 1 : 0;
                    const bool accepted = omega <= 1.2;
                    const Decision d = control(a.P, mem, tau, m, R_.eps, omega, R_.normH1, a.t_end - sh.tk, accepted);
                    if (S.nattempts < a.att_cap) {
                        SsAttempt &A = a.att[S.nattempts];
                        A.t_k = sh.tk;
                        A.tau = tau;
                        A.omega = omega;
                        A.eps = R_.eps;
                        A.normH1 = R_.normH1;
                        A.beta = R_.beta;
                        A.m = m;
                        A.mu = R_.mu;
                        A.accepted = accepted ? 1 : 0;
                        A.branch = d.branch;
                    }
                    S.nattempts++;
                    sh.tau_used = tau;
                    S.m_peak = ctl_imax(S.m_peak, m);
                    if (accepted) S.m_last = m;
                    sh.tau = d.tau_next;
                    sh.m = d.m_next;
                    sh.accepted = accepted ? 1 : 0;
                    if (!accepted) {
                        S.nreject++;
                        if (attempts >= 100 || sh.tau < 1e-15 * a.t_end) sh.status = SS_STEP;
                    }
                }
            }
            __syncthreads();
            SS_CLK(4)
            if (sh.status != SS_OK || sh.accepted) break;
        }
        if (sh.status == SS_STEP) {                          // w := u_k, as the host path
            const double *src = sh.step0 ? a.u[0] : a.ucur;
            for (int r = t; r < n; r += SS_NT) a.w[r] = src[r];
        }
        if (sh.status != SS_OK) break;
        // ---------------- combine (Eq. step): u_{k+1} = sum comb_i v~_i + sum tau^j/j! w_j ----------------
        {
            const bool last = sh.tau_used >= a.t_end - sh.tk;
            double *out = last ? a.w : a.ucur;
            const double *base = sh.step0 ? a.u[0] : a.ucur;
            const int nbase = (p >= 1) ? 1 : 0;
            const int nc = sh.mu + sh.corr;
            const int ne = p > 1 ? p - 1 : 0;
            const int nitem = nbase + nc + ne;
            for (int k = t; k < nitem; k += SS_NT) {          // axpy_small_kernel's item order
                double c;
                const double *src;
                if (k < nbase) {
                    c = 1.0 * a.combd[0];
                    src = base;
                } else if (k < nbase + nc) {
                    const int kc = k - nbase;
                    c = 1.0 * a.comb[kc];
                    src = wk.V + (int64_t)kc * wk.ldv;
                } else {
                    const int i = k - nbase - nc;
                    c = 1.0 * a.combd[1 + i];
                    src = a.W + (int64_t)(i + 1) * wk.ldv;
                }
                s_coef[k] = c;
                s_src[k] = src;
            }
            __syncthreads();
            for (int r = t; r < n; r += SS_NT) {
                double acc = 0.0;
                int k = 0;
                for (; k + 8 <= nitem; k += 8) {
                    double x[8];
#pragma unroll
                    for (int u = 0; u < 8; u++) x[u] = s_src[k + u][r];
#pragma unroll
                    for (int u = 0; u < 8; u++) acc = fma(s_coef[k + u], x[u], acc);
                }
                for (; k < nitem; k++) acc = fma(s_coef[k], s_src[k][r], acc);
                out[r] = acc;
            }
            __syncthreads();
            if (t == 0) {
                if (last) sh.tk = a.t_end;
                else sh.tk += sh.tau_used;
                S.nsteps++;
                sh.step0 = 0;
                S.t_reached = sh.tk;
                sh.done = last ? 1 : (sh.tk < a.t_end ? 0 : 1);
            }
            __syncthreads();
            SS_CLK(5)
            if (sh.done) break;
        }
    }
    if (a.clk && t == 0)
        for (int i = 0; i < 6; i++) a.clk[i] = ss_acc[i];
    if (t == 0) {
        S.status = sh.status;
        if (sh.status != SS_OK) S.t_reached = sh.tk;
        *a.out = S;
    }
}

} // namespace phipm
