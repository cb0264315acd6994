// expm.cuh — single-CTA kernel for the small dense part of a phipm attempt (Sec. 3.1-3.2):
//
//   Hhat = [[tau H_mu, e1, 0], [0, 0, I_p], [0, 0, 0]]   (Eq. hathm P:368-377 with p+1)
//   E = exp(Hhat) by scaling and squaring (here with a Taylor polynomial, see cta_expm)
//   phi_p(tau H)e1 = E[0:mu, mu+p-1] (p = 0: column 0), phi_{p+1}(tau H)e1 = E[0:mu, mu+p]
//   eps = tau^p beta tau |h_{mu+1,mu} [phi_{p+1}]_mu|                 (Eq. errest with R9/R10)
//   combine coefficients of Eq. (step)/(phipapprox2) for the assembly kernel.
//
// All K x K matrices (K <= m_max + p_max + 1) live in shared memory when 6 K^2 doubles fit,
// otherwise in an L2-resident global scratch; generic addressing serves both.  Every step of the
// exponential is a K x K product on the fp64 tensor cores (DMMA) shared by all warps of the CTA.
#pragma once

#include "kernels.cuh"

namespace phipm {

constexpr int EXPM_NT = 512;
constexpr int EXPM_KMAX = 136;         // padded K bound (m_max + p_max + 1 <= 128 + 8)

// result block read by the host controller (mapped pinned memory)
struct AttemptResult {
    double eps;        // error estimate (R10)
    double normH1;     // ||H_mu||_1
    double beta;       // ||w_p||_2
    double h;          // h_{mu+1,mu} used by the corrector (0 on breakdown)
    int mu;            // Krylov dimension used
    int brk;           // -1 or the breakdown position
    int status;        // 0 ok, 5 non-finite, 6 singular, 7 Chebyshev interval too wide
    int seq;           // attempt sequence number (host sanity check)
    double eps_noise;  // Chebyshev method: rounding-noise bound of eps (0 for the augmented exponential)
    int accepted;      // ExpmArgs.dec given: the acceptance decision taken on the device (1 / 0), else -1
    int pad_;
};

// Publish an attempt result to the host (mapped pinned memory), one thread: the fields with
// seq = -1, a system-scope fence, then the sequence number the host spins on (wait_attempt), so the
// host never sees a new seq next to stale fields.  Every path of expm_kernel publishes through here.
__device__ inline void publish_result(AttemptResult *dst, AttemptResult r, int seq)
{
    r.seq = -1;
    *dst = r;
    __threadfence_system();
    *(volatile int *)&dst->seq = seq;
}

struct ExpmArgs {
    int mode;          // 0: phipm attempt; 1: plain expm of Ain; 2: phi pair of H (mu = m)
    int method;        // PHIPM_EXPM_TAYLOR (0) or PHIPM_EXPM_PADE13 (1)
    int m, p;          // requested Krylov dimension, phi order
    int tridiag;       // Lanczos: H is tridiagonal, read only the band
    double tau;
    const double *H;   // Hessenberg (ld ldh)
    int ldh;
    const double *sigma;
    DevState *st;
    double *comb;      // out: coefficients of v~_0..v~_mu (length mu+1)
    double *combd;     // out: coefficients of w_0..w_{p-1}
    double *scratch;   // 6 * Kmax^2 doubles (global fallback)
    int use_smem;
    int K;             // mode 1: matrix size
    const double *Ain; // mode 1
    double *Eout;      // mode 1
    double *phip_out, *phip1_out;   // mode 2
    AttemptResult *res;
    int seq;
    long long *clk;    // optional phase timestamps (PHIPM_EXPM_CLOCKS)
    // mode 0, optional: the acceptance test of Algorithm 3 on the device, omega = t_end eps / (tau tol) <= 1.2
    // (the host's expression with the same IEEE operations), for a combine kernel enqueued before the host has
    // seen the result: dec[0] = seq if accepted else -seq, dec[1] = number of basis columns of the combine
    int *dec;
    double t_end, tol;
};

// leading dimension of the K x K work matrices: Kp rounded up to 4 (mod 16) doubles, so the
// 32 lanes of a DMMA fragment load (8 rows x 4 columns, or 4 rows x 8 columns) touch every bank
// pair at most twice (256 B = 2 wavefronts, the minimum)
__host__ __device__ inline int expm_ld(int Kp) { return Kp + ((4 - Kp % 16) + 16) % 16; }

// C = epi(row, col, (A B)[row, col]) for Kp x Kp column-major matrices (Kp a multiple of 8, zero
// padded) on the fp64 tensor cores: each warp computes 8x8 output tiles with mma.sync.m8n8k4.f64
// (SASS DMMA).  Fragment layouts (PTX ISA, m8n8k4 .f64): A row-major 8x4, a0 = A[lane/4][lane%4];
// B column-major 4x8, b0 = B[lane%4][lane/4]; C 8x8, c_i = C[lane/4][2 (lane%4) + i].
template <class Epi>
__device__ __forceinline__ void cta_matmul_e(int Kp, int ld, const double *A, const double *B, double *C, Epi epi)
{
    // each warp computes a 2 x 2 block of 8x8 tiles (16 x 16 outputs): per k-step it loads two A
    // and two B fragments for four DMMAs, half the shared-memory fragment traffic of one tile at a
    // time (fragment loads, not the DMMA rate, bound the product)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int nt = Kp >> 3, nb = (nt + 1) >> 1;          // tiles per side, 2x2 blocks per side
    const int ar = lane >> 2, ac = lane & 3;
    for (int bI = warp; bI < nb * nb; bI += nw) {
        const int bi = bI % nb, bj = bI / nb;
        const int ti0 = 2 * bi, tj0 = 2 * bj;
        const bool ri = ti0 + 1 < nt, rj = tj0 + 1 < nt;   // second tile row / column exists
        const double *A0 = A + (ti0 * 8 + ar) + (size_t)ac * ld;
        const double *A1 = ri ? A0 + 8 : A0;
        const double *B0 = B + ac + (size_t)(tj0 * 8 + ar) * ld;
        const double *B1 = rj ? B0 + (size_t)8 * ld : B0;
        double c[2][2][2];
#pragma unroll
        for (int x = 0; x < 2; x++)
#pragma unroll
            for (int y = 0; y < 2; y++) c[x][y][0] = c[x][y][1] = 0.0;
        // two k-steps per iteration, both fragment sets loaded first (tools/mm_probe.cu: 5-6 % faster
        // products than one set prefetched one step ahead at Kp = 40, 56, 64)
#define EXPM_DMMA4(A0_, A1_, B0_, B1_)                                                                             \
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"                   \
                 : "+d"(c[0][0][0]), "+d"(c[0][0][1]) : "d"(A0_), "d"(B0_));                                      \
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"                   \
                 : "+d"(c[0][1][0]), "+d"(c[0][1][1]) : "d"(A0_), "d"(B1_));                                      \
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"                   \
                 : "+d"(c[1][0][0]), "+d"(c[1][0][1]) : "d"(A1_), "d"(B0_));                                      \
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"                   \
                 : "+d"(c[1][1][0]), "+d"(c[1][1][1]) : "d"(A1_), "d"(B1_));
        int k = 0;
        for (; k + 8 <= Kp; k += 8) {
            const double a0 = A0[(size_t)k * ld], a1 = A1[(size_t)k * ld], b0 = B0[k], b1 = B1[k];
            const double e0 = A0[(size_t)(k + 4) * ld], e1 = A1[(size_t)(k + 4) * ld], f0 = B0[k + 4],
                         f1 = B1[k + 4];
            EXPM_DMMA4(a0, a1, b0, b1)
            EXPM_DMMA4(e0, e1, f0, f1)
        }
        if (k < Kp) {                                    // (not reached: Kp is a multiple of 8)
            const double a0 = A0[(size_t)k * ld], a1 = A1[(size_t)k * ld], b0 = B0[k], b1 = B1[k];
            EXPM_DMMA4(a0, a1, b0, b1)
        }
#undef EXPM_DMMA4
#pragma unroll
        for (int x = 0; x < 2; x++)
#pragma unroll
            for (int y = 0; y < 2; y++) {
                if ((x && !ri) || (y && !rj)) continue;
                const int row = (ti0 + x) * 8 + ar, col = (tj0 + y) * 8 + 2 * ac;
                C[row + (size_t)col * ld] = epi(row, col, c[x][y][0]);
                C[row + (size_t)(col + 1) * ld] = epi(row, col + 1, c[x][y][1]);
            }
    }
    __syncthreads();
}

struct EpiNone {
    __device__ double operator()(int, int, double v) const { return v; }
};

__device__ __forceinline__ void cta_matmul(int Kp, int ld, const double *A, const double *B, double *C)
{
    cta_matmul_e(Kp, ld, A, B, C, EpiNone{});
}

// Paterson-Stockmeyer block B_k = c0 I + c1 A + c2 A^2 + c3 A^3 added in the product's epilogue
struct EpiBlock {
    const double *A1, *A2, *A3;
    int ld;
    double fv;                       // exact power-of-two factor of the product (the scaling 2^-4s)
    double c0, c1, c2, c3;
    __device__ double operator()(int r, int c, double v) const
    {
        const size_t e = r + (size_t)c * ld;
        double b = c3 * A3[e];
        b = fma(c2, A2[e], b);
        b = fma(c1, A1[e], b);
        if (r == c) b += c0;
        return fv * v + b;
    }
};

// optional phase timestamps (PHIPM_EXPM_CLOCKS)
#define EXPM_CLK(i) \
    if (clk && threadIdx.x == 0) clk[i] = clock64();

__device__ __forceinline__ double block_max_colsum(int K, int ld, const double *A, double *sred)
{
    // ||A||_1 = max_j sum_i |a_ij|
    double m = 0.0;
    for (int jc = threadIdx.x; jc < K; jc += blockDim.x) {
        double s = 0.0;
        for (int i = 0; i < K; i++) s += fabs(A[i + (size_t)jc * ld]);
        m = fmax(m, s);
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = m;
    __syncthreads();
    double r = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) r = fmax(r, sred[w]);
    __syncthreads();
    return r;
}

// Pade [13/13] coefficients c_j = (26-j)! 13! / (26! j! (13-j)!), c_0 = 1, via the ratio
// c_{j+1}/c_j = (13-j)/((26-j)(j+1)).
__device__ __forceinline__ void pade13(double *c)
{
    c[0] = 1.0;
    for (int j = 0; j < 13; j++) c[j + 1] = c[j] * (double)(13 - j) / ((double)(26 - j) * (double)(j + 1));
}

// PHIPM_EXPM_PADE13: the paper's method: [13/13] Pade with s = ceil_+(log2(||A||_1 /
// 5.37)) squarings; U, V from A^2, A^4, A^6 (6 DMMA products), then (V - U) X = (V + U) by
// Gauss-Jordan with partial pivoting (implicit: no row interchanges, pivot row of column c is
// prow[c]).  One barrier per column: warp 0 updates the next pivot column, searches its pivot and
// prepares the multipliers while the other warps eliminate the current column.  K dependent pivot
// steps on one SM: the latency the Taylor method avoids.  Returns exp(M0); status 0/5/6.
__device__ double *cta_expm_pade(int K, int Kp, int ld, double *M0, double *M1, double *M2, double *M3, double *M4, double *M5,
                            double *sred, int *s_int, double *fcol, int *status, long long *clk)
{
    const int KK = ld * Kp, t = threadIdx.x;         // whole buffers (padding rows are never read)
    double c[14];
    pade13(c);
    // scaling: s = ceil_+(log2(||A||_1 / 5.37)) (theta_13 = 5.37 as printed, R26)
    const double nrm = block_max_colsum(Kp, ld, M0, sred);
    int s = 0;
    if (nrm > 0.0) {
        const double l = ceil(log2(nrm / 5.37));
        s = l > 0.0 ? (int)l : 0;
    }
    if (!isfinite(nrm)) { *status = 5; return M0; }
    const double sc = ldexp(1.0, -s);
    for (int e = t; e < KK; e += blockDim.x) M0[e] *= sc;
    __syncthreads();
    cta_matmul(Kp, ld, M0, M0, M1);            // A2
    cta_matmul(Kp, ld, M1, M1, M2);            // A4
    cta_matmul(Kp, ld, M2, M1, M3);            // A6
    EXPM_CLK(2)
    // U = A [A6 (c13 A6 + c11 A4 + c9 A2) + c7 A6 + c5 A4 + c3 A2 + c1 I]
    for (int e = t; e < KK; e += blockDim.x) M4[e] = c[13] * M3[e] + c[11] * M2[e] + c[9] * M1[e];
    __syncthreads();
    cta_matmul(Kp, ld, M3, M4, M5);
    for (int e = t; e < KK; e += blockDim.x) M5[e] = M5[e] + c[7] * M3[e] + c[5] * M2[e] + c[3] * M1[e];
    __syncthreads();
    for (int i = t; i < Kp; i += blockDim.x) M5[i * (ld + 1)] += c[1];
    __syncthreads();
    cta_matmul(Kp, ld, M0, M5, M4);            // U in M4
    // V = A6 (c12 A6 + c10 A4 + c8 A2) + c6 A6 + c4 A4 + c2 A2 + c0 I
    for (int e = t; e < KK; e += blockDim.x) M5[e] = c[12] * M3[e] + c[10] * M2[e] + c[8] * M1[e];
    __syncthreads();
    cta_matmul(Kp, ld, M3, M5, M0);            // A no longer needed
    for (int e = t; e < KK; e += blockDim.x) M0[e] = M0[e] + c[6] * M3[e] + c[4] * M2[e] + c[2] * M1[e];
    __syncthreads();
    for (int i = t; i < Kp; i += blockDim.x) M0[i * (ld + 1)] += c[0];   // V
    __syncthreads();
    // P = V + U (M1), Q = V - U (M2)
    for (int e = t; e < KK; e += blockDim.x) {
        const double v = M0[e], u = M4[e];
        M1[e] = v + u;
        M2[e] = v - u;
    }
    __syncthreads();
    EXPM_CLK(3)
    // Gauss-Jordan with partial pivoting: Q X = P, implicit pivoting (no row interchanges; the
    // pivot row of column c is prow[c]), ONE barrier per column: warp 0 updates the next pivot
    // column first, searches its pivot among the unused rows and prepares the multipliers while
    // the other warps eliminate the current column from the rest of [Q | P].
    double *Q = M2, *P = M1;
    int *prow = s_int + 8, *used = s_int + 8 + EXPM_KMAX;
    double *fb = fcol;                                    // 2 x EXPM_KMAX multipliers
    __shared__ int s_pr[2], s_bad;
    __shared__ double s_rq[EXPM_KMAX];
    const int warp = t >> 5, lane = t & 31;
    for (int r = t; r < K; r += blockDim.x) used[r] = 0;
    if (t == 0) s_bad = 0;
    __syncthreads();
    auto lookahead = [&](int c, int b) {                 // warp 0; column c of Q is final
        double best = -1.0;
        int bi = K;
        for (int r = lane; r < K; r += 32)
            if (!used[r]) {
                const double a = fabs(Q[r + (size_t)c * ld]);
                if (a > best) { best = a; bi = r; }
            }
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if (!(best >= 1e-300) || bi >= K) {
            if (lane == 0) s_bad = 1;
            return;
        }
        const double rp = 1.0 / Q[bi + (size_t)c * ld];
        for (int r = lane; r < K; r += 32) fb[b * EXPM_KMAX + r] = (r == bi) ? 0.0 : Q[r + (size_t)c * ld] * rp;
        __syncwarp();
        if (lane == 0) {
            s_pr[b] = bi;
            used[bi] = 1;
            prow[c] = bi;
        }
        __syncwarp();
    };
    if (warp == 0) lookahead(0, 0);
    __syncthreads();
    const int t2 = t - 32, n2 = (int)blockDim.x - 32;
    const int er = t2 % K, eg = t2 / K, neg = n2 / K;     // elimination warps: fixed row, column group
    for (int col = 0; col < K; col++) {
        if (s_bad) { *status = 6; return P; }
        const int b = col & 1;
        const int pr = s_pr[b];
        const double *f = fb + b * EXPM_KMAX;
        if (warp == 0) {
            if (col + 1 < K) {
                const int j = col + 1;
                const double pv = Q[pr + (size_t)j * ld];
                for (int r = lane; r < K; r += 32)
                    if (r != pr) Q[r + (size_t)j * ld] -= f[r] * pv;
                __syncwarp();
                lookahead(col + 1, b ^ 1);
            }
        } else if (eg < neg && er != pr) {
            const double fr = f[er];
            if (fr != 0.0) {
                // Q columns col+2 .. K-1 and P columns 0 .. K-1 owned by this thread's column group,
                // four loads in flight before the stores
                auto rank1 = [&](double *M, int j) {
                    for (; j + 3 * neg < K; j += 4 * neg) {
                        const double p0 = M[pr + (size_t)j * ld], p1 = M[pr + (size_t)(j + neg) * ld];
                        const double p2 = M[pr + (size_t)(j + 2 * neg) * ld], p3 = M[pr + (size_t)(j + 3 * neg) * ld];
                        const double x0 = M[er + (size_t)j * ld], x1 = M[er + (size_t)(j + neg) * ld];
                        const double x2 = M[er + (size_t)(j + 2 * neg) * ld], x3 = M[er + (size_t)(j + 3 * neg) * ld];
                        M[er + (size_t)j * ld] = x0 - fr * p0;
                        M[er + (size_t)(j + neg) * ld] = x1 - fr * p1;
                        M[er + (size_t)(j + 2 * neg) * ld] = x2 - fr * p2;
                        M[er + (size_t)(j + 3 * neg) * ld] = x3 - fr * p3;
                    }
                    for (; j < K; j += neg) M[er + (size_t)j * ld] -= fr * M[pr + (size_t)j * ld];
                };
                rank1(Q, col + 2 + eg);
                rank1(P, eg);
            }
        }
        __syncthreads();
    }
    // X[c, :] = P[prow(c), :] / Q[prow(c), c]   (the pivot row's diagonal value is final)
    for (int c = t; c < K; c += blockDim.x) s_rq[c] = 1.0 / Q[prow[c] + (size_t)c * ld];
    __syncthreads();
    double *Xo = M3;
    for (int e = t; e < K * K; e += blockDim.x) {
        const int c = e % K, j = e / K;
        Xo[c + (size_t)j * ld] = P[prow[c] + (size_t)j * ld] * s_rq[c];
    }
    // padding block of X: identity (Q and P were identity there)
    for (int e = t; e < Kp * Kp; e += blockDim.x) {
        const int c = e % Kp, j = e / Kp;
        if (c >= K || j >= K) Xo[c + (size_t)j * ld] = (c == j) ? 1.0 : 0.0;
    }
    __syncthreads();
    P = Xo;
    EXPM_CLK(4)
    // squaring
    double *X = P, *T = M4;
    for (int q = 0; q < s; q++) {
        cta_matmul(Kp, ld, X, X, T);
        double *tmp = X;
        X = T;
        T = tmp;
    }
    EXPM_CLK(5)
    return X;
}

// Taylor degrees evaluable from A, A^2, A^3, A^4 by Paterson-Stockmeyer (m = 4 r), the products
// they cost including the three powers, and their backward-error thresholds theta_m: the largest
// alpha with sum_{k>m} |c_k| alpha^(k-1) <= 2^-53 for h_m(x) = log(exp(-x) T_m(x)) = sum c_k x^k
// (exact rational series, tools/taylor_theta.py).
constexpr int TAYLOR_NDEG = 3;
__device__ constexpr int TAYLOR_M[TAYLOR_NDEG] = {8, 12, 16};
__device__ constexpr int TAYLOR_PROD[TAYLOR_NDEG] = {4, 5, 6};
__device__ constexpr double TAYLOR_THETA[TAYLOR_NDEG] = {0.049912288711153226, 0.29961589138115802,
                                                         0.78028742566265741};

// Taylor coefficients 1/k!, k = 0..16, correctly rounded from the exact rationals
__device__ constexpr double TAYLOR_INVFACT[17] = {
    1.0, 1.0, 0.5, 0.16666666666666666, 0.041666666666666664, 0.008333333333333333, 0.001388888888888889,
    0.0001984126984126984, 2.48015873015873e-05, 2.7557319223985893e-06, 2.755731922398589e-07,
    2.505210838544172e-08, 2.08767569878681e-09, 1.6059043836821613e-10, 1.1470745597729725e-11,
    7.647163731819816e-13, 4.779477332387385e-14};

// exp(M0) -> returned pointer (one of the buffers); M0..M5 are Kp x Kp buffers (Kp = K rounded
// up to a multiple of 8, padding zero: exp(blockdiag(A, 0)) = blockdiag(exp A, I)).  status 0/5.
//
// Scaling and squaring with a truncated Taylor polynomial evaluated by Paterson-Stockmeyer, all
// products on DMMA across the CTA.  The paper's MATLAB expm (and the oracle) uses the [13/13]
// Pade approximant, whose linear solve (V - U) X = (V + U) is a chain of K dependent pivot steps
// on one SM; the polynomial needs only matrix products.  Both approximate exp to unit-roundoff
// backward error; the GPU's number of squarings is chosen from
//   alpha = max(||A^3||_1^(1/3), ||A^4||_1^(1/4))  (>= the spectral growth; Al-Mohy & Higham's
// alpha_3 bound, valid for m >= 5), which the nilpotent shift block of Hhat does not inflate.
__device__ double *cta_expm(int K, int Kp, int ld, double *M0, double *M1, double *M2, double *M3, double *M4, double *M5,
                            double *sred, int *status, long long *clk)
{
    (void)K;
    const int KK = ld * Kp, t = threadIdx.x;         // whole buffers (padding rows are never read)
    cta_matmul(Kp, ld, M0, M0, M1);            // A^2
    cta_matmul(Kp, ld, M1, M0, M2);            // A^3
    cta_matmul(Kp, ld, M1, M1, M3);            // A^4
    EXPM_CLK(2)
    // ||A||_1, ||A^3||_1, ||A^4||_1: one thread per (matrix, column) with four interleaved partial sums over
    // the rows, then the max over columns (warp shuffle trees, then the warps)
    const int lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
    double m1 = 0.0, m3 = 0.0, m4 = 0.0;
    for (int q = t; q < 3 * Kp; q += blockDim.x) {
        const int w = q / Kp, jc = q - w * Kp;
        const double *col = (w == 0 ? M0 : w == 1 ? M2 : M3) + (size_t)jc * ld;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        for (int i = 0; i < Kp; i += 4) {                  // (Kp is a multiple of 8)
            s0 += fabs(col[i]);
            s1 += fabs(col[i + 1]);
            s2 += fabs(col[i + 2]);
            s3 += fabs(col[i + 3]);
        }
        const double sc = (s0 + s1) + (s2 + s3);
        if (w == 0) m1 = fmax(m1, sc);
        else if (w == 1) m3 = fmax(m3, sc);
        else m4 = fmax(m4, sc);
    }
    for (int o = 16; o > 0; o >>= 1) {
        m1 = fmax(m1, __shfl_xor_sync(0xffffffffu, m1, o));
        m3 = fmax(m3, __shfl_xor_sync(0xffffffffu, m3, o));
        m4 = fmax(m4, __shfl_xor_sync(0xffffffffu, m4, o));
    }
    EXPM_CLK(8)
    if (lane == 0) { sred[warp] = m1; sred[warp + 16] = m3; sred[warp + 32] = m4; }
    __syncthreads();
    EXPM_CLK(9)
    // max over the warps by a shuffle tree (identical in every warp)
    auto wmax = [&](double v) {
        for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
        return v;
    };
    const double nrm = wmax(lane < nw ? sred[lane] : 0.0);
    const double n3 = wmax(lane < nw ? sred[lane + 16] : 0.0);
    const double n4 = wmax(lane < nw ? sred[lane + 32] : 0.0);
    __syncthreads();
    if (!isfinite(nrm)) { *status = 5; return M0; }
    // alpha = min(max(||A^3||^(1/3), ||A^4||^(1/4)), ||A||) <= T  <=>  (n3 <= T^3 and n4 <= T^4) or
    // nrm <= T: the smallest s with alpha <= theta_d 2^s from exact comparisons (no cbrt / log2),
    // starting a little below a single-precision estimate
    auto fits = [&](double T) { return (n3 <= T * T * T && n4 <= (T * T) * (T * T)) || nrm <= T; };
    const float l3 = n3 > 0.0 ? __log2f((float)n3) * (1.0f / 3.0f) : -1e30f;
    const float l4 = n4 > 0.0 ? __log2f((float)n4) * 0.25f : -1e30f;
    const float la = fminf(fmaxf(l3, l4), nrm > 0.0 ? __log2f((float)nrm) : -1e30f);   // ~log2 alpha
    EXPM_CLK(10)
    // degree and squarings: minimise products (powers + Horner) + squarings, smallest m on ties.
    // theta 2^s by adding s to the exponent field (exact; theta is normal, s <= 1000)
    auto pow2 = [](double th, int sd) {
        return __longlong_as_double(__double_as_longlong(th) + ((long long)sd << 52));
    };
    int m = TAYLOR_M[0], s = 0, best = 1 << 30;
#pragma unroll
    for (int d = 0; d < TAYLOR_NDEG; d++) {
        const double th = TAYLOR_THETA[d];
        int sd = 0;
        if (!fits(th)) {
            sd = min(1000, max(1, (int)(la - __log2f((float)th))));   // estimate, then exact fix-up
            if (sd > 1 && fits(pow2(th, sd - 1))) {
                sd--;
                while (sd > 1 && fits(pow2(th, sd - 1))) sd--;
            } else {
                while (sd < 1000 && !fits(pow2(th, sd))) sd++;
            }
        }
        if (TAYLOR_PROD[d] + sd < best) { best = TAYLOR_PROD[d] + sd; m = TAYLOR_M[d]; s = sd; }
    }
    EXPM_CLK(11)
    // the powers of 2^-s A are 2^-sk A^k: the scale factors (exact powers of two) are folded into
    // the polynomial's coefficients and the products' epilogue (f4 (Y A^4) = Y (f4 A^4) exactly),
    // instead of a pass over four matrices
    const double f1 = ldexp(1.0, -s), f2 = ldexp(1.0, -2 * s), f3 = ldexp(1.0, -3 * s), f4 = ldexp(1.0, -4 * s);
    auto c = [](int k) { return TAYLOR_INVFACT[k]; };
    EXPM_CLK(4)
    // Horner in A^4: Y = B_{r-1} + c_m A^4;  Y <- Y A^4 + B_k, k = r-2 .. 0
    const int r = m >> 2;
    double *Y = M4, *Z = M5;
    {
        const int b = 4 * (r - 1);
        const double cm = c(m) * f4, cb0 = c(b), cb1 = c(b + 1) * f1, cb2 = c(b + 2) * f2, cb3 = c(b + 3) * f3;
        for (int e = t; e < KK; e += blockDim.x) {
            double v = cm * M3[e];
            v = fma(cb3, M2[e], v);
            v = fma(cb2, M1[e], v);
            v = fma(cb1, M0[e], v);
            Y[e] = v;
        }
        __syncthreads();
        for (int i = t; i < Kp; i += blockDim.x) Y[i * (ld + 1)] += cb0;
        __syncthreads();
    }
    for (int k = r - 2; k >= 0; k--) {
        const int b = 4 * k;
        cta_matmul_e(Kp, ld, Y, M3, Z, EpiBlock{M0, M1, M2, ld, f4, c(b), c(b + 1) * f1, c(b + 2) * f2, c(b + 3) * f3});
        double *tmp = Y;
        Y = Z;
        Z = tmp;
    }
    EXPM_CLK(3)
    // squaring (Z and M0 are free)
    double *X = Y, *T = Z;
    for (int q = 0; q < s; q++) {
        cta_matmul(Kp, ld, X, X, T);
        double *tmp = X;
        X = T;
        T = tmp;
    }
    EXPM_CLK(5)
    if (clk && t == 0) clk[7] = ((long long)m << 16) | s;
    return X;
}

// PADE: method PHIPM_EXPM_PADE13 (separate instantiations keep each kernel's code small: the
// kernel runs cold, after the streaming kernels, once per attempt)
template <bool SMEM, bool PADE>
__device__ __forceinline__ void expm_body(const ExpmArgs &a, double *esm)
{
    __shared__ double sred[3 * (EXPM_NT / 32)];
    __shared__ int s_int[PADE ? 8 + 2 * EXPM_KMAX : 1];     // Pade: pivot rows, used flags
    __shared__ double fcol[PADE ? 2 * EXPM_KMAX : 1];       // Pade: multipliers
    __shared__ int s_mu, s_brk;
    const int t = threadIdx.x;
    // phase stamps go to shared memory (a store to host-mapped memory followed by a barrier would
    // stall and distort the phases); copied out to a.clk once at the end
    __shared__ long long s_clk[16];
    long long *clk = a.clk ? s_clk : nullptr;
    if (clk && t == 0) {
        for (int i = 0; i < 16; i++) s_clk[i] = 0;
        clk[0] = clock64();
    }
    int mu, K;
    if (a.mode == 1) {
        mu = 0;
        K = a.K;
    } else {
        if (t == 0) {
            int m = a.m;
            s_brk = -1;
            if (a.mode == 0) {
                // one read of the breakdown position; a breakdown beyond m belongs to a speculative
                // extension still running on the second stream (phipm.cu) and not to this attempt
                const int brk = a.st->brk;
                s_brk = (brk >= 0 && brk <= m) ? brk : -1;
                if (s_brk >= 0 && s_brk < m) m = s_brk;
            }
            s_mu = m;
        }
        __syncthreads();
        mu = s_mu;
        K = mu + a.p + 1;
    }
    const double beta = (a.mode == 0) ? a.st->beta : 1.0;
    if (a.mode == 0 && (mu == 0 || a.st->nonfinite)) {
        // w_p = 0 (R23) or breakdown at the seed: F = 0, eps = 0
        if (t == 0) {
            double d = 1.0;
            for (int j = 0; j < a.p; j++) {
                if (j > 0) d = d * a.tau / (double)j;
                a.combd[j] = d;
            }
            a.comb[0] = 0.0;
            AttemptResult r{};
            r.eps = 0.0; r.normH1 = 0.0; r.beta = beta; r.h = 0.0; r.mu = 0;
            r.brk = s_brk; r.status = a.st->nonfinite ? 5 : 0;
            r.accepted = -1;                         // no device decision: the host decides and launches
            if (a.dec) a.dec[0] = -a.seq;
            publish_result(a.res, r, a.seq);
        }
        return;
    }
    const int Kp = (K + 7) & ~7;                         // padded to the DMMA tile size
    const int ld = expm_ld(Kp);                          // bank-conflict-free DMMA fragment loads
    const size_t KK = (size_t)ld * Kp;
    double *base = SMEM ? esm : a.scratch;          // compile-time address space (LDS/STS when SMEM)
    double *M0 = base, *M1 = base + KK, *M2 = base + 2 * KK, *M3 = base + 3 * KK, *M4 = base + 4 * KK,
           *M5 = base + 5 * KK;
    // build the matrix to exponentiate (zero padded to Kp)
    for (size_t e = t; e < KK; e += blockDim.x) M0[e] = 0.0;
    __syncthreads();
    if (a.mode == 1) {
        for (size_t e = t; e < (size_t)K * K; e += blockDim.x) {
            const int i = (int)(e % K), jc = (int)(e / K);
            M0[i + (size_t)jc * ld] = a.Ain[e];
        }
    } else {
        // tau H_mu into M0 and ||H_mu||_1 (unscaled, for the cost model, R20): one thread per column reads
        // only the column's Hessenberg part (Lanczos: the tridiagonal band; entries below the subdiagonal are
        // never written by the Krylov kernels and are zero by definition) and sums |h| in row order, the
        // order of a full column sum (the zeros add nothing)
        double m = 0.0;
        for (int jc = t; jc < mu; jc += blockDim.x) {
            const int i0 = a.tridiag ? max(jc - 1, 0) : 0, i1 = min(jc + 1, mu - 1);
            double s = 0.0;
#pragma unroll 8
            for (int i = i0; i <= i1; i++) {
                const double hv = a.H[i + (size_t)jc * a.ldh];
                M0[i + (size_t)jc * ld] = a.tau * hv;
                s += fabs(hv);
            }
            m = fmax(m, s);
        }
        if (t == 0) {
            M0[0 + (size_t)mu * ld] = 1.0;
            for (int i = 1; i <= a.p; i++) M0[(mu + i - 1) + (size_t)(mu + i) * ld] = 1.0;
        }
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if ((t & 31) == 0) sred[t >> 5] = m;
    }
    __syncthreads();
    double normH1 = 0.0;
    if (a.mode != 1) {
        for (int w = 0; w < EXPM_NT / 32; w++) normH1 = fmax(normH1, sred[w]);
        __syncthreads();
    }
    __shared__ int s_status;
    if (t == 0) s_status = 0;
    __syncthreads();
    if (clk && t == 0) clk[1] = clock64();
    int status = 0;
    double *E;
    if constexpr (PADE) E = cta_expm_pade(K, Kp, ld, M0, M1, M2, M3, M4, M5, sred, s_int, fcol, &status, clk);
    else E = cta_expm(K, Kp, ld, M0, M1, M2, M3, M4, M5, sred, &status, clk);
    if (clk && t == 0)
        for (int i = 0; i < 16; i++) a.clk[i] = s_clk[i];
    if (t == 0 && status) s_status = status;
    __syncthreads();
    status = s_status;
    if (a.mode == 1) {
        for (size_t e = t; e < (size_t)K * K; e += blockDim.x) {
            const int i = (int)(e % K), jc = (int)(e / K);
            a.Eout[e] = E[i + (size_t)jc * ld];
        }
        if (t == 0) {
            AttemptResult r{};
            r.status = status;
            publish_result(a.res, r, a.seq);
        }
        return;
    }
    const int cp = (a.p == 0) ? 0 : mu + a.p - 1;
    const int cp1 = mu + a.p;
    if (a.mode == 2) {
        for (int i = t; i < mu; i += blockDim.x) {
            a.phip_out[i] = E[i + (size_t)cp * ld];
            a.phip1_out[i] = E[i + (size_t)cp1 * ld];
        }
        if (t == 0) {
            AttemptResult r{};
            r.normH1 = normH1; r.status = status; r.mu = mu;
            publish_result(a.res, r, a.seq);
        }
        return;
    }
    // mode 0: error estimate and combine coefficients
    const int brk = s_brk;
    const bool corr = !(brk >= 0 && brk <= mu);          // v~_mu and h_{mu+1,mu} exist
    const double h = corr ? a.H[mu + (size_t)(mu - 1) * a.ldh] : 0.0;
    double taup = 1.0;
    for (int j = 0; j < a.p; j++) taup *= a.tau;
    const double phl = E[(mu - 1) + (size_t)cp1 * ld];
    for (int i = t; i < mu; i += blockDim.x) a.comb[i] = taup * beta * E[i + (size_t)cp * ld] * a.sigma[i];
    __shared__ int s_fin;
    if (t == 0) s_fin = 1;
    __syncthreads();
    for (int i = t; i < mu; i += blockDim.x)
        if (!isfinite(E[i + (size_t)cp * ld])) s_fin = 0;
    __syncthreads();
    if (t == 0) {
        a.comb[mu] = corr ? taup * beta * a.tau * h * phl * a.sigma[mu] : 0.0;
        double d = 1.0;
        for (int j = 0; j < a.p; j++) {
            if (j > 0) d = d * a.tau / (double)j;
            a.combd[j] = d;
        }
        const double eps = taup * beta * a.tau * fabs(h * phl);
        AttemptResult r{};
        r.eps = eps;
        r.normH1 = normH1;
        r.beta = beta;
        r.h = h;
        r.mu = mu;
        r.brk = brk;
        r.status = a.st->aborted ? 3 : status ? status : ((s_fin && isfinite(eps) && isfinite(phl)) ? 0 : 5);
        r.accepted = -1;
        if (a.dec) {
            const double omega = __ddiv_rn(__dmul_rn(a.t_end, eps), __dmul_rn(a.tau, a.tol));
            const int acc = (r.status == 0 && omega - omega == 0.0 && omega <= 1.2) ? 1 : 0;
            a.dec[1] = mu + ((corr && h != 0.0) ? 1 : 0);       // (the host's rule for the corrector column)
            a.dec[0] = acc ? a.seq : -a.seq;
            r.accepted = acc;
        }
        // published before the kernel retires: the host can act on it right away
        publish_result(a.res, r, a.seq);
        if (a.clk) a.clk[6] = clock64();                 // (after the copy above: epilogue end)
    }
}

template <bool SMEM, bool PADE>
__global__ void __launch_bounds__(EXPM_NT, 1) expm_kernel(ExpmArgs a)
{
    extern __shared__ double esm[];
    pdl_wait();
    expm_body<SMEM, PADE>(a, esm);
}

} // namespace phipm
