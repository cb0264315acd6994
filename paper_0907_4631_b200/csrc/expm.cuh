// expm.cuh — single-CTA kernel for the small dense part of a phipm attempt (Sec. 3.1-3.2):
//
//   Hhat = [[tau H_mu, e1, 0], [0, 0, I_p], [0, 0, 0]]   (Eq. hathm P:368-377 with p+1)
//   E = exp(Hhat) by the degree-13 Pade approximant with scaling and squaring (Eq. 8)
//   phi_p(tau H)e1 = E[0:mu, mu+p-1] (p = 0: column 0), phi_{p+1}(tau H)e1 = E[0:mu, mu+p]
//   eps = tau^p beta tau |h_{mu+1,mu} [phi_{p+1}]_mu|                 (Eq. errest with R9/R10)
//   combine coefficients of Eq. (step)/(phipapprox2) for the assembly kernel.
//
// All K x K matrices (K <= m_max + p_max + 1) live in shared memory when 6 K^2 doubles fit,
// otherwise in an L2-resident global scratch; generic addressing serves both.  The linear solve
// (V - U) X = (V + U) uses Gauss-Jordan elimination with partial pivoting (parallel over the
// CTA; the oracle uses LU with triangular solves — same pivoting, different operation order).
#pragma once

#include "kernels.cuh"

namespace phipm {

constexpr int EXPM_NT = 512;

// result block read by the host controller (mapped pinned memory)
struct AttemptResult {
    double eps;        // error estimate (R10)
    double normH1;     // ||H_mu||_1
    double beta;       // ||w_p||_2
    double h;          // h_{mu+1,mu} used by the corrector (0 on breakdown)
    int mu;            // Krylov dimension used
    int brk;           // -1 or the breakdown position
    int status;        // 0 ok, 5 non-finite, 6 singular
    int seq;           // attempt sequence number (host sanity check)
};

struct ExpmArgs {
    int mode;          // 0: phipm attempt; 1: plain expm of Ain; 2: phi pair of H (mu = m)
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
};

// C = A B (K x K, column-major); two accumulators to shorten the dependent FMA chain
__device__ __forceinline__ void cta_matmul(int K, const double *A, const double *B, double *C)
{
    const int KK = K * K;
    for (int o = threadIdx.x; o < KK; o += blockDim.x) {
        const int i = o % K, jc = o / K;
        const double *a = A + i;
        const double *b = B + (size_t)jc * K;
        double s0 = 0.0, s1 = 0.0;
        int l = 0;
        for (; l + 1 < K; l += 2) {
            s0 = fma(a[(size_t)l * K], b[l], s0);
            s1 = fma(a[(size_t)(l + 1) * K], b[l + 1], s1);
        }
        if (l < K) s0 = fma(a[(size_t)l * K], b[l], s0);
        C[o] = s0 + s1;
    }
    __syncthreads();
}

__device__ __forceinline__ double block_max_colsum(int K, const double *A, double *sred)
{
    // ||A||_1 = max_j sum_i |a_ij|
    double m = 0.0;
    for (int jc = threadIdx.x; jc < K; jc += blockDim.x) {
        double s = 0.0;
        for (int i = 0; i < K; i++) s += fabs(A[i + (size_t)jc * K]);
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

// exp(M0) -> returned pointer (one of the buffers); M0..M5 are K x K buffers.  status: 0/5/6
__device__ double *cta_expm(int K, double *M0, double *M1, double *M2, double *M3, double *M4, double *M5,
                            double *sred, int *s_int, int *status)
{
    const int KK = K * K, t = threadIdx.x;
    double c[14];
    pade13(c);
    // scaling: s = ceil_+(log2(||A||_1 / 5.37)) (theta_13 = 5.37 as printed, R26)
    const double nrm = block_max_colsum(K, M0, sred);
    int s = 0;
    if (nrm > 0.0) {
        const double l = ceil(log2(nrm / 5.37));
        s = l > 0.0 ? (int)l : 0;
    }
    if (!isfinite(nrm)) { *status = 5; return M0; }
    const double sc = ldexp(1.0, -s);
    for (int e = t; e < KK; e += blockDim.x) M0[e] *= sc;
    __syncthreads();
    cta_matmul(K, M0, M0, M1);            // A2
    cta_matmul(K, M1, M1, M2);            // A4
    cta_matmul(K, M2, M1, M3);            // A6
    // U = A [A6 (c13 A6 + c11 A4 + c9 A2) + c7 A6 + c5 A4 + c3 A2 + c1 I]
    for (int e = t; e < KK; e += blockDim.x) M4[e] = c[13] * M3[e] + c[11] * M2[e] + c[9] * M1[e];
    __syncthreads();
    cta_matmul(K, M3, M4, M5);
    for (int e = t; e < KK; e += blockDim.x) {
        double v = M5[e] + c[7] * M3[e] + c[5] * M2[e] + c[3] * M1[e];
        if (e % (K + 1) == 0) v += c[1];
        M5[e] = v;
    }
    __syncthreads();
    cta_matmul(K, M0, M5, M4);            // U in M4
    // V = A6 (c12 A6 + c10 A4 + c8 A2) + c6 A6 + c4 A4 + c2 A2 + c0 I
    for (int e = t; e < KK; e += blockDim.x) M5[e] = c[12] * M3[e] + c[10] * M2[e] + c[8] * M1[e];
    __syncthreads();
    cta_matmul(K, M3, M5, M0);            // A no longer needed
    for (int e = t; e < KK; e += blockDim.x) {
        double v = M0[e] + c[6] * M3[e] + c[4] * M2[e] + c[2] * M1[e];
        if (e % (K + 1) == 0) v += c[0];
        M0[e] = v;                        // V
    }
    __syncthreads();
    // P = V + U (M1), Q = V - U (M2)
    for (int e = t; e < KK; e += blockDim.x) {
        const double v = M0[e], u = M4[e];
        M1[e] = v + u;
        M2[e] = v - u;
    }
    __syncthreads();
    // Gauss-Jordan with partial pivoting: Q X = P, X overwrites P
    double *Q = M2, *P = M1;
    for (int col = 0; col < K; col++) {
        if (t < 32) {
            double best = -1.0;
            int bi = col;
            for (int r = col + t; r < K; r += 32) {
                const double a = fabs(Q[r + (size_t)col * K]);
                if (a > best) { best = a; bi = r; }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
            }
            if (t == 0) {
                s_int[0] = bi;
                s_int[1] = (best >= 1e-300) ? 0 : 1;
            }
        }
        __syncthreads();
        if (s_int[1]) { *status = 6; return P; }
        const int pr = s_int[0];
        if (pr != col) {
            for (int jc = t; jc < 2 * K; jc += blockDim.x) {
                double *Mx = (jc < K) ? Q : P;
                const int cc = (jc < K) ? jc : jc - K;
                const double tmp = Mx[col + (size_t)cc * K];
                Mx[col + (size_t)cc * K] = Mx[pr + (size_t)cc * K];
                Mx[pr + (size_t)cc * K] = tmp;
            }
        }
        __syncthreads();
        // eliminate column col from every other row, using the unscaled pivot row
        const double piv = Q[col + (size_t)col * K];
        const int ncolq = K - col - 1;
        const int width = ncolq + K;                   // Q columns col+1..K-1, then P columns
        const int work = (K - 1) * width;
        for (int w = t; w < work; w += blockDim.x) {
            int r = w % (K - 1);
            const int cc = w / (K - 1);
            if (r >= col) r++;                          // skip the pivot row
            const double f = Q[r + (size_t)col * K] / piv;
            if (cc < ncolq) {
                const int qc = col + 1 + cc;
                Q[r + (size_t)qc * K] -= f * Q[col + (size_t)qc * K];
            } else {
                const int pc = cc - ncolq;
                P[r + (size_t)pc * K] -= f * P[col + (size_t)pc * K];
            }
        }
        __syncthreads();
        // scale the pivot row (Q part right of the pivot is no longer needed except by later
        // pivots' eliminations, which read row col's Q entries only for columns > col)
        for (int jc = t; jc < width; jc += blockDim.x) {
            if (jc < ncolq) Q[col + (size_t)(col + 1 + jc) * K] /= piv;
            else P[col + (size_t)(jc - ncolq) * K] /= piv;
        }
        __syncthreads();
    }
    // squaring
    double *X = P, *T = M3;
    for (int q = 0; q < s; q++) {
        cta_matmul(K, X, X, T);
        double *tmp = X; X = T; T = tmp;
    }
    return X;
}

__global__ void __launch_bounds__(EXPM_NT) expm_kernel(ExpmArgs a)
{
    extern __shared__ double esm[];
    __shared__ double sred[EXPM_NT / 32];
    __shared__ int s_int[4];
    __shared__ int s_mu;
    const int t = threadIdx.x;
    int mu, K;
    if (a.mode == 1) {
        mu = 0;
        K = a.K;
    } else {
        if (t == 0) {
            int m = a.m;
            if (a.mode == 0) {
                const int brk = a.st->brk;
                if (brk >= 0 && brk < m) m = brk;
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
            AttemptResult r;
            r.eps = 0.0; r.normH1 = 0.0; r.beta = beta; r.h = 0.0; r.mu = 0;
            r.brk = a.st->brk; r.status = a.st->nonfinite ? 5 : 0; r.seq = a.seq;
            *a.res = r;
        }
        return;
    }
    const size_t KK = (size_t)K * K;
    double *base = a.use_smem ? esm : a.scratch;
    double *M0 = base, *M1 = base + KK, *M2 = base + 2 * KK, *M3 = base + 3 * KK, *M4 = base + 4 * KK,
           *M5 = base + 5 * KK;
    // build the matrix to exponentiate
    if (a.mode == 1) {
        for (size_t e = t; e < KK; e += blockDim.x) M0[e] = a.Ain[e];
    } else {
        for (size_t e = t; e < KK; e += blockDim.x) M0[e] = 0.0;
        __syncthreads();
        for (size_t e = t; e < (size_t)mu * mu; e += blockDim.x) {
            const int i = (int)(e % mu), jc = (int)(e / mu);
            if (!a.tridiag || (i - jc <= 1 && jc - i <= 1)) M0[i + (size_t)jc * K] = a.tau * a.H[i + (size_t)jc * a.ldh];
        }
        if (t == 0) {
            M0[0 + (size_t)mu * K] = 1.0;
            for (int i = 1; i <= a.p; i++) M0[(mu + i - 1) + (size_t)(mu + i) * K] = 1.0;
        }
    }
    __syncthreads();
    // ||H_mu||_1 (unscaled) for the cost model (R20)
    double normH1 = 0.0;
    if (a.mode != 1) {
        double m = 0.0;
        for (int jc = t; jc < mu; jc += blockDim.x) {
            double s = 0.0;
            const int i0 = a.tridiag ? max(jc - 1, 0) : 0, i1 = a.tridiag ? min(jc + 2, mu) : mu;
            for (int i = i0; i < i1; i++) s += fabs(a.H[i + (size_t)jc * a.ldh]);
            m = fmax(m, s);
        }
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if ((t & 31) == 0) sred[t >> 5] = m;
        __syncthreads();
        for (int w = 0; w < EXPM_NT / 32; w++) normH1 = fmax(normH1, sred[w]);
        __syncthreads();
    }
    __shared__ int s_status;
    if (t == 0) s_status = 0;
    __syncthreads();
    int status = 0;
    double *E = cta_expm(K, M0, M1, M2, M3, M4, M5, sred, s_int, &status);
    if (t == 0 && status) s_status = status;
    __syncthreads();
    status = s_status;
    if (a.mode == 1) {
        for (size_t e = t; e < KK; e += blockDim.x) a.Eout[e] = E[e];
        if (t == 0) {
            AttemptResult r{};
            r.status = status; r.seq = a.seq;
            *a.res = r;
        }
        return;
    }
    const int cp = (a.p == 0) ? 0 : mu + a.p - 1;
    const int cp1 = mu + a.p;
    if (a.mode == 2) {
        for (int i = t; i < mu; i += blockDim.x) {
            a.phip_out[i] = E[i + (size_t)cp * K];
            a.phip1_out[i] = E[i + (size_t)cp1 * K];
        }
        if (t == 0) {
            AttemptResult r{};
            r.normH1 = normH1; r.status = status; r.mu = mu; r.seq = a.seq;
            *a.res = r;
        }
        return;
    }
    // mode 0: error estimate and combine coefficients
    const int brk = a.st->brk;
    const bool corr = !(brk >= 0 && brk <= mu);          // v~_mu and h_{mu+1,mu} exist
    const double h = corr ? a.H[mu + (size_t)(mu - 1) * a.ldh] : 0.0;
    double taup = 1.0;
    for (int j = 0; j < a.p; j++) taup *= a.tau;
    const double phl = E[(mu - 1) + (size_t)cp1 * K];
    for (int i = t; i < mu; i += blockDim.x) a.comb[i] = taup * beta * E[i + (size_t)cp * K] * a.sigma[i];
    __shared__ int s_fin;
    if (t == 0) s_fin = 1;
    __syncthreads();
    for (int i = t; i < mu; i += blockDim.x)
        if (!isfinite(E[i + (size_t)cp * K])) s_fin = 0;
    __syncthreads();
    if (t == 0) {
        a.comb[mu] = corr ? taup * beta * a.tau * h * phl * a.sigma[mu] : 0.0;
        double d = 1.0;
        for (int j = 0; j < a.p; j++) {
            if (j > 0) d = d * a.tau / (double)j;
            a.combd[j] = d;
        }
        const double eps = taup * beta * a.tau * fabs(h * phl);
        AttemptResult r;
        r.eps = eps;
        r.normH1 = normH1;
        r.beta = beta;
        r.h = h;
        r.mu = mu;
        r.brk = brk;
        r.status = status ? status : ((s_fin && isfinite(eps) && isfinite(phl)) ? 0 : 5);
        r.seq = a.seq;
        *a.res = r;
    }
}

} // namespace phipm
