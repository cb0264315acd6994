// phicheb.cuh — phi-functions of the symmetric Lanczos matrix directly.
//
// PAPER.md §5: "Perhaps it is better to compute the phi-function of H_m directly. This
// also allows us to exploit the fact that H_m is symmetric ... for instance by using rational Chebyshev
// approximants"; §3.1: "Only the last column of the matrix exponential ... is needed; it is
// natural to ask if this can be exploited", and "we generally do not require this accuracy" (full
// machine precision of a dense exponential).
//
// For a Lanczos solve H_mu = T is symmetric tridiagonal, so with T~ = (tau T - c I) / r mapping the
// Gershgorin interval [c - r, c + r] of tau T onto [-1, 1]:
//
//   phi_k(tau T) e1 = sum_j a_j^(k) T_j(T~) e1,    a^(k) = Chebyshev coefficients of phi_k(c + r x)
//
// and || sum_{j > n} a_j T_j(T~) e1 ||_2 <= sum_{j > n} |a_j| because ||T_j(T~)||_2 <= 1 (T~ symmetric
// with spectrum in [-1, 1]).  The kernel needs the two vectors Eq. (phipapprox2)/(errest) use,
// phi_p(tau T)e1 and phi_{p+1}(tau T)e1, which share one three-term recurrence
// v_{j+1} = 2 T~ v_j - v_{j-1} (mu-vectors: one warp, O(mu) per step, no K^3 products):
//   1. Gershgorin interval of tau T (the tridiagonal band), ||H_mu||_1 for the cost model (R20);
//   2. phi_p, phi_{p+1} at N Chebyshev points (scalar, stable: Taylor for |z| <= 4, exp and the
//      recurrence phi_{k+1}(z) = (phi_k(z) - 1/k!)/z (Eq. phirelation) beyond);
//   3. coefficients by the discrete cosine sum at the N points; truncation where |a_j| drops below
//      8 u of the largest (the sums' rounding noise); N ~ 10.5 sqrt(r) + 32 (the decay of I_j(r), e^{r x}'s coefficients),
//      N <= CHEB_NMAX, else status 7 and the host runs the augmented exponential instead;
//   4. the recurrence on warp 0 (rows 4l..4l+3 per lane, two shuffles per step);
//   5. the same epilogue as expm_kernel (error estimate, combine coefficients, published result).
#pragma once

#include "expm.cuh"

namespace phipm {

constexpr int CHEB_NT = 256;
constexpr int CHEB_NMAX = 512;
constexpr int CHEB_STATUS_RANGE = 7;      // interval too wide for CHEB_NMAX points: use the augmented expm

// reciprocals 1/i, i < 48 (no fp64 division in the scalar phi loops)
__constant__ double c_recip[48] = {
    0.0, 1.0, 1.0 / 2, 1.0 / 3, 1.0 / 4, 1.0 / 5, 1.0 / 6, 1.0 / 7, 1.0 / 8, 1.0 / 9, 1.0 / 10, 1.0 / 11,
    1.0 / 12, 1.0 / 13, 1.0 / 14, 1.0 / 15, 1.0 / 16, 1.0 / 17, 1.0 / 18, 1.0 / 19, 1.0 / 20, 1.0 / 21,
    1.0 / 22, 1.0 / 23, 1.0 / 24, 1.0 / 25, 1.0 / 26, 1.0 / 27, 1.0 / 28, 1.0 / 29, 1.0 / 30, 1.0 / 31,
    1.0 / 32, 1.0 / 33, 1.0 / 34, 1.0 / 35, 1.0 / 36, 1.0 / 37, 1.0 / 38, 1.0 / 39, 1.0 / 40, 1.0 / 41,
    1.0 / 42, 1.0 / 43, 1.0 / 44, 1.0 / 45, 1.0 / 46, 1.0 / 47};

// phi_k(z) for k >= 0 (PAPER.md Eq. phidef): Taylor sum_j z^j/(j+k)! for |z| <= 4 and k >= 1
// (alternating-sign loss <= phi_k(4)/phi_k(-4) ~ 55 at k = 1); otherwise e^z and the upward recurrence
// phi_{j+1} = (phi_j - 1/j!)/z, whose error growth per step is (1/j!)/(|z| phi_{j+1}(z)) <= 2.4 for
// |z| >= 4, j <= 6.
__device__ inline double phi_scalar(double z, int k)
{
    if (k >= 1 && fabs(z) <= 4.0) {
        // Horner from the far end: sum_{j=0}^{36} z^j / (j+k)!  =  (1/k!) (1 + z/(k+1) (1 + z/(k+2) (...)))
        // (4^36 / 37! < 1e-20 phi_1(-4)); the factors z/(k+j) by reciprocal multiplication
        double s = 1.0;
        for (int j = 36; j >= 1; j--) s = fma(s, z * c_recip[j + k], 1.0);
        double f = 1.0;                       // 1/k!  (k <= P_MAX + 1 = 7)
        for (int i = 2; i <= k; i++) f *= c_recip[i];
        return f * s;
    }
    double ph = exp(z), inv_fact = 1.0;       // phi_0, 1/0!
    const double iz = 1.0 / z;
    for (int j = 0; j < k; j++) {
        ph = (ph - inv_fact) * iz;
        inv_fact *= c_recip[j + 1];
    }
    return ph;
}

__global__ void __launch_bounds__(CHEB_NT, 1) phi_cheb_kernel(ExpmArgs a)
{
    __shared__ double f0[CHEB_NMAX], f1[CHEB_NMAX];        // function values at the nodes, then coefficients
    __shared__ double cs[4 * CHEB_NMAX];                   // cos(pi q / (2N)), q < 4N
    __shared__ double s_red[2 * (CHEB_NT / 32)];
    __shared__ double s_lo, s_hi, s_nh;
    __shared__ int s_n, s_mu, s_bad, s_brk;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    pdl_wait();
    __shared__ long long s_clk[16];                         // PHIPM_EXPM_CLOCKS phase stamps
    long long *clk = a.clk ? s_clk : nullptr;
#define CHEB_CLK(i) \
    if (clk && t == 0) clk[i] = clock64();
    CHEB_CLK(0)
    if (t == 0) {
        int m = a.m;
        s_brk = -1;
        if (a.mode == 0) {
            const int brk = a.st->brk;                 // (as expm_kernel: one read, breakdowns beyond m ignored)
            s_brk = (brk >= 0 && brk <= m) ? brk : -1;
            if (s_brk >= 0 && s_brk < m) m = s_brk;
        }
        s_mu = m;
        s_bad = 0;
    }
    __syncthreads();
    const int mu = s_mu, p = a.p;
    const double beta = (a.mode == 0) ? a.st->beta : 1.0;
    if (a.mode == 0 && (mu == 0 || a.st->nonfinite)) {
        if (t == 0) {                          // w_p = 0 (R23) or breakdown at the seed: F = 0, eps = 0
            double d = 1.0;
            for (int j = 0; j < p; j++) {
                if (j > 0) d = d * a.tau / (double)j;
                a.combd[j] = d;
            }
            a.comb[0] = 0.0;
            AttemptResult r{};
            r.beta = beta;
            r.brk = s_brk;
            r.status = a.st->nonfinite ? 5 : 0;
            publish_result(a.res, r, a.seq);
        }
        return;
    }
    const double tau = a.tau;
    // 1. band of T (alpha_i = T_ii, b_i = T_{i+1,i} = T_{i,i+1}), Gershgorin interval of tau T and
    //    ||T||_1 (column sums of the band: the unscaled ||H_mu||_1 of the cost model, R20)
    {
        double lo = INFINITY, hi = -INFINITY, nh = 0.0;
        for (int i = t; i < mu; i += CHEB_NT) {
            const double al = a.H[i + (size_t)i * a.ldh];
            const double bl = i > 0 ? fabs(a.H[i + (size_t)(i - 1) * a.ldh]) : 0.0;
            const double br = i + 1 < mu ? fabs(a.H[(i + 1) + (size_t)i * a.ldh]) : 0.0;
            lo = fmin(lo, tau * (al - bl - br));
            hi = fmax(hi, tau * (al + bl + br));
            nh = fmax(nh, bl + fabs(al) + br);
            if (!isfinite(al) || !isfinite(bl) || !isfinite(br)) s_bad = 1;
        }
        for (int o = 16; o > 0; o >>= 1) {
            lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
            nh = fmax(nh, __shfl_xor_sync(0xffffffffu, nh, o));
        }
        if (lane == 0) {
            s_red[warp] = lo;
            s_red[CHEB_NT / 32 + warp] = hi;
            f0[warp] = nh;
        }
        __syncthreads();
        if (t == 0) {
            double l = s_red[0], h = s_red[CHEB_NT / 32], n1 = f0[0];
            for (int w = 1; w < CHEB_NT / 32; w++) {
                l = fmin(l, s_red[w]);
                h = fmax(h, s_red[CHEB_NT / 32 + w]);
                n1 = fmax(n1, f0[w]);
            }
            s_lo = l;
            s_hi = h;
            s_nh = n1;
        }
        __syncthreads();
        CHEB_CLK(1)
        // 1b. tighten [lo, hi] to the spectrum of tau T by multisection with Sturm counts: the
        //     interpolation error is relative to max |phi_k| on the interval, attained at its upper
        //     end (phi_k is increasing on the real line), and Gershgorin's upper end can lie far
        //     above lambda_max (e^{hi - lambda_max} amplification); the lower end sets the degree.
        //     Round 1: 256 common points; round 2 (if a bracket is still wider than 1): 128 points
        //     in each end's bracket.
        //     The counts run in fp32 on the band scaled by 1/max(|lo|, |hi|) (a count that is off near
        //     an eigenvalue moves a bound by ~1e-6 of the width; the bounds get a 1e-5 margin).
        float *sa = reinterpret_cast<float *>(cs), *sb2 = sa + 128;
        {
            const double scl = 1.0 / fmax(fmax(fabs(s_lo), fabs(s_hi)), 1e-300);
            for (int i = t; i < mu; i += CHEB_NT) {
                sa[i] = (float)(tau * a.H[i + (size_t)i * a.ldh] * scl);
                const double bb = i + 1 < mu ? tau * a.H[(i + 1) + (size_t)i * a.ldh] * scl : 0.0;
                sb2[i] = (float)(bb * bb);
            }
        }
        __syncthreads();
        if (!s_bad && mu > 1 && s_hi > s_lo) {
            const double scl = 1.0 / fmax(fmax(fabs(s_lo), fabs(s_hi)), 1e-300);
            auto below = [&](double xd) {           // eigenvalues of tau T below x (Sturm sequence)
                const float x = (float)(xd * scl);
                int cnt = 0;
                float q = sa[0] - x;
                cnt += q < 0.0f;
                for (int i = 1; i < mu; i++) {
                    if (q == 0.0f) q = 1e-30f;
                    q = (sa[i] - x) - __fdividef(sb2[i - 1], q);
                    cnt += q < 0.0f;
                }
                return cnt;
            };
            __shared__ int s_up, s_dn;
            const double lo0 = s_lo, w0 = s_hi - s_lo;
            if (t == 0) { s_up = CHEB_NT; s_dn = -1; }
            __syncthreads();
            const double x = lo0 + w0 * (double)(t + 1) / (double)(CHEB_NT + 1);
            const int cb = below(x);
            if (cb == mu) atomicMin(&s_up, t);              // every eigenvalue below x: upper bound
            if (cb == 0) atomicMax(&s_dn, t);               // none below x: lower bound
            __syncthreads();
            const double h1 = w0 / (double)(CHEB_NT + 1);
            double up_hi = s_up < CHEB_NT ? lo0 + w0 * (double)(s_up + 1) / (double)(CHEB_NT + 1) : s_hi;
            double dn_lo = s_dn >= 0 ? lo0 + w0 * (double)(s_dn + 1) / (double)(CHEB_NT + 1) : s_lo;
            __syncthreads();
            if (h1 > 1.0) {
                // round 2: threads < 128 refine the upper bracket [up_hi - h1, up_hi], the others the
                // lower bracket [dn_lo, dn_lo + h1]
                if (t == 0) { s_up = CHEB_NT; s_dn = -1; }
                __syncthreads();
                const int half = CHEB_NT / 2, j = t & (half - 1);
                const double h2 = h1 / (double)(half + 1);
                if (t < half) {
                    const double xu = up_hi - h1 + h2 * (double)(j + 1);
                    if (below(xu) == mu) atomicMin(&s_up, j);
                } else {
                    const double xd = dn_lo + h2 * (double)(j + 1);
                    if (below(xd) == 0) atomicMax(&s_dn, j);
                }
                __syncthreads();
                if (s_up < CHEB_NT) up_hi = up_hi - h1 + h2 * (double)(s_up + 1);
                if (s_dn >= 0) dn_lo = dn_lo + h2 * (double)(s_dn + 1);
            }
            __syncthreads();
            if (t == 0) {
                const double mg = 1e-5 * (s_hi - s_lo);
                s_lo = fmax(s_lo, dn_lo - mg);
                s_hi = fmin(s_hi, up_hi + mg);
            }
        }
        __syncthreads();
        if (t == 0) {
            // nodes: 10.5 sqrt(r) + 32 (e^{r x}'s Chebyshev coefficients I_j(r) fall below 1e-18 of the
            // largest near j = 9.3 sqrt(r)), rounded up to a multiple of 32
            const double r = 0.5 * (s_hi - s_lo);
            const double ne = 10.5 * sqrt(fmax(r, 0.0)) + 32.0;
            s_n = (isfinite(ne) && ne <= (double)CHEB_NMAX) ? (((int)ne + 31) & ~31) : -1;
        }
        __syncthreads();
    }
    CHEB_CLK(2)
    const double normH1 = s_nh;
    const double c = 0.5 * (s_lo + s_hi);
    double r = 0.5 * (s_hi - s_lo);
    if (!(r > 1e-8 * fmax(fabs(c), 1.0))) r = 1e-8 * fmax(fabs(c), 1.0);   // (near) point spectrum
    const int N = s_n;
    int status = 0;
    if (s_bad) status = 5;
    else if (N < 0) status = CHEB_STATUS_RANGE;
    if (status) {
        if (t == 0) {
            AttemptResult res{};
            res.normH1 = normH1;
            res.beta = beta;
            res.mu = mu;
            res.brk = a.mode == 0 ? a.st->brk : -1;
            res.status = status;
            publish_result(a.res, res, a.seq);
        }
        return;
    }
    // 2. phi_p and phi_{p+1} at the Chebyshev points x_q = cos(pi (q + 1/2) / N); the cosine table
    for (int q = t; q < 4 * N; q += CHEB_NT) cs[q] = cospi((double)q / (double)(2 * N));
    for (int q = t; q < N; q += CHEB_NT) {
        const double x = cospi(((double)q + 0.5) / (double)N);
        const double z = c + r * x;
        f0[q] = phi_scalar(z, p);
        f1[q] = phi_scalar(z, p + 1);
    }
    __syncthreads();
    CHEB_CLK(3)
    // 3. a_j = (2/N) sum_q f(x_q) cos(pi j (2q+1) / (2N)), a_0 halved
    double aj0[CHEB_NMAX / CHEB_NT], aj1[CHEB_NMAX / CHEB_NT];
#pragma unroll
    for (int u = 0; u < CHEB_NMAX / CHEB_NT; u++) {
        const int j = t + u * CHEB_NT;
        double s0 = 0.0, s1 = 0.0;
        if (j < N) {
            int idx = j % (4 * N), step = (2 * j) % (4 * N);       // j (2q + 1) mod 4N
            for (int q = 0; q < N; q++) {
                const double cv = cs[idx];
                s0 = fma(f0[q], cv, s0);
                s1 = fma(f1[q], cv, s1);
                idx += step;
                if (idx >= 4 * N) idx -= 4 * N;
            }
            const double sc = (j == 0 ? 1.0 : 2.0) / (double)N;
            s0 *= sc;
            s1 *= sc;
        }
        aj0[u] = s0;
        aj1[u] = s1;
    }
    __syncthreads();                                        // f0/f1 are overwritten with the coefficients
    CHEB_CLK(4)
    double amax = 0.0;
#pragma unroll
    for (int u = 0; u < CHEB_NMAX / CHEB_NT; u++) {
        const int j = t + u * CHEB_NT;
        if (j < N) {
            f0[j] = aj0[u];
            f1[j] = aj1[u];
            amax = fmax(amax, fmax(fabs(aj0[u]), fabs(aj1[u])));
        }
    }
    for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if (lane == 0) s_red[warp] = amax;
    __syncthreads();
    if (t == 0) {
        double m = 0.0;
        for (int w = 0; w < CHEB_NT / 32; w++) m = fmax(m, s_red[w]);
        s_red[0] = m;
    }
    __syncthreads();
    // truncation degree: last j with |a_j| > 8 u max |a| (the cosine sums carry rounding noise of a few
    // u max |f|; past the true decay the coefficients are noise, and their sum is below 1e-13 max |f|)
    {
        const double thr = s_red[0] * 8.8817841970012523e-16;
        int last = 0;
#pragma unroll
        for (int u = 0; u < CHEB_NMAX / CHEB_NT; u++) {
            const int j = t + u * CHEB_NT;
            if (j < N && (fabs(f0[j]) > thr || fabs(f1[j]) > thr)) last = j;
        }
        for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
        __syncthreads();
        if (lane == 0) ((int *)s_red)[warp] = last;
        __syncthreads();
        if (t == 0) {
            int l = 0;
            for (int w = 0; w < CHEB_NT / 32; w++) l = max(l, ((int *)s_red)[w]);
            s_n = l;
        }
        __syncthreads();
    }
    const int nd = s_n;
    CHEB_CLK(5)
    // 4. recurrence on warp 0: lane holds rows 4 lane .. 4 lane + 3 (mu <= 128)
    __shared__ double s_noise;
    if (warp == 0) {
        __syncwarp();                                       // converged: the shuffles take the fast path
        double d[4], e[4], v0[4], v1[4], acc0[4], acc1[4];
        // magnitudes for the rounding-noise bound of the last component (the error estimate's input):
        // sa1 = sum_j |a_j^(p+1)| |v_j[i]|, sv = sum_j |v_j[i]|
        double sa1[4], sv[4];
        const double ir = 1.0 / r;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int i = 4 * lane + k;
            d[k] = i < mu ? (tau * a.H[i + (size_t)i * a.ldh] - c) * ir : 0.0;
            e[k] = i + 1 < mu ? tau * a.H[(i + 1) + (size_t)i * a.ldh] * ir : 0.0;   // T~_{i+1,i} = T~_{i,i+1}
            v0[k] = (i == 0) ? 1.0 : 0.0;                  // T_0(T~) e1
        }
        // v1 = T~ e1
        double em1 = __shfl_up_sync(0xffffffffu, e[3], 1);   // e_{4 lane - 1}
        if (lane == 0) em1 = 0.0;
        {
            double vl = __shfl_up_sync(0xffffffffu, v0[3], 1), vr = __shfl_down_sync(0xffffffffu, v0[0], 1);
            if (lane == 0) vl = 0.0;
            if (lane == 31) vr = 0.0;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const double left = k == 0 ? vl : v0[k - 1];
                const double right = k == 3 ? vr : v0[k + 1];
                const double el = k == 0 ? em1 : e[k - 1];
                v1[k] = el * left + d[k] * v0[k] + e[k] * right;
            }
        }
#pragma unroll
        for (int k = 0; k < 4; k++) {
            acc0[k] = f0[0] * v0[k];
            acc1[k] = f1[0] * v0[k];
            sa1[k] = fabs(f1[0] * v0[k]);
            sv[k] = fabs(v0[k]);
            if (nd >= 1) {
                acc0[k] = fma(f0[1], v1[k], acc0[k]);
                acc1[k] = fma(f1[1], v1[k], acc1[k]);
                sa1[k] = fma(fabs(f1[1]), fabs(v1[k]), sa1[k]);
                sv[k] += fabs(v1[k]);
            }
        }
        for (int j = 2; j <= nd; j++) {
            double vl = __shfl_up_sync(0xffffffffu, v1[3], 1), vr = __shfl_down_sync(0xffffffffu, v1[0], 1);
            if (lane == 0) vl = 0.0;
            if (lane == 31) vr = 0.0;
            const double c0j = f0[j], c1j = f1[j];
            double v2[4];
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const double left = k == 0 ? vl : v1[k - 1];
                const double right = k == 3 ? vr : v1[k + 1];
                const double el = k == 0 ? em1 : e[k - 1];
                const double w = el * left + d[k] * v1[k] + e[k] * right;
                v2[k] = 2.0 * w - v0[k];
            }
#pragma unroll
            for (int k = 0; k < 4; k++) {
                acc0[k] = fma(c0j, v2[k], acc0[k]);
                acc1[k] = fma(c1j, v2[k], acc1[k]);
                sa1[k] = fma(fabs(c1j), fabs(v2[k]), sa1[k]);
                sv[k] += fabs(v2[k]);
                v0[k] = v1[k];
                v1[k] = v2[k];
            }
        }
        // noise bound of [phi_{p+1}(tau T) e1]_{mu-1}: the recurrence's rounding relative to the terms
        // it sums, (nd + 1) u sum_j |a_j v_j|, plus the coefficients' cosine-sum noise, 4 u max|f| per
        // coefficient (max|f| <= sum_j |a_j|) times sum_j |v_j|.  Large when the last component is a
        // cancellation of large terms (interval half-width r > mu): then the estimate is unreliable.
        double a1s = 0.0;
        for (int j = lane; j <= nd; j += 32) a1s += fabs(f1[j]);
        for (int o = 16; o > 0; o >>= 1) a1s += __shfl_xor_sync(0xffffffffu, a1s, o);
#pragma unroll
        for (int k = 0; k < 4; k++)
            if (4 * lane + k == mu - 1)
                s_noise = 1.1102230246251565e-16 * ((double)(nd + 1) * sa1[k] + 4.0 * a1s * sv[k]);
        // results to shared memory (reuse cs): phi_p e1 in cs[0..mu), phi_{p+1} e1 in cs[128..128+mu)
#pragma unroll
        for (int k = 0; k < 4; k++) {
            cs[4 * lane + k] = acc0[k];
            cs[128 + 4 * lane + k] = acc1[k];
        }
    }
    __syncthreads();
    CHEB_CLK(6)
    if (clk && t == 0) {
        clk[7] = ((long long)N << 32) | ((long long)nd << 16) | mu;
        for (int i = 0; i < 8; i++) a.clk[i] = s_clk[i];
        for (int i = 8; i < 16; i++) a.clk[i] = -1;        // marks a Chebyshev record
        a.clk[9] = __double_as_longlong(s_lo);
        a.clk[10] = __double_as_longlong(s_hi);
    }
    const double *php = cs, *php1 = cs + 128;
    if (a.mode == 2) {
        for (int i = t; i < mu; i += CHEB_NT) {
            a.phip_out[i] = php[i];
            a.phip1_out[i] = php1[i];
        }
        if (t == 0) {
            AttemptResult res{};
            res.normH1 = normH1;
            res.mu = mu;
            res.status = 0;
            publish_result(a.res, res, a.seq);
        }
        return;
    }
    // 5. mode 0 epilogue (as expm_kernel): error estimate and combine coefficients
    const int brk = s_brk;
    const bool corr = !(brk >= 0 && brk <= mu);
    const double h = corr ? a.H[mu + (size_t)(mu - 1) * a.ldh] : 0.0;
    double taup = 1.0;
    for (int j = 0; j < p; j++) taup *= tau;
    const double phl = php1[mu - 1];
    __shared__ int s_fin;
    if (t == 0) s_fin = 1;
    __syncthreads();
    for (int i = t; i < mu; i += CHEB_NT) {
        a.comb[i] = taup * beta * php[i] * a.sigma[i];
        if (!isfinite(php[i])) s_fin = 0;
    }
    __syncthreads();
    if (t == 0) {
        a.comb[mu] = corr ? taup * beta * tau * h * phl * a.sigma[mu] : 0.0;
        double dd = 1.0;
        for (int j = 0; j < p; j++) {
            if (j > 0) dd = dd * tau / (double)j;
            a.combd[j] = dd;
        }
        const double eps = taup * beta * tau * fabs(h * phl);
        AttemptResult res{};
        res.eps = eps;
        res.normH1 = normH1;
        res.beta = beta;
        res.h = h;
        res.mu = mu;
        res.brk = brk;
        res.status = a.st->aborted ? 3 : ((s_fin && isfinite(eps) && isfinite(phl)) ? 0 : 5);
        res.eps_noise = taup * beta * tau * fabs(h) * s_noise;
        publish_result(a.res, res, a.seq);
    }
}

} // namespace phipm
