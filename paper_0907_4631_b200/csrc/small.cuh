// small.cuh — the whole Krylov extension k0 -> k1 (Algorithm 1 in CGS form / Algorithm 2) in ONE
// single-CTA kernel, for small n (n <= SMALL_N).  At that size every step is latency-bound: two
// grid-wide kernels per step cost far more in launch and reduction tails than the work itself,
// while one CTA keeps y in shared memory and V in L2 and synchronises with block barriers only.
// Arithmetic per step is the same as the streaming kernels (same unnormalised basis, sigma
// scaling, finalize formulas), and rows are summed in ascending column order.
#pragma once

#include "kernels.cuh"

namespace phipm {

constexpr int SMALL_N = 8192;
constexpr int SMALL_NT = 1024;

struct SmallArgs {
    int k0, k1;          // extend the basis from k0 to k1 columns of H
    int symmetric;       // Lanczos (Alg. 2) or Arnoldi (Alg. 1, CGS)
    int orth;            // PHIPM_ORTH_CGS2: second CGS pass per step
    double bthr;         // breakdown threshold
};

// (A x)_r, ascending column order with separately rounded products (= sequential CSR row sum)
__device__ __forceinline__ double row_apply(const StencilOp &S, const double *__restrict__ x, int64_t r)
{
    if (S.dim == 1) {                                    // no grid coordinates to recover
        double s = 0.0;
        if (r > 0) s = __dadd_rn(s, __dmul_rn(S.c[1], x[r - 1]));
        s = __dadd_rn(s, __dmul_rn(S.c[0], x[r]));
        if (r < S.nx - 1) s = __dadd_rn(s, __dmul_rn(S.c[2], x[r + 1]));
        return s;
    }
    const unsigned ur = (unsigned)r, unx = (unsigned)S.nx;
    const unsigned q = ur / unx;
    const int i = (int)(ur - q * unx);
    int jj = 0, kk = 0;
    if (S.dim >= 2) {
        const unsigned uny = (unsigned)S.ny;
        const unsigned q2 = q / uny;
        jj = (int)(q - q2 * uny);
        kk = (int)q2;
    }
    const int64_t pl = (int64_t)S.nx * S.ny;
    const bool dg = S.diag != 0;
    double s = 0.0;
    if (S.dim >= 3 && kk > 0) s = __dadd_rn(s, __dmul_rn(S.c[5], x[r - pl]));
    if (dg && jj > 0 && i > 0) s = __dadd_rn(s, __dmul_rn(S.c[7], x[r - S.nx - 1]));
    if (S.dim >= 2 && jj > 0) s = __dadd_rn(s, __dmul_rn(S.c[3], x[r - S.nx]));
    if (dg && jj > 0 && i < S.nx - 1) s = __dadd_rn(s, __dmul_rn(S.c[8], x[r - S.nx + 1]));
    if (i > 0) s = __dadd_rn(s, __dmul_rn(S.c[1], x[r - 1]));
    s = __dadd_rn(s, __dmul_rn(S.c[0], x[r]));
    if (i < S.nx - 1) s = __dadd_rn(s, __dmul_rn(S.c[2], x[r + 1]));
    if (dg && jj < S.ny - 1 && i > 0) s = __dadd_rn(s, __dmul_rn(S.c[9], x[r + S.nx - 1]));
    if (S.dim >= 2 && jj < S.ny - 1) s = __dadd_rn(s, __dmul_rn(S.c[4], x[r + S.nx]));
    if (dg && jj < S.ny - 1 && i < S.nx - 1) s = __dadd_rn(s, __dmul_rn(S.c[10], x[r + S.nx + 1]));
    if (S.dim >= 3 && kk < S.nz - 1) s = __dadd_rn(s, __dmul_rn(S.c[6], x[r + pl]));
    return s;
}

__device__ __forceinline__ double row_apply(const CsrOp &A, const double *__restrict__ x, int64_t r)
{
    double s = 0.0;
    for (int e = A.rp[r]; e < A.rp[r + 1]; e++) s = __dadd_rn(s, __dmul_rn(A.val[e], x[A.col[e]]));
    return s;
}

__device__ __forceinline__ double row_apply(const IdentOp &, const double *__restrict__ x, int64_t r) { return x[r]; }

// block sum with one barrier: the caller alternates two scratch arrays, so the array written here
// was last read two sums ago, before the barrier of the sum in between
__device__ __forceinline__ double block_sum1(double v, double *red)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    return warp_sum(lane < nw ? red[lane] : 0.0);
}

// block sum of one value per thread (all threads receive the same total: a warp shuffle tree over
// the warp totals, identical in every warp)
__device__ __forceinline__ double block_sum(double v, double *red)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    return warp_sum(lane < nw ? red[lane] : 0.0);
}

// Lanczos (Alg. 2) for n <= SLZ_NT * SLZ_R in a single CTA of SLZ_NT threads with up to SLZ_R rows
// per thread (rows t + SLZ_NT i).  The step is a chain of two dependent block sums; with 8 warps
// instead of 32 each sum has a 3-level second stage and a cheaper barrier, and a thread's rows give
// the SpMV some instruction-level parallelism.  Arithmetic per row is that of krylov_small_kernel
// (the dot and norm are summed in another order).
constexpr int SLZ_NT = 256;
constexpr int SLZ_R = 4;

template <class Op>
__global__ void __launch_bounds__(SLZ_NT) krylov_small_lanczos_kernel(Op op, SmallArgs a, Work wk)
{
    extern __shared__ double vs[];                      // n doubles: v~_j
    __shared__ double red[SLZ_NT / 32];
    __shared__ double red2[SLZ_NT / 32];
    const int t = threadIdx.x;
    const int n = (int)op.n;
    pdl_wait();
    double sj = wk.sigma[a.k0];
    double lz = wk.st->lz;
    int brk = wk.st->brk;
    double zv[SLZ_R];
#pragma unroll
    for (int i = 0; i < SLZ_R; i++) {
        const int r = t + SLZ_NT * i;
        zv[i] = 0.0;
        if (r < n) {
            vs[r] = wk.V[(int64_t)a.k0 * wk.ldv + r];
            if (a.k0 > 0) zv[i] = wk.V[(int64_t)(a.k0 - 1) * wk.ldv + r];
        }
    }
    __syncthreads();
    for (int j = a.k0; j < a.k1 && brk < 0; j++) {
        double y[SLZ_R], xv[SLZ_R];
        double dl = 0.0;
#pragma unroll
        for (int i = 0; i < SLZ_R; i++) {
            const int r = t + SLZ_NT * i;
            y[i] = 0.0;
            xv[i] = 0.0;
            if (r < n) {
                y[i] = sj * row_apply(op, vs, r);
                xv[i] = vs[r];
                if (j > 0) y[i] = fma(-lz, zv[i], y[i]);
            }
            dl = fma(xv[i], y[i], dl);
        }
        const double d = block_sum1(dl, red);
        const double al = sj * d;                          // t_jj = sigma_j v~_j^T y
        const double g = al * sj;
        double wl = 0.0;
#pragma unroll
        for (int i = 0; i < SLZ_R; i++) {
            const int r = t + SLZ_NT * i;
            if (r < n) {
                const double w = fma(-g, xv[i], y[i]);     // v~_{j+1} = y - g v~_j
                wk.V[(int64_t)(j + 1) * wk.ldv + r] = w;
                vs[r] = w;                                 // every thread has read vs (block sum above)
                wl = fma(w, w, wl);
            }
            zv[i] = xv[i];
        }
        const double tot = block_sum1(wl, red2);
        const double h = sqrt(tot);
        const double sn = 1.0 / h;
        const double lzn = h * sj;
        int b = -1;
        if (!isfinite(h)) b = j + 1;
        else if (h <= a.bthr) b = j + 1;
        if (t == 0) {
            wk.H[j + (size_t)j * wk.ldh] = al;
            wk.g[0] = g;
            wk.H[(j + 1) + (size_t)j * wk.ldh] = h;
            if (j + 1 < wk.hcols) wk.H[j + (size_t)(j + 1) * wk.ldh] = h;
            wk.st->lz = lzn;
            wk.sigma[j + 1] = sn;
            if (!isfinite(h)) wk.st->nonfinite = 1;
            if (b >= 0) wk.st->brk = b;
        }
        sj = sn;
        lz = lzn;
        brk = b;
    }
}

template <class Op>
__global__ void __launch_bounds__(SMALL_NT) krylov_small_kernel(Op op, SmallArgs a, Work wk)
{
    extern __shared__ double ys[];                      // n doubles (dynamic)
    __shared__ double dres[MAXD + 2];
    __shared__ double gs[MAXD + 2];
    __shared__ double red[SMALL_NT / 32];
    __shared__ double red2[SMALL_NT / 32];
    __shared__ int s_brk;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = SMALL_NT / 32;
    const int n = (int)op.n;
    pdl_wait();
    if (t == 0) s_brk = wk.st->brk;
    __syncthreads();
    if (a.symmetric && n <= SMALL_NT) {
        // Lanczos with one row per thread: every reduction is a block sum whose total every thread
        // receives, so alpha, g, h, sigma and the breakdown test are computed by all threads alike
        // (no single-thread stage between barriers); thread 0 writes them for the host / expm.
        // v~_j lives in shared memory (the SpMV's neighbour reads are shared-memory loads, not L2
        // round trips on a vector written a step ago) and v~_{j-1} of this thread's row in a register.
        extern __shared__ double vs[];                   // n doubles: v~_j
        double sj = wk.sigma[a.k0];
        double lz = wk.st->lz;
        int brk = s_brk;
        double zv = 0.0;
        if (t < n) {
            vs[t] = wk.V[(int64_t)a.k0 * wk.ldv + t];
            if (a.k0 > 0) zv = wk.V[(int64_t)(a.k0 - 1) * wk.ldv + t];
        }
        __syncthreads();
        for (int j = a.k0; j < a.k1 && brk < 0; j++) {
            double y = 0.0, xv = 0.0;
            if (t < n) {
                y = sj * row_apply(op, vs, t);
                xv = vs[t];
                if (j > 0) y = fma(-lz, zv, y);
            }
            const double d = block_sum1(xv * y, red);
            const double al = sj * d;                      // t_jj = sigma_j v~_j^T y
            const double g = al * sj;
            double w = 0.0;
            if (t < n) {
                w = fma(-g, xv, y);                        // v~_{j+1} = y - g v~_j
                wk.V[(int64_t)(j + 1) * wk.ldv + t] = w;
                vs[t] = w;                                 // every thread has read vs (block sum above)
            }
            zv = xv;
            const double tot = block_sum1(w * w, red2);
            const double h = sqrt(tot);
            const double sn = 1.0 / h;
            const double lzn = h * sj;
            int b = -1;
            if (!isfinite(h)) b = j + 1;
            else if (h <= a.bthr) b = j + 1;
            if (t == 0) {
                wk.H[j + (size_t)j * wk.ldh] = al;
                wk.g[0] = g;
                wk.H[(j + 1) + (size_t)j * wk.ldh] = h;
                if (j + 1 < wk.hcols) wk.H[j + (size_t)(j + 1) * wk.ldh] = h;
                wk.st->lz = lzn;
                wk.sigma[j + 1] = sn;
                if (!isfinite(h)) wk.st->nonfinite = 1;
                if (b >= 0) wk.st->brk = b;
            }
            sj = sn;
            lz = lzn;
            brk = b;
        }
        return;
    }
    for (int j = a.k0; j < a.k1; j++) {
        if (s_brk >= 0) break;                           // uniform: written before the last barrier
        const double *vj = wk.V + (int64_t)j * wk.ldv;
        const double sj = wk.sigma[j];
        const double lz = (a.symmetric && j > 0) ? wk.st->lz : 0.0;
        const double *vjm = (a.symmetric && j > 0) ? vj - wk.ldv : nullptr;
        // y = sigma_j A v~_j  [- h_{j,j-1} sigma_{j-1} v~_{j-1}]
        for (int r = t; r < n; r += SMALL_NT) {
            double y = sj * row_apply(op, vj, r);
            if (vjm) y = fma(-lz, vjm[r], y);
            ys[r] = y;
        }
        __syncthreads();
        // dot products with the basis columns (Arnoldi: 0..j, Lanczos: j), one warp per column
        const int c0 = a.symmetric ? j : 0;
        const int nd = j - c0 + 1;
        for (int kk = warp; kk < nd; kk += nw) {
            const double *vc = wk.V + (int64_t)(c0 + kk) * wk.ldv;
            double d0 = 0.0, d1 = 0.0;
            int r = lane;
            for (; r + 32 < n; r += 64) {
                d0 = fma(vc[r], ys[r], d0);
                d1 = fma(vc[r + 32], ys[r + 32], d1);
            }
            if (r < n) d0 = fma(vc[r], ys[r], d0);
            const double d = warp_sum(d0 + d1);
            if (lane == 0) dres[kk] = d;
        }
        __syncthreads();
        if (a.symmetric) {
            if (t == 0) {
                const double al = wk.sigma[j] * dres[0];
                wk.H[j + (size_t)j * wk.ldh] = al;
                gs[0] = al * wk.sigma[j];
            }
        } else {
            for (int k = t; k < nd; k += SMALL_NT) {
                const double h = wk.sigma[k] * dres[k];
                wk.H[k + (size_t)j * wk.ldh] = h;
                gs[k] = h * wk.sigma[k];
            }
        }
        __syncthreads();
        // v~_{j+1} = y - sum_k g_k v~_k, ||v~_{j+1}||^2
        double *vn = wk.V + (int64_t)(j + 1) * wk.ldv;
        double nrm = 0.0;
        for (int r = t; r < n; r += SMALL_NT) {
            double v = ys[r];
#pragma unroll 8
            for (int k = 0; k < nd; k++) v = fma(-gs[k], wk.V[r + (int64_t)(c0 + k) * wk.ldv], v);
            vn[r] = v;
            nrm = fma(v, v, nrm);
        }
        double tot = block_sum(nrm, red);
        if (!a.symmetric && a.orth == 1) {
            // CGS2: second pass on v~_{j+1}
            __syncthreads();
            for (int kk = warp; kk < nd; kk += nw) {
                const double *vc = wk.V + (int64_t)kk * wk.ldv;
                double d = 0.0;
                for (int r = lane; r < n; r += 32) d = fma(vc[r], vn[r], d);
                d = warp_sum(d);
                if (lane == 0) dres[kk] = d;
            }
            __syncthreads();
            for (int k = t; k < nd; k += SMALL_NT) {
                const double c = wk.sigma[k] * dres[k];
                wk.H[k + (size_t)j * wk.ldh] += c;
                gs[k] = c * wk.sigma[k];
            }
            __syncthreads();
            nrm = 0.0;
            for (int r = t; r < n; r += SMALL_NT) {
                double v = vn[r];
                for (int k = 0; k < nd; k++) v = fma(-gs[k], wk.V[r + (int64_t)k * wk.ldv], v);
                vn[r] = v;
                nrm = fma(v, v, nrm);
            }
            tot = block_sum(nrm, red);
        }
        if (t == 0) {
            const double h = sqrt(tot);
            wk.H[(j + 1) + (size_t)j * wk.ldh] = h;
            if (a.symmetric) {
                if (j + 1 < wk.hcols) wk.H[j + (size_t)(j + 1) * wk.ldh] = h;
                wk.st->lz = h * wk.sigma[j];
            }
            wk.sigma[j + 1] = 1.0 / h;
            if (!isfinite(h)) { wk.st->nonfinite = 1; wk.st->brk = j + 1; s_brk = j + 1; }
            else if (h <= a.bthr) { wk.st->brk = j + 1; s_brk = j + 1; }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------------
// One-CTA versions of the two generic streaming kernels for n <= SMALL_N (w-recurrence, seed,
// combine, kernel-level entry points): no grid reduction, no halo copies.  Per row the arithmetic
// is that of spmv_stream / axpy_stream (same operand order, same FMA chains; stencil rows bit-exact
// with a sequential CSR sum); block sums replace the grid reduction and feed the same finalize().

constexpr int SMALL_NR = SMALL_N / SMALL_NT;          // rows per thread (r = t + i SMALL_NT)
constexpr int SMALL_NW = SMALL_NT / 32;

// d_k = sum_r V[r, c0 + k] x_r for k < nd into dres (fixed order: rows per thread, warp shuffle
// tree, warps in order); each thread issues the loads of 8 columns at once
__device__ __forceinline__ void small_dots(const double *V, int64_t ldv, int c0, int nd, int n,
                                           const double (&x)[SMALL_NR], double *wpart, double *dres)
{
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    for (int k0 = 0; k0 < nd; k0 += 8) {
        double d[8];
#pragma unroll
        for (int u = 0; u < 8; u++) d[u] = 0.0;
#pragma unroll
        for (int i = 0; i < SMALL_NR; i++) {
            const int r = t + i * SMALL_NT;
            if (r < n) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; u++) v[u] = (k0 + u < nd) ? V[r + (int64_t)(c0 + k0 + u) * ldv] : 0.0;
#pragma unroll
                for (int u = 0; u < 8; u++) d[u] = fma(v[u], x[i], d[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const double w = warp_sum(d[u]);
            if (lane == 0 && k0 + u < nd) wpart[(k0 + u) * SMALL_NW + warp] = w;
        }
    }
    __syncthreads();
    for (int k = t; k < nd; k += SMALL_NT) {
        double s = 0.0;
        for (int w = 0; w < SMALL_NW; w++) s += wpart[k * SMALL_NW + w];
        dres[k] = s;
    }
    __syncthreads();
}

template <class Op>
__global__ void __launch_bounds__(SMALL_NT) spmv_small_kernel(Op op, SpmvArgs a, Work wk)
{
    __shared__ double wpart[(MAXD + 2) * SMALL_NW];
    __shared__ double red[MAXD + 2];
    __shared__ double wsum[SMALL_NW];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int n = (int)op.n;
    pdl_wait();
    if (a.check_brk && wk.st->brk >= 0) return;            // uniform
    const double sc = a.xscale ? *a.xscale : 1.0;
    double y[SMALL_NR];
    double ysq = 0.0;
#pragma unroll
    for (int i = 0; i < SMALL_NR; i++) {
        const int r = t + i * SMALL_NT;
        double v = 0.0;
        if (r < n) {
            v = row_apply(op, a.x, r) * sc;
            for (int l = 0; l < a.nz; l++) v = fma(a.zc[l] * (a.zcd[l] ? *a.zcd[l] : 1.0), a.z[l][r], v);
            if (a.y) a.y[r] = v;
            ysq = fma(v, v, ysq);
        }
        y[i] = v;
    }
    if (a.nd > 0) small_dots(a.V, a.ldv, a.d0, a.nd, n, y, wpart, red);
    if (a.ynorm) {
        const double v = warp_sum(ysq);
        if (lane == 0) wsum[warp] = v;
        __syncthreads();
        if (t == 0) {
            double s = 0.0;
            for (int w = 0; w < SMALL_NW; w++) s += wsum[w];
            red[a.nd] = s;
        }
    }
    __syncthreads();
    if (a.nd + (a.ynorm ? 1 : 0) == 0) return;
    finalize(a.fin, a.j, a.nd, red, wk, a.bthr, 0);
}

__global__ void __launch_bounds__(SMALL_NT) axpy_small_kernel(int64_t n64, AxpyArgs a, Work wk)
{
    __shared__ double coef[MAXD + MAXZ + 2];
    __shared__ const double *src[MAXD + MAXZ + 2];
    __shared__ double red[2];
    __shared__ double wsum[SMALL_NW];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int n = (int)n64;
    pdl_wait();
    if (a.check_brk && wk.st->brk >= 0) return;            // uniform
    const int nbase = (a.a0h != 0.0) ? 1 : 0;
    const int nitem = nbase + a.nc + a.ne;
    for (int k = t; k < nitem; k += SMALL_NT) {            // same item order as axpy_stream
        double c;
        const double *p;
        if (k < nbase) {
            c = a.a0h * (a.a0d ? *a.a0d : 1.0);
            p = a.base;
        } else if (k < nbase + a.nc) {
            const int kc = a.rev ? (a.nc - 1 - (k - nbase)) : (k - nbase);
            c = a.gsign * a.g[kc];
            p = a.V + (int64_t)(a.c0 + kc) * a.ldv;
        } else {
            const int i = k - nbase - a.nc;
            c = a.ec[i] * (a.ecd ? a.ecd[i] : 1.0);
            p = a.e[i];
        }
        coef[k] = c;
        src[k] = p;
    }
    __syncthreads();
    double nrm = 0.0;
#pragma unroll
    for (int i = 0; i < SMALL_NR; i++) {
        const int r = t + i * SMALL_NT;
        if (r >= n) continue;
        // eight independent loads in flight before their FMAs (a one-at-a-time chain of L2 round
        // trips cost ~10 us at mu = 35); same item order, so the sums are unchanged
        double acc = 0.0;
        int k = 0;
        for (; k + 8 <= nitem; k += 8) {
            double x[8];
#pragma unroll
            for (int u = 0; u < 8; u++) x[u] = src[k + u][r];
#pragma unroll
            for (int u = 0; u < 8; u++) acc = fma(coef[k + u], x[u], acc);
        }
        for (; k < nitem; k++) acc = fma(coef[k], src[k][r], acc);
        a.out[r] = acc;
        nrm = fma(acc, acc, nrm);
    }
    if (!a.onorm) return;
    const double v = warp_sum(nrm);
    if (lane == 0) wsum[warp] = v;
    __syncthreads();
    if (t == 0) {
        double s = 0.0;
        for (int w = 0; w < SMALL_NW; w++) s += wsum[w];
        red[0] = s;
    }
    __syncthreads();
    finalize(a.fin, a.j, 1, red, wk, a.bthr, a.lanczos);
}

} // namespace phipm
