// kernels.cuh — device code of libphipm (sm_100a, fp64).
//
// The n-sized work of one phipm step (Sec. 3.1-3.3) is done by two streaming kernels:
//
//   spmv_fused   y = s * (A x) + sum_i c_i z_i          (Eq. wrecurrence P:536-540 epilogue;
//                 [+ d_k = V_k^T y for a column range]   Alg. 1 line "h_ij = v_i^T w" / Alg. 2
//                 [+ ||y||^2]                            "t_jj = v_j^T w", fused in the same pass)
//   axpy_fused   out = a0 * base + sign * sum_k g_k V_k + sum_i e_i E_i   (Gram-Schmidt update,
//                 [+ ||out||^2]                            Eq. step P:518-522 assembly)
//
// Each ends in a deterministic grid reduction (per-block partials, last block sums them in a
// fixed order) whose last block runs a tiny "finalize" that turns the sums into H entries,
// normalisation factors and next-kernel coefficients, so the Krylov loop never returns to the
// host.  Krylov vectors are stored UNNORMALISED (v~_k) with sigma_k = 1/||v~_k||; sigma is folded
// into the next kernel's coefficients, which saves a normalisation pass per step.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace phipm {

constexpr int NT = 256;               // threads per block of the streaming kernels
constexpr int NWARP = NT / 32;
constexpr int RPT = 4;                // rows per thread per tile
constexpr int TILE = NT * RPT;        // rows per tile
constexpr int MAXZ = 6;               // epilogue vectors (p_max <= 5)
constexpr int MAXD = 128;             // dot / axpy columns per launch (m_max + 1 <= MAXD)

enum Fin : int {
    FIN_NONE = 0,
    FIN_ARNOLDI = 1,       // spmv dots d_k, k=0..j  -> H(k,j) = sigma_k d_k ; g_k = H(k,j) sigma_k
    FIN_LANCZOS = 2,       // spmv dot d = v~_j^T y  -> alpha_j = sigma_j d ; g_0 = alpha_j sigma_j
    FIN_SEED = 3,          // ||w_p||^2 -> beta, sigma_0 = 1/beta, brk reset
    FIN_NORM = 4,          // ||v~_{j+1}||^2 -> h_{j+1,j}, sigma_{j+1}, breakdown, Lanczos coupling
    FIN_REORTH = 5,        // CGS2 second pass dots: c_k = sigma_k d_k ; H(k,j) += c_k ; g_k = c_k sigma_k
    FIN_RAW = 6,           // copy the sums to out_raw (kernel-level parity entry points)
};

// device-resident scalars of the current time step
struct DevState {
    double beta;       // ||w_p||_2 (Krylov seed norm)
    double wnorm2;     // ||y||^2 of the latest fused SpMV
    double lz;         // Lanczos: h_{j+1,j} sigma_j, the coefficient of v~_j in step j+1
    int brk;           // -1: no breakdown; otherwise the number of valid H columns
    int nonfinite;     // a non-finite norm was met
};

// pointers into the context workspace, shared by all kernels of a solve
struct Work {
    double *V;             // basis, column k = v~_k (unnormalised), leading dimension ldv
    int64_t ldv;
    double *H;             // (m_max+1) x m_max, column-major, leading dimension ldh
    int ldh, hcols;
    double *sigma;         // sigma_k = 1 / ||v~_k||
    double *g;             // coefficients for the next axpy_fused (length MAXD)
    double *part;          // grid-reduction partials, [value][block], stride pstride
    int pstride;
    unsigned *counter;     // last-block ticket (reset by the last block)
    DevState *st;
    double *out_raw;       // FIN_RAW destination
};

struct StencilOp {
    int dim, nx, ny, nz;
    int64_t n;
    double c[7];           // center, xm, xp, ym, yp, zm, zp
};

struct CsrOp {
    int64_t n;
    const int32_t *__restrict__ rp;
    const int32_t *__restrict__ col;
    const double *__restrict__ val;
    int glog;              // log2(lanes per row)
};

struct SpmvArgs {
    const double *x;
    const double *xscale;        // device scalar s (sigma_j) or null -> 1
    double *y;
    int nz;
    const double *z[MAXZ];
    double zc[MAXZ];             // host factor of c_i
    const double *zcd[MAXZ];     // device factor of c_i or null
    const double *V;             // dot columns V[:, d0 .. d0+nd-1] (nd = 0: none)
    int64_t ldv;
    int d0, nd;
    int ynorm;                   // also reduce ||y||^2
    int fin, j;
    int check_brk;               // exit early if a breakdown happened earlier in this step
};

struct AxpyArgs {
    double *out;                 // may alias base
    const double *base;
    double a0h;                  // a0 = a0h * (a0d ? *a0d : 1); base unused if a0h == 0
    const double *a0d;
    const double *V;             // columns V[:, c0 .. c0+nc-1] with coefficients gsign * g[k]
    int64_t ldv;
    int c0, nc;
    const double *g;             // device coefficients
    double gsign;
    int ne;                      // extra vectors E_i with coefficient ec[i] * (ecd ? ecd[i] : 1)
    const double *e[MAXZ];
    double ec[MAXZ];
    const double *ecd;
    int onorm;                   // reduce ||out||^2
    int fin, j;
    int check_brk;
    double bthr;                 // breakdown threshold n eps ||A||_inf (FIN_NORM)
    int lanczos;                 // FIN_NORM: also store the symmetric entry and the coupling
};

// ------------------------------------------------------------------------------------------
// helpers

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double ldg_stream(const double *p)
{
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}

__device__ __forceinline__ double2 ldg_stream2(const double *p)
{
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}

// Publish nv block totals and take a ticket; true in the block that arrives last.
__device__ __forceinline__ bool publish_partials(const Work &wk, const double *bsum, int nv)
{
    __shared__ unsigned s_ticket;
    for (int v = threadIdx.x; v < nv; v += blockDim.x) wk.part[(size_t)v * wk.pstride + blockIdx.x] = bsum[v];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_ticket = atomicAdd(wk.counter, 1u);
    __syncthreads();
    return s_ticket == gridDim.x - 1;
}

// Last block: out[v] = sum over blocks in a fixed order (deterministic), then reset the ticket.
__device__ __forceinline__ void final_reduce(const Work &wk, int nv, double *out)
{
    __threadfence();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int v = warp; v < nv; v += nw) {
        const double *pv = wk.part + (size_t)v * wk.pstride;
        double s = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) s += __ldcg(pv + b);
        s = warp_sum(s);
        if (lane == 0) out[v] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) *wk.counter = 0u;
}

// Turn the reduced sums into step state (runs in the last block only).
__device__ void finalize(int fin, int j, int nd, const double *red, const Work &wk, double bthr, int lanczos)
{
    const int t = threadIdx.x;
    switch (fin) {
    case FIN_ARNOLDI:
        for (int k = t; k < nd; k += blockDim.x) {
            double h = wk.sigma[k] * red[k];
            wk.H[k + (size_t)j * wk.ldh] = h;
            wk.g[k] = h * wk.sigma[k];
        }
        if (t == 0) wk.st->wnorm2 = red[nd];
        break;
    case FIN_LANCZOS:
        if (t == 0) {
            double a = wk.sigma[j] * red[0];
            wk.H[j + (size_t)j * wk.ldh] = a;
            wk.g[0] = a * wk.sigma[j];
            wk.st->wnorm2 = red[1];
        }
        break;
    case FIN_SEED:
        if (t == 0) {
            double b = sqrt(red[0]);
            wk.st->beta = b;
            wk.sigma[0] = 1.0 / b;
            wk.st->brk = (b > 0.0 && isfinite(b)) ? -1 : 0;
            wk.st->nonfinite = isfinite(b) ? 0 : 1;
            wk.st->lz = 0.0;
        }
        break;
    case FIN_NORM:
        if (t == 0) {
            double h = sqrt(red[0]);
            wk.H[(j + 1) + (size_t)j * wk.ldh] = h;
            if (lanczos) {
                if (j + 1 < wk.hcols) wk.H[j + (size_t)(j + 1) * wk.ldh] = h;
                wk.st->lz = h * wk.sigma[j];
            }
            wk.sigma[j + 1] = 1.0 / h;
            if (!isfinite(h)) { wk.st->nonfinite = 1; wk.st->brk = j + 1; }
            else if (h <= bthr) wk.st->brk = j + 1;
        }
        break;
    case FIN_REORTH:
        for (int k = t; k < nd; k += blockDim.x) {
            double c = wk.sigma[k] * red[k];
            wk.H[k + (size_t)j * wk.ldh] += c;
            wk.g[k] = c * wk.sigma[k];
        }
        break;
    case FIN_RAW:
        for (int k = t; k < nd; k += blockDim.x) wk.out_raw[k] = red[k];
        break;
    default:
        break;
    }
}

// ------------------------------------------------------------------------------------------
// operator rows (phase 1): raw (A x)_r for the rows of a tile, into ys[]

// Stencil row, summed in ascending column order with separately rounded products (no FMA), the
// same order and rounding as a CSR row of orc-style sequential SpMV: bit-exact y.
__device__ __forceinline__ double stencil_row(const StencilOp &S, const double *__restrict__ x, int64_t r)
{
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
    double s = 0.0;
    if (S.dim >= 3 && kk > 0) s = __dadd_rn(s, __dmul_rn(S.c[5], __ldg(x + r - pl)));
    if (S.dim >= 2 && jj > 0) s = __dadd_rn(s, __dmul_rn(S.c[3], __ldg(x + r - S.nx)));
    if (i > 0) s = __dadd_rn(s, __dmul_rn(S.c[1], __ldg(x + r - 1)));
    s = __dadd_rn(s, __dmul_rn(S.c[0], __ldg(x + r)));
    if (i < S.nx - 1) s = __dadd_rn(s, __dmul_rn(S.c[2], __ldg(x + r + 1)));
    if (S.dim >= 2 && jj < S.ny - 1) s = __dadd_rn(s, __dmul_rn(S.c[4], __ldg(x + r + S.nx)));
    if (S.dim >= 3 && kk < S.nz - 1) s = __dadd_rn(s, __dmul_rn(S.c[6], __ldg(x + r + pl)));
    return s;
}

__device__ __forceinline__ void op_tile(const StencilOp &S, const double *__restrict__ x, int64_t r0, int rows,
                                        double *ys)
{
    for (int q = threadIdx.x; q < rows; q += NT) ys[q] = stencil_row(S, x, r0 + q);
}

// CSR: G = 2^glog lanes per row, strided over the row's entries, tree-reduced with shuffles.
__device__ __forceinline__ void op_tile(const CsrOp &A, const double *__restrict__ x, int64_t r0, int rows,
                                        double *ys)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int G = 1 << A.glog;
    const int rpw = 32 >> A.glog;                      // rows per warp iteration
    const int sub = lane >> A.glog, li = lane & (G - 1);
    for (int base = warp * rpw; base < rows; base += NWARP * rpw) {
        const int q = base + sub;
        double acc = 0.0;
        if (q < rows) {
            const int64_t r = r0 + q;
            const int e1 = __ldg(A.rp + r + 1);
            for (int e = __ldg(A.rp + r) + li; e < e1; e += G)
                acc = fma(ldg_stream(A.val + e), __ldg(x + __ldg(A.col + e)), acc);
        }
        for (int o = G >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (q < rows && li == 0) ys[q] = acc;
    }
}

// identity "operator" (multi-dot of a stored vector against V columns; CGS2 second pass)
struct IdentOp {
    int64_t n;
};

__device__ __forceinline__ void op_tile(const IdentOp &, const double *__restrict__ x, int64_t r0, int rows, double *ys)
{
    for (int q = threadIdx.x; q < rows; q += NT) ys[q] = ldg_stream(x + r0 + q);
}

template <class Op>
__device__ __forceinline__ int64_t op_n(const Op &op) { return op.n; }

// ------------------------------------------------------------------------------------------
// spmv_fused

template <class Op>
__global__ void __launch_bounds__(NT) spmv_fused_kernel(Op op, SpmvArgs a, Work wk)
{
    extern __shared__ double smem[];
    double *ys = smem;                     // TILE
    double *lacc = smem + TILE;            // nd x 32 per-lane dot partials
    __shared__ double bsum[MAXD + 2];
    __shared__ double wsum[NWARP];
    __shared__ int s_exit;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (a.check_brk) {
        if (tid == 0) s_exit = wk.st->brk >= 0;
        __syncthreads();
        if (s_exit) return;
    }
    const int64_t n = op_n(op);
    const double s = a.xscale ? *a.xscale : 1.0;
    double zc[MAXZ];
#pragma unroll
    for (int i = 0; i < MAXZ; i++) zc[i] = (i < a.nz) ? a.zc[i] * (a.zcd[i] ? *a.zcd[i] : 1.0) : 0.0;
    for (int i = tid; i < a.nd * 32; i += NT) lacc[i] = 0.0;
    double ysq = 0.0;
    __syncthreads();

    for (int64_t r0 = (int64_t)blockIdx.x * TILE; r0 < n; r0 += (int64_t)gridDim.x * TILE) {
        const int rows = (int)min((int64_t)TILE, n - r0);
        op_tile(op, a.x, r0, rows, ys);
        __syncthreads();
        // phase 2: scale + epilogue, store y, ||y||^2
        for (int q = tid; q < rows; q += NT) {
            const int64_t r = r0 + q;
            double y = s * ys[q];
#pragma unroll
            for (int i = 0; i < MAXZ; i++)
                if (i < a.nz) y = fma(zc[i], __ldg(a.z[i] + r), y);
            ys[q] = y;
            if (a.y) a.y[r] = y;
            ysq = fma(y, y, ysq);
        }
        __syncthreads();
        // phase 3: dots with V columns, one warp per column, lane partials kept in smem
        if (a.nd > 0) {
            for (int kk = warp; kk < a.nd; kk += NWARP) {
                const double *__restrict__ vc = a.V + (int64_t)(a.d0 + kk) * a.ldv + r0;
                double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
                int q = lane;
                for (; q + 96 < rows; q += 128) {
                    const double v0 = ldg_stream(vc + q), v1 = ldg_stream(vc + q + 32);
                    const double v2 = ldg_stream(vc + q + 64), v3 = ldg_stream(vc + q + 96);
                    c0 = fma(v0, ys[q], c0);
                    c1 = fma(v1, ys[q + 32], c1);
                    c2 = fma(v2, ys[q + 64], c2);
                    c3 = fma(v3, ys[q + 96], c3);
                }
                for (; q < rows; q += 32) c0 = fma(ldg_stream(vc + q), ys[q], c0);
                lacc[kk * 32 + lane] += (c0 + c1) + (c2 + c3);
            }
        }
        __syncthreads();
    }
    // block totals
    const int nv = a.nd + (a.ynorm ? 1 : 0);
    if (nv == 0) return;
    for (int kk = warp; kk < a.nd; kk += NWARP) {
        double v = warp_sum(lacc[kk * 32 + lane]);
        if (lane == 0) bsum[kk] = v;
    }
    if (a.ynorm) {
        double v = warp_sum(ysq);
        if (lane == 0) wsum[warp] = v;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < NWARP; w++) t += wsum[w];
            bsum[a.nd] = t;
        }
    }
    __syncthreads();
    if (!publish_partials(wk, bsum, nv)) return;
    __shared__ double red[MAXD + 2];
    final_reduce(wk, nv, red);
    finalize(a.fin, a.j, a.nd, red, wk, 0.0, 0);
}

// ------------------------------------------------------------------------------------------
// axpy_fused: out = a0 base + gsign sum_k g_k V[:, c0+k] + sum_i ec_i E_i  [+ ||out||^2]

template <bool VEC2>
__global__ void __launch_bounds__(NT) axpy_fused_kernel(int64_t n, AxpyArgs a, Work wk)
{
    __shared__ double gs[MAXD];
    __shared__ double bsum[2];
    __shared__ double wsum[NWARP];
    __shared__ int s_exit;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (a.check_brk) {
        if (tid == 0) s_exit = wk.st->brk >= 0;
        __syncthreads();
        if (s_exit) return;
    }
    for (int k = tid; k < a.nc; k += NT) gs[k] = a.gsign * a.g[k];
    const double a0 = a.a0h * (a.a0d ? *a.a0d : 1.0);
    double ec[MAXZ];
#pragma unroll
    for (int i = 0; i < MAXZ; i++) ec[i] = (i < a.ne) ? a.ec[i] * (a.ecd ? a.ecd[i] : 1.0) : 0.0;
    __syncthreads();
    double nrm = 0.0;
    const double *__restrict__ V = a.V + (int64_t)a.c0 * a.ldv;
    if (VEC2) {
        const int64_t npair = n >> 1;
        for (int64_t pi = (int64_t)blockIdx.x * NT + tid; pi < npair; pi += (int64_t)gridDim.x * NT) {
            const int64_t r = pi * 2;
            double2 acc = make_double2(0.0, 0.0);
            if (a.a0h != 0.0) {
                const double2 b = *reinterpret_cast<const double2 *>(a.base + r);
                acc.x = a0 * b.x;
                acc.y = a0 * b.y;
            }
            int k = 0;
            for (; k + 8 <= a.nc; k += 8) {
                double2 v[8];
#pragma unroll
                for (int u = 0; u < 8; u++) v[u] = ldg_stream2(V + (int64_t)(k + u) * a.ldv + r);
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    acc.x = fma(gs[k + u], v[u].x, acc.x);
                    acc.y = fma(gs[k + u], v[u].y, acc.y);
                }
            }
            for (; k < a.nc; k++) {
                const double2 v = ldg_stream2(V + (int64_t)k * a.ldv + r);
                acc.x = fma(gs[k], v.x, acc.x);
                acc.y = fma(gs[k], v.y, acc.y);
            }
#pragma unroll
            for (int i = 0; i < MAXZ; i++)
                if (i < a.ne) {
                    const double2 e = ldg_stream2(a.e[i] + r);
                    acc.x = fma(ec[i], e.x, acc.x);
                    acc.y = fma(ec[i], e.y, acc.y);
                }
            *reinterpret_cast<double2 *>(a.out + r) = acc;
            nrm = fma(acc.x, acc.x, nrm);
            nrm = fma(acc.y, acc.y, nrm);
        }
        if ((n & 1) && blockIdx.x == 0 && tid == 0) {
            const int64_t r = n - 1;
            double acc = (a.a0h != 0.0) ? a0 * a.base[r] : 0.0;
            for (int k = 0; k < a.nc; k++) acc = fma(gs[k], V[(int64_t)k * a.ldv + r], acc);
            for (int i = 0; i < a.ne; i++) acc = fma(ec[i], a.e[i][r], acc);
            a.out[r] = acc;
            nrm = fma(acc, acc, nrm);
        }
    } else {
        for (int64_t r = (int64_t)blockIdx.x * NT + tid; r < n; r += (int64_t)gridDim.x * NT) {
            double acc = (a.a0h != 0.0) ? a0 * a.base[r] : 0.0;
            int k = 0;
            for (; k + 8 <= a.nc; k += 8) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; u++) v[u] = ldg_stream(V + (int64_t)(k + u) * a.ldv + r);
#pragma unroll
                for (int u = 0; u < 8; u++) acc = fma(gs[k + u], v[u], acc);
            }
            for (; k < a.nc; k++) acc = fma(gs[k], ldg_stream(V + (int64_t)k * a.ldv + r), acc);
#pragma unroll
            for (int i = 0; i < MAXZ; i++)
                if (i < a.ne) acc = fma(ec[i], __ldg(a.e[i] + r), acc);
            a.out[r] = acc;
            nrm = fma(acc, acc, nrm);
        }
    }
    if (!a.onorm) return;
    double v = warp_sum(nrm);
    if (lane == 0) wsum[warp] = v;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < NWARP; w++) t += wsum[w];
        bsum[0] = t;
    }
    __syncthreads();
    if (!publish_partials(wk, bsum, 1)) return;
    __shared__ double red[2];
    final_reduce(wk, 1, red);
    finalize(a.fin, a.j, 1, red, wk, a.bthr, a.lanczos);
}

// ------------------------------------------------------------------------------------------
// small utility kernels

// max_i |x_i| for up to MAXZ vectors at once (grid reduction by max: order-independent, exact)
struct MaxAbsArgs {
    int nv;
    const double *x[MAXZ];
};

__global__ void __launch_bounds__(NT) maxabs_kernel(int64_t n, MaxAbsArgs a, Work wk)
{
    __shared__ double wmax[MAXZ][NWARP];
    __shared__ double bsum[MAXZ];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int v = 0; v < a.nv; v++) {
        double m = 0.0;
        for (int64_t r = (int64_t)blockIdx.x * NT + tid; r < n; r += (int64_t)gridDim.x * NT) m = fmax(m, fabs(a.x[v][r]));
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) wmax[v][warp] = m;
    }
    __syncthreads();
    if (tid < a.nv) {
        double m = 0.0;
        for (int w = 0; w < NWARP; w++) m = fmax(m, wmax[tid][w]);
        bsum[tid] = m;
    }
    __syncthreads();
    if (!publish_partials(wk, bsum, a.nv)) return;
    __threadfence();
    for (int v = warp; v < a.nv; v += NWARP) {
        double m = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) m = fmax(m, __ldcg(wk.part + (size_t)v * wk.pstride + b));
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) wk.out_raw[v] = m;
    }
    __syncthreads();
    if (tid == 0) *wk.counter = 0u;
}

// ||A||_inf of a CSR matrix: rows summed sequentially in ascending column order (bit-exact with
// a sequential reference), max over rows (exact).
__global__ void __launch_bounds__(NT) csr_infnorm_kernel(CsrOp A, Work wk)
{
    __shared__ double wmax[NWARP];
    __shared__ double bsum[1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double m = 0.0;
    for (int64_t r = (int64_t)blockIdx.x * NT + tid; r < A.n; r += (int64_t)gridDim.x * NT) {
        double s = 0.0;
        for (int e = A.rp[r]; e < A.rp[r + 1]; e++) s = __dadd_rn(s, fabs(A.val[e]));
        m = fmax(m, s);
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) wmax[warp] = m;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < NWARP; w++) t = fmax(t, wmax[w]);
        bsum[0] = t;
    }
    __syncthreads();
    if (!publish_partials(wk, bsum, 1)) return;
    __threadfence();
    if (warp == 0) {
        double t = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) t = fmax(t, __ldcg(wk.part + b));
        for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
        if (lane == 0) wk.out_raw[0] = t;
    }
    __syncthreads();
    if (tid == 0) *wk.counter = 0u;
}

// CSR of a stencil: every row independently, with the closed-form row pointer
//   rp[r] = (2 dim + 1) r - (#neighbours missing in rows < r)
// (integer-exact; equal to a sequential build).
__global__ void __launch_bounds__(NT) csr_from_stencil_kernel(StencilOp S, int32_t *rp, int32_t *col, double *val)
{
    const int64_t n = S.n, nx = S.nx, pl = (int64_t)S.nx * S.ny;
    for (int64_t r = (int64_t)blockIdx.x * NT + threadIdx.x; r <= n; r += (int64_t)gridDim.x * NT) {
        // entries before row r
        int64_t miss = (r + nx - 1) / nx + r / nx;               // x- missing (i==0), x+ missing (i==nx-1)
        if (S.dim >= 2) {
            const int64_t k = r / pl, rem = r - k * pl;
            miss += k * nx + (rem < nx ? rem : nx);                 // y- missing (j==0)
            miss += k * nx + (rem > pl - nx ? rem - (pl - nx) : 0); // y+ missing (j==ny-1)
        }
        if (S.dim >= 3) {
            miss += (r < pl ? r : pl);                              // z- missing (k==0)
            miss += (r > n - pl ? r - (n - pl) : 0);                // z+ missing (k==nz-1)
        }
        const int64_t e0 = (2 * S.dim + 1) * r - miss;
        rp[r] = (int32_t)e0;
        if (r == n) break;
        const int64_t i = r % nx, jj = (r / nx) % S.ny, kk = r / pl;
        int64_t e = e0;
        if (S.dim >= 3 && kk > 0) { col[e] = (int32_t)(r - pl); val[e] = S.c[5]; e++; }
        if (S.dim >= 2 && jj > 0) { col[e] = (int32_t)(r - nx); val[e] = S.c[3]; e++; }
        if (i > 0) { col[e] = (int32_t)(r - 1); val[e] = S.c[1]; e++; }
        col[e] = (int32_t)r; val[e] = S.c[0]; e++;
        if (i < nx - 1) { col[e] = (int32_t)(r + 1); val[e] = S.c[2]; e++; }
        if (S.dim >= 2 && jj < S.ny - 1) { col[e] = (int32_t)(r + nx); val[e] = S.c[4]; e++; }
        if (S.dim >= 3 && kk < S.nz - 1) { col[e] = (int32_t)(r + pl); val[e] = S.c[6]; e++; }
    }
}

// out[:, k] = sigma_k V[:, k] for k < ncols (normalised basis for the kernel-level export)
__global__ void scale_columns_kernel(int64_t n, int ncols, const double *V, int64_t ldv, const double *sigma,
                                     double *out, int64_t ldo)
{
    for (int k = blockIdx.y; k < ncols; k += gridDim.y) {
        const double s = sigma[k];
        for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
            out[r + (int64_t)k * ldo] = s * V[r + (int64_t)k * ldv];
    }
}

} // namespace phipm
