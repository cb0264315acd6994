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

#include <type_traits>

namespace phipm {

constexpr int NT = 256;               // threads per block of the streaming kernels
constexpr int NWARP = NT / 32;
constexpr int RPT = 4;                // rows per thread per tile
constexpr int TILE = NT * RPT;        // rows per tile
constexpr int MAXZ = 6;               // epilogue vectors (<= p_max <= P_MAX_ABS = 6)
constexpr int MAXD = 128;             // dot / axpy columns per launch (m_max + 1 <= MAXD)

enum Fin : int {
    FIN_NONE = 0,
    FIN_ARNOLDI = 1,       // spmv dots d_k, k=0..j  -> H(k,j) = sigma_k d_k ; g_k = H(k,j) sigma_k
    FIN_LANCZOS = 2,       // spmv dot d = v~_j^T y  -> alpha_j = sigma_j d ; g_0 = alpha_j sigma_j
    FIN_SEED = 3,          // ||w_p||^2 -> beta, sigma_0 = 1/beta, brk reset
    FIN_NORM = 4,          // ||v~_{j+1}||^2 -> h_{j+1,j}, sigma_{j+1}, breakdown, Lanczos coupling
    FIN_REORTH = 5,        // CGS2 second pass dots: c_k = sigma_k d_k ; H(k,j) += c_k ; g_k = c_k sigma_k
    FIN_RAW = 6,           // copy the sums to out_raw (kernel-level parity entry points)
    FIN_ARNOLDI_LAG = 7,   // lagged normalisation: raw dots D_k = v~_k^T A v~_j (k=0..j), ||A v~_j||^2 and
                           // ||v~_j||^2 -> h_{j,j-1}, sigma_j, breakdown; H(k,j) = sigma_k sigma_j D_k
};

// device-resident scalars of the current time step
struct DevState {
    double beta;       // ||w_p||_2 (Krylov seed norm)
    double wnorm2;     // ||y||^2 of the latest fused SpMV
    double lz;         // Lanczos: h_{j+1,j} sigma_j, the coefficient of v~_j in step j+1
    int brk;           // -1: no breakdown; otherwise the number of valid H columns
    int nonfinite;     // a non-finite norm was met
    int aborted;       // the persistent Krylov kernel timed out waiting for a grid phase
    unsigned long long anorm_bits;   // ||A||_inf accumulated by the first SpMV of a CSR solve (bits of a
                                     // non-negative double; atomicMax), when the analysis pass skipped val
    double bthr_d;                   // n eps ||A||_inf from that SpMV (finalize uses it when bthr < 0)
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
    double *part2;         // partials an SpMV kernel leaves for the next update kernel (deferred finalize)
    int pstride;
    unsigned *counter;     // last-block ticket (reset by the last block)
    DevState *st;
    double *out_raw;       // FIN_RAW destination
};

struct StencilOp {
    int dim, nx, ny, nz;
    int64_t n;
    double c[11];          // center, xm, xp, ym, yp, zm, zp, xmym, xpym, xmyp, xpyp
    int diag;              // 2-D 9-point: the four corner neighbours (c[7..10]) exist
    int sdi, sdj;          // dim >= 2: 2 SNT rows = sdj grid lines + sdi points (host-computed)
};

struct CsrOp {
    int64_t n;
    const int32_t *__restrict__ rp;
    const int32_t *__restrict__ col;
    const double *__restrict__ val;
    int glog;              // log2(lanes per row)
    // x-window mode (tile rows' columns within a band): per-tile [tlo, thi] column range for tiles
    // of `wtile` rows; tiles whose range fits `wcap` doubles gather x from shared memory
    const int32_t *__restrict__ tlo;
    const int32_t *__restrict__ thi;
    int wtile, wcap;
    int ell;               // > 0: every row has exactly `ell` entries (row_ptr[r] = ell r), ell % 4 == 0,
                           // ell <= 128: vectorised fast path (4 entries per lane)
    int ring;              // ell > 0 and every column within [r - blo, r + bhi]: x from a shared ring
    int blo, bhi;          // band below / above the diagonal (even, >= 0)
    const int16_t *__restrict__ off16;   // optional (uniform rows, band <= 32767): col - row as int16,
                                         // written by the analysis pass; the x-ring SpMV streams these
                                         // 2 B per entry instead of the 4 B column indices
    int pf;                // x-ring path: L2 prefetch distance of val/col in rows (0 = off;
                           // PHIPM_OPT_CSR_PREFETCH)
    int64_t pf_end;        // (set per launch) rows >= pf_end are not prefetched (the CTA's range end)
};

struct SpmvArgs {
    const double *x;             // workspace vector padded to ldx (TMA halo reads) or, for CSR, any
    int64_t ldx;
    const double *xscale;        // device scalar s (sigma_j) or null -> 1
    double *y;
    int nz;
    const double *z[MAXZ];
    double zc[MAXZ];             // host factor of c_i
    const double *zcd[MAXZ];     // device factor of c_i or null
    const double *V;             // dot columns V[:, d0 .. d0+nd-1] (nd = 0: none)
    int64_t ldv;
    int d0, nd;
    int xcol;                    // dot column index (relative to d0) that equals x, or -1: its
                                 // values are taken from the x tile already on chip
    int ynorm;                   // also reduce ||y||^2
    int fin, j;
    int check_brk;               // exit early if a breakdown happened earlier in this step
    int64_t rpc;                 // rows per CTA (balanced contiguous ranges; multiple of 32)
    int pfc;                     // L2-prefetch the streamed columns / z vectors one group ahead (PHIPM_OPT_COL_PREFETCH)
    unsigned long long *dbg;     // optional per-CTA %globaltimer stamps (PHIPM_KCLOCKS tool), 8 per CTA
    int xnorm;                   // also reduce ||x||^2 (after ||y||^2), for FIN_ARNOLDI_LAG
    double bthr;                 // breakdown threshold (FIN_ARNOLDI_LAG)
    int anorm;                   // CSR x-ring path: also ||A||_inf (row |a| sums in entry order per lane,
                                 // lanes by a shuffle tree) -> st->anorm_bits, st->bthr_d, and *anorm_pub
    double *anorm_pub;           // mapped pinned memory: ||A||_inf, then
    volatile int *anorm_seq;     // ... this sequence number (after a system-scope fence)
    int anorm_seqv;
    int defer;                   // deferred finalize: write the nv partials to wk.part2 and end (no ticket);
                                 // the update kernel that follows reduces them (AxpyArgs.dfin)
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
    int64_t rpc;                 // rows per CTA (balanced contiguous ranges; multiple of 32)
    int rev;                     // stream the V columns in descending order (L2 ping-pong with the
                                 // ascending dot pass of the SpMV kernel)
    int pfc;                     // L2-prefetch the streamed vectors one group ahead (PHIPM_OPT_COL_PREFETCH)
    unsigned long long *dbg;     // optional per-CTA %globaltimer stamps (PHIPM_KCLOCKS tool)
    // deferred finalize of the preceding SpMV kernel (SpmvArgs.defer): its fin mode (FIN_ARNOLDI,
    // FIN_LANCZOS or FIN_ARNOLDI_LAG; 0 = none), grid size, dot count, value count, step and threshold
    int dfin, dnb, dnd, dnv, dj;
    double dbthr;
    // guarded launch (a combine enqueued before the host has seen the attempt's result): the kernel runs only
    // if guard[0] == guard_val (written by the exponential's epilogue) and takes nc from guard[1]
    const int *guard;
    int guard_val;
};

// ------------------------------------------------------------------------------------------
// helpers

// Programmatic Dependent Launch: wait for the predecessor grid (no-op without PDL), then let the
// successor grid start launching.  Called before any access to data written by earlier kernels.
__device__ __forceinline__ void pdl_wait()
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define KSTAMP(i) \
    if (a.dbg && threadIdx.x == 0) a.dbg[(size_t)blockIdx.x * 8 + (i)] = gtimer();

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

__device__ __forceinline__ int4 ldg_stream_i4(const int4 *p)
{
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
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
    __syncthreads();
    // one acq_rel gpu-scope ticket after the CTA barrier: release orders every thread's partial
    // (observed through the barrier) before the ticket; acquire, propagated by the next barrier,
    // makes the other CTAs' partials visible to the last CTA.  No per-thread fences.
    if (threadIdx.x == 0) {
        unsigned tk;
        asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(tk) : "l"(wk.counter) : "memory");
        s_ticket = tk;
    }
    __syncthreads();
    return s_ticket == gridDim.x - 1;
}

// Last block: out[v] = sum over blocks in a fixed order (deterministic), then reset the ticket.
// Each lane issues 8 independent L2 loads per batch (fixed lane/slot assignment, fixed combine
// order), so the tail costs about one L2 round trip per value instead of one per 32 blocks.
// reduce_partials: the same sums from any partials buffer of nb blocks (every thread of the calling CTA
// must call it; out[] is visible to all of them on return).
__device__ __forceinline__ void reduce_partials(const double *part, int pstride, int nb, int nv, double *out)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int v = warp; v < nv; v += nw) {
        const double *pv = part + (size_t)v * pstride;
        double acc[8];
#pragma unroll
        for (int u = 0; u < 8; u++) acc[u] = 0.0;
        for (int b0 = 0; b0 < nb; b0 += 256) {
            double x[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const int b = b0 + u * 32 + lane;
                x[u] = (b < nb) ? __ldcg(pv + b) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; u++) acc[u] += x[u];
        }
        double s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
        s = warp_sum(s);
        if (lane == 0) out[v] = s;
    }
    __syncthreads();
}

__device__ __forceinline__ void final_reduce(const Work &wk, int nv, double *out)
{
    reduce_partials(wk.part, wk.pstride, gridDim.x, nv, out);
    if (threadIdx.x == 0) *wk.counter = 0u;
}

// Turn the reduced sums into step state (runs in the last block only).
__device__ void finalize(int fin, int j, int nd, const double *red, const Work &wk, double bthr, int lanczos)
{
    const int t = threadIdx.x;
    if (bthr < 0.0) bthr = wk.st->bthr_d;     // threshold from the SpMV that computed ||A||_inf
    switch (fin) {
    case FIN_ARNOLDI:
        for (int k = t; k < nd; k += blockDim.x) {
            double h = wk.sigma[k] * red[k];
            wk.H[k + (size_t)j * wk.ldh] = h;
            wk.g[k] = h * wk.sigma[k];
        }
        if (t == 0) wk.st->wnorm2 = red[nd];
        break;
    case FIN_ARNOLDI_LAG: {
        // red[0..nd-1] raw dots, red[nd] ||A x||^2, red[nd+1] ||x||^2 with x = v~_j (j >= 1)
        __shared__ double s_sj;
        __shared__ int s_ok;
        if (t == 0) {
            const double hh = sqrt(red[nd + 1]);
            const double sj = 1.0 / hh;
            wk.H[j + (size_t)(j - 1) * wk.ldh] = hh;
            wk.sigma[j] = sj;
            int ok = 1;
            if (!isfinite(hh)) { wk.st->nonfinite = 1; wk.st->brk = j; ok = 0; }
            else if (hh <= bthr) { wk.st->brk = j; ok = 0; }
            if (ok) wk.st->wnorm2 = red[nd] * sj * sj;
            s_sj = sj;
            s_ok = ok;
        }
        __syncthreads();
        if (s_ok) {
            const double sj = s_sj;
            for (int k = t; k < nd; k += blockDim.x) {
                const double sk = (k == j) ? sj : wk.sigma[k];
                const double h = sk * (sj * red[k]);
                wk.H[k + (size_t)j * wk.ldh] = h;
                wk.g[k] = h * sk;
            }
        }
        break;
    }
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

// Deferred finalize (AxpyArgs.dfin, PHIPM_OPT_DEFER), run by EVERY CTA of the update kernel that follows an
// SpMV launched with SpmvArgs.defer.  The SpMV's partials are summed by reduce_partials in final_reduce's
// order, and the step state is derived with finalize()'s expressions, so every CTA holds bit for bit what the
// SpMV's last CTA would have computed; CTA 0 writes it (H(:, j), sigma_j, wnorm2, g, brk) for the later
// kernels and the exponential.  This removes the SpMV's ticket, last-block reduction and finalize from the
// critical path: the update kernel's CTAs do the same reduction concurrently.
// g_out[k] (k < dnd): the update coefficients g_k; *a0s: the factor of the base vector (sigma_j for
// FIN_ARNOLDI_LAG, where the SpMV produced the raw A v~_j; else 1).  Returns false on breakdown.
__device__ bool deferred_finalize(const AxpyArgs &a, const Work &wk, double *red, double *g_out, double *a0s)
{
    __shared__ int s_ok;
    __shared__ double s_sj;
    reduce_partials(wk.part2, wk.pstride, a.dnb, a.dnv, red);
    const int t = threadIdx.x, j = a.dj, nd = a.dnd;
    const bool lead = blockIdx.x == 0;
    switch (a.dfin) {
    case FIN_ARNOLDI:
        for (int k = t; k < nd; k += blockDim.x) {
            const double sk = wk.sigma[k];
            const double h = sk * red[k];
            const double gk = h * sk;
            g_out[k] = gk;
            if (lead) {
                wk.H[k + (size_t)j * wk.ldh] = h;
                wk.g[k] = gk;
            }
        }
        if (t == 0) {
            if (lead) wk.st->wnorm2 = red[nd];
            *a0s = 1.0;
            s_ok = 1;
        }
        break;
    case FIN_LANCZOS:
        if (t == 0) {
            const double sj = wk.sigma[j];
            const double al = sj * red[0];
            const double g0 = al * sj;
            g_out[0] = g0;
            if (lead) {
                wk.H[j + (size_t)j * wk.ldh] = al;
                wk.g[0] = g0;
                wk.st->wnorm2 = red[1];
            }
            *a0s = 1.0;
            s_ok = 1;
        }
        break;
    case FIN_ARNOLDI_LAG: {
        // red[0..nd-1] raw dots, red[nd] ||A x||^2, red[nd+1] ||x||^2 with x = v~_j (j >= 1)
        if (t == 0) {
            double bthr = a.dbthr;
            if (bthr < 0.0) bthr = wk.st->bthr_d;
            const double hh = sqrt(red[nd + 1]);
            const double sj = 1.0 / hh;
            int ok = 1, nonfin = 0;
            if (!isfinite(hh)) { nonfin = 1; ok = 0; }
            else if (hh <= bthr) ok = 0;
            if (lead) {
                wk.H[j + (size_t)(j - 1) * wk.ldh] = hh;
                wk.sigma[j] = sj;
                if (nonfin) wk.st->nonfinite = 1;
                if (!ok) wk.st->brk = j;
                else wk.st->wnorm2 = red[nd] * sj * sj;
            }
            s_sj = sj;
            s_ok = ok;
            *a0s = sj;
        }
        __syncthreads();
        if (s_ok) {
            const double sj = s_sj;
            for (int k = t; k < nd; k += blockDim.x) {
                const double sk = (k == j) ? sj : wk.sigma[k];
                const double h = sk * (sj * red[k]);
                const double gk = h * sk;
                g_out[k] = gk;
                if (lead) {
                    wk.H[k + (size_t)j * wk.ldh] = h;
                    wk.g[k] = gk;
                }
            }
        }
        break;
    }
    default:
        if (t == 0) {
            *a0s = 1.0;
            s_ok = 1;
        }
        break;
    }
    __syncthreads();
    return s_ok != 0;
}

// ------------------------------------------------------------------------------------------
// operators

// identity "operator" (multi-dot of a stored vector against V columns; CGS2 second pass)
struct IdentOp {
    int64_t n;
};

// ------------------------------------------------------------------------------------------
// small utility kernels

// max_i |x_i| for up to MAXZ vectors at once (grid reduction by max: order-independent, exact)
struct MaxAbsArgs {
    int nv;
    const double *x[MAXZ];
    double *pub;                 // optional: results to mapped pinned memory, then ...
    volatile int *pub_seq;       // ... this sequence number (after a system-scope fence)
    int seq;
};

// max that propagates NaN (fmax drops it): once m is NaN it stays NaN, so a NaN input gives a NaN
// ||.||_inf and the solve reports PHIPM_ENONFINITE instead of taking the all-zero shortcut
__device__ __forceinline__ double nanmax(double m, double x) { return (x > m || x != x) ? x : m; }

__global__ void __launch_bounds__(NT) maxabs_kernel(int64_t n, MaxAbsArgs a, Work wk)
{
    __shared__ double wmax[MAXZ][NWARP];
    __shared__ double bsum[MAXZ];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t stride = (int64_t)gridDim.x * NT;
    for (int v = 0; v < a.nv; v++) {
        // eight independent loads in flight per thread (a one-load grid-stride loop ran at ~1 TB/s);
        // max is exact, so the order does not matter
        const double *x = a.x[v];
        double m = 0.0;
        int64_t r = (int64_t)blockIdx.x * NT + tid;
        // (predicated: at full occupancy a thread has fewer than 8 elements of a 2M-row vector, and a
        // scalar tail loop issued them one dependent round trip at a time)
        for (; r < n; r += 8 * stride) {
            double t[8];
#pragma unroll
            for (int u = 0; u < 8; u++) t[u] = (r + u * stride < n) ? __ldg(x + r + u * stride) : 0.0;
#pragma unroll
            for (int u = 0; u < 8; u++) m = nanmax(m, fabs(t[u]));
        }
        for (int o = 16; o > 0; o >>= 1) m = nanmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) wmax[v][warp] = m;
    }
    __syncthreads();
    if (tid < a.nv) {
        double m = 0.0;
        for (int w = 0; w < NWARP; w++) m = nanmax(m, wmax[tid][w]);
        bsum[tid] = m;
    }
    __syncthreads();
    if (!publish_partials(wk, bsum, a.nv)) return;
    // publish_partials acquired the other CTAs' partials
    for (int v = warp; v < a.nv; v += NWARP) {
        double m = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) m = nanmax(m, __ldcg(wk.part + (size_t)v * wk.pstride + b));
        for (int o = 16; o > 0; o >>= 1) m = nanmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) {
            if (a.pub) a.pub[v] = m;
            else wk.out_raw[v] = m;
        }
    }
    __syncthreads();
    if (tid == 0) {
        *wk.counter = 0u;
        if (a.pub) {
            // the host spins on the sequence number: publish it last
            __threadfence_system();
            *a.pub_seq = a.seq;
        }
    }
}

// One pass over a CSR matrix (row_ptr, col, val), coalesced: each warp takes 32 consecutive rows,
// copies their entries into shared memory (skewed: entry i at i + i/32, so that lanes walking rows
// of equal length hit different banks) and each lane then walks its own row in order:
//   ||A||_inf = max_r sum_e |a_re|   (summed sequentially in entry order: bit-exact with a
//                                     sequential reference; the max is exact)
//   uniform   = row_ptr[r] == L r for all r  (L = nnz / n, or -1)
//   band      = max(r - col), max(col - r)
// Rows of a group with more than CSRA_CAP entries are walked in global memory instead.
constexpr int CSRA_CAP = 512;                  // staged entries per warp (32 rows of 16)
constexpr int CSRA_NT = 128, CSRA_NW = CSRA_NT / 32;
struct CsrAnalysis {
    unsigned long long norm_bits;              // ||A||_inf (bits of a non-negative double)
    int nonuniform, blo, bhi, pad;
};

__device__ __forceinline__ int clamp_band(int64_t d) { return d < 0 ? 0 : (d > 0x3fffffff ? 0x3fffffff : (int)d); }

// mode bit 0: ||A||_inf (reads val); bit 1: uniform rows and band (reads col); bit 2 (with bit 1 and
// L > 0): also write off16[e] = col[e] - row (clamped to int16; used only if the band fits).
// row_ptr always.
__global__ void __launch_bounds__(CSRA_NT) csr_analyze_kernel(CsrOp A, int L, CsrAnalysis *out, int mode = 3,
                                                              int16_t *off16 = nullptr)
{
    const bool dn = mode & 1, ds = (mode & 2) != 0, wo = (mode & 4) && off16 && L > 0;
    constexpr int SK = CSRA_CAP + CSRA_CAP / 32;
    __shared__ double sv[CSRA_NW][SK];
    __shared__ int sc[CSRA_NW][SK];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n = A.n, ngroups = (n + 31) / 32;
    double nrm = 0.0;
    int bad = 0, blo = 0, bhi = 0;
    for (int64_t g = (int64_t)blockIdx.x * CSRA_NW + warp; g < ngroups; g += (int64_t)gridDim.x * CSRA_NW) {
        const int64_t r = g * 32 + lane;
        const bool ok = r < n;
        const int eb = ok ? A.rp[r] : 0, ee = ok ? A.rp[r + 1] : 0;
        if (ok && L > 0 && ((int64_t)eb != (int64_t)L * r || (int64_t)ee != (int64_t)L * (r + 1))) bad = 1;
        const int64_t rem = n - 1 - g * 32;
        const int last = rem < 31 ? (int)rem : 31;
        const int g0 = __shfl_sync(0xffffffffu, eb, 0), g1 = __shfl_sync(0xffffffffu, ee, last);
        double s = 0.0;
        int lo = 0, hi = 0;
        if (g1 - g0 <= CSRA_CAP) {
            for (int i = lane; i < g1 - g0; i += 32) {
                const int k = i + (i >> 5);
                if (dn) sv[warp][k] = A.val[g0 + i];
                if (ds) {
                    const int cv = A.col[g0 + i];
                    sc[warp][k] = cv;
                    if (wo) {
                        const int64_t e = (int64_t)g0 + i;
                        const int64_t d = (int64_t)cv - e / L;          // uniform rows: row = e / L
                        off16[e] = (int16_t)(d < -32768 ? -32768 : (d > 32767 ? 32767 : d));
                    }
                }
            }
            __syncwarp();
            for (int e = eb - g0; e < ee - g0; e++) {
                const int k = e + (e >> 5);
                if (dn) s = __dadd_rn(s, fabs(sv[warp][k]));
                if (ds) {
                    const int64_t d = (int64_t)sc[warp][k] - r;
                    lo = max(lo, clamp_band(-d));
                    hi = max(hi, clamp_band(d));
                }
            }
            __syncwarp();
        } else {
            for (int e = eb; e < ee; e++) {
                if (dn) s = __dadd_rn(s, fabs(A.val[e]));
                if (ds) {
                    const int64_t d = (int64_t)A.col[e] - r;
                    lo = max(lo, clamp_band(-d));
                    hi = max(hi, clamp_band(d));
                }
            }
        }
        nrm = fmax(nrm, s);
        blo = max(blo, lo);
        bhi = max(bhi, hi);
    }
    for (int o = 16; o > 0; o >>= 1) {
        nrm = fmax(nrm, __shfl_xor_sync(0xffffffffu, nrm, o));
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
        blo = max(blo, __shfl_xor_sync(0xffffffffu, blo, o));
        bhi = max(bhi, __shfl_xor_sync(0xffffffffu, bhi, o));
    }
    if (lane == 0) {
        atomicMax(&out->norm_bits, (unsigned long long)__double_as_longlong(nrm));
        if (bad) atomicOr(&out->nonuniform, 1);
        atomicMax(&out->blo, blo);
        atomicMax(&out->bhi, bhi);
    }
}

// The uniform-row case of csr_analyze_kernel's mode 2 (band and uniformity only; the fused-||A|| CSR path),
// as a plain stream: rows of L = 2^lgL entries (L >= 4), so an aligned 16-B group of 4 column indices lies
// in one row, row = e >> lgL, and the pass is two coalesced int4 streams (row_ptr, col) with four loads in
// flight per thread.  Same results as csr_analyze_kernel (max of clamp_band(+-(col - row)) over the entries
// and the row_ptr check) whenever the rows are uniform; when they are not (nonuniform set), the band is
// that of entry e's nominal row e / L and the host reruns csr_analyze_kernel.
__global__ void __launch_bounds__(256) csr_analyze_ell_kernel(int64_t n, const int32_t *__restrict__ rp,
                                                              const int32_t *__restrict__ col, int lgL,
                                                              CsrAnalysis *out)
{
    const int64_t L = (int64_t)1 << lgL;
    const int64_t nnz = n << lgL;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    int bad = 0, blo = 0, bhi = 0;
    // row_ptr: rp[r] == L r for r = 0 .. n
    for (int64_t r = tid; r <= n; r += nth)
        if ((int64_t)rp[r] != L * r) bad = 1;
    // col, four int4 groups per thread per iteration
    const int4 *c4 = reinterpret_cast<const int4 *>(col);
    const int64_t ng = nnz >> 2;
    // the four entries of a group share their row and clamp_band is monotone: the group's band is that of its
    // smallest and largest column (6 integer min / max and two clamps instead of eight 64-bit differences)
    auto band = [&](const int4 &v, int64_t g) {
        const int64_t row = (g << 2) >> lgL;
        const int cmin = min(min(v.x, v.y), min(v.z, v.w)), cmax = max(max(v.x, v.y), max(v.z, v.w));
        blo = max(blo, clamp_band(row - (int64_t)cmin));
        bhi = max(bhi, clamp_band((int64_t)cmax - row));
    };
    int64_t g = tid;
    for (; g + 3 * nth < ng; g += 4 * nth) {
        const int4 v0 = ldg_stream_i4(c4 + g), v1 = ldg_stream_i4(c4 + g + nth);
        const int4 v2 = ldg_stream_i4(c4 + g + 2 * nth), v3 = ldg_stream_i4(c4 + g + 3 * nth);
        band(v0, g);
        band(v1, g + nth);
        band(v2, g + 2 * nth);
        band(v3, g + 3 * nth);
    }
    for (; g < ng; g += nth) band(ldg_stream_i4(c4 + g), g);
    for (int o = 16; o > 0; o >>= 1) {
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
        blo = max(blo, __shfl_xor_sync(0xffffffffu, blo, o));
        bhi = max(bhi, __shfl_xor_sync(0xffffffffu, bhi, o));
    }
    __shared__ int sb[3][8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        sb[0][warp] = bad;
        sb[1][warp] = blo;
        sb[2][warp] = bhi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); w++) {
            bad |= sb[0][w];
            blo = max(blo, sb[1][w]);
            bhi = max(bhi, sb[2][w]);
        }
        if (bad) atomicOr(&out->nonuniform, 1);
        atomicMax(&out->blo, blo);
        atomicMax(&out->bhi, bhi);
    }
}

// Column range [min, max] of every tile of `tile` rows (one warp per tile); empty tile -> [0, -1].
__global__ void csr_tile_range_kernel(int64_t n, const int32_t *__restrict__ rp, const int32_t *__restrict__ col,
                                      int tile, int32_t *tlo, int32_t *thi)
{
    const int lane = threadIdx.x & 31;
    const int64_t ntiles = (n + tile - 1) / tile;
    for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < ntiles;
         t += (int64_t)gridDim.x * (blockDim.x >> 5)) {
        const int64_t r0 = t * tile, r1 = min(n, r0 + tile);
        const int e0 = rp[r0], e1 = rp[r1];
        int lo = 0x7fffffff, hi = -1;
        for (int e = e0 + lane; e < e1; e += 32) {
            const int c = col[e];
            lo = min(lo, c);
            hi = max(hi, c);
        }
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) {
            tlo[t] = hi >= 0 ? lo : 0;
            thi[t] = hi;
        }
    }
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
        int64_t e0 = (2 * S.dim + 1) * r - miss;
        if (S.diag) {
            // 9-point: row (i, j) holds (1 + [j>0] + [j<ny-1]) (1 + [i>0] + [i<nx-1]) entries; a full
            // x-line sums to 3 nx - 2 per y-factor, the first i rows of a line to 3 i - [i > 0]
            const int64_t ny = S.ny, jr = r / nx, ir = r - jr * nx;
            auto yf = [&](int64_t j) { return 1 + (j > 0) + (j < ny - 1); };
            int64_t full = 0;                              // sum of y-factors of lines 0 .. jr-1
            if (jr > 0) full = 3 * jr - 1 - (jr > ny - 1 ? 1 : 0);
            e0 = full * (3 * nx - 2) + (jr < ny ? yf(jr) * (3 * ir - (ir > 0 ? 1 : 0)) : 0);
        }
        rp[r] = (int32_t)e0;
        if (r == n) break;
        const int64_t i = r % nx, jj = (r / nx) % S.ny, kk = r / pl;
        int64_t e = e0;
        if (S.diag) {
            // ascending columns: (i-1,j-1) (i,j-1) (i+1,j-1) (i-1,j) (i,j) (i+1,j) (i-1,j+1) (i,j+1) (i+1,j+1)
            const double cy[3][3] = {{S.c[7], S.c[3], S.c[8]}, {S.c[1], S.c[0], S.c[2]}, {S.c[9], S.c[4], S.c[10]}};
            for (int dy = -1; dy <= 1; dy++) {
                if ((dy < 0 && jj == 0) || (dy > 0 && jj == S.ny - 1)) continue;
                for (int dx = -1; dx <= 1; dx++) {
                    if ((dx < 0 && i == 0) || (dx > 0 && i == nx - 1)) continue;
                    col[e] = (int32_t)(r + dy * nx + dx);
                    val[e] = cy[dy + 1][dx + 1];
                    e++;
                }
            }
            continue;
        }
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
