// persist_cl.cuh — the Lanczos extension k0 -> k1 (Algorithm 2) of a stencil operator on
// ONE thread-block cluster of CS <= 16 CTAs, for the latency-bound sizes (c2: n = 65536).
//
// The grid-wide kernels pay a grid barrier (1-2 us) per reduction, two per Lanczos step.  Here the
// vector lives in the cluster's shared memory instead: CTA c owns rows [c rpc, (c+1) rpc), keeps
// v~_j for them plus `reach` halo rows on each side (reach = the stencil's largest offset) in shared
// memory (padded by one zero slot per grid line, see cl_pad) and v~_j, v~_{j-1} of its rows in
// registers, and every exchange is a push over DSMEM:
//   * the two block totals of a step (t_jj's dot, ||v~_{j+1}||^2): each CTA st.async's its total into
//     slot c of every CTA's slot array, completing `bytes` on that CTA's mbarrier; every CTA then sums
//     the CS slots in the same fixed pairwise order, so all CTAs hold the identical value;
//   * the halo of v~_{j+1}: the first / last `reach` rows of a CTA go to the neighbours' halo rows,
//     again completing bytes on the receiver's mbarrier.
// No buffer needs double-buffering: a CTA can only push step j+1's data after receiving every
// CTA's contribution to a later reduction, which each CTA sends after it has finished reading the
// step-j data in question (see the ordering notes at the pushes).  Each mbarrier is re-armed by
// thread 0 right after its wait; a push that lands before the re-arm only makes the tx-count
// transiently negative (the phase still needs thread 0's arrival to complete).  With the norm
// pipelined (below), the slot array of the norm is rewritten at step j+1 only after every CTA's
// dot total of step j+1 was received, which each CTA sends after reading the norm of step j.
//
// Per row the arithmetic is krylov_small_lanczos_kernel's (rows summed in ascending column order as
// a sequential CSR sum, the same sigma scaling and Lanczos term); the dot and norm are summed in
// another order (rows per thread, warps, CTAs).  CTA 0's thread 0 writes H, sigma and the state.
#pragma once

#include "kernels.cuh"
#include "small.cuh"

#include <algorithm>

namespace phipm {

constexpr int CLZ_MAXCS = 16;

// phase clock of CTA 0 / thread 0 (tools/clz_probe.cu builds with CLZ_CLOCKS; the library never does)
#ifdef CLZ_CLOCKS
__device__ long long clz_clk[16];
#define CLZ_STAMP(i)                                                  \
    {                                                                 \
        const long long c_ = clock64();                               \
        clz_acc[i] += c_ - clz_prev;                                  \
        clz_prev = c_;                                                \
    }
#else
#define CLZ_STAMP(i)
#endif

__device__ __forceinline__ uint32_t cl_smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint32_t cl_mapa(uint32_t a, uint32_t rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}

__device__ __forceinline__ void cl_st_async(uint32_t raddr, double v, uint32_t rbar)
{
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];"
                 ::"r"(raddr), "d"(v), "r"(rbar) : "memory");
}

__device__ __forceinline__ void cl_bar_init(uint64_t *bar)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cl_smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void cl_arm(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(cl_smem_u32(bar)), "r"(bytes)
                 : "memory");
}

// wait for phase `par`, bounded (a lost push must not hang the GPU): false after ~2 s
__device__ __forceinline__ bool cl_wait(uint64_t *bar, uint32_t par)
{
    const uint32_t a = cl_smem_u32(bar);
    unsigned long long t0 = 0;
    for (int it = 0;; it++) {
        uint32_t ok;
        asm volatile(
            "{\n.reg .pred p;\n"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(a), "r"(par)
            : "memory");
        if (ok) return true;
        if ((it & 1023) == 1023) {
            if (t0 == 0) t0 = gtimer();
            else if (gtimer() - t0 > 2000000000ull) return false;
        }
    }
}

__device__ __forceinline__ void cl_cluster_sync()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t cl_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// Padded row index: every grid line is followed by one ghost slot and, in 3-D, every plane by one
// ghost line, P(r) = i + (nx+1) (j + (ny+1) k) for r = i + nx (j + ny k) (floor division for the
// halo rows below the grid; 1-D and 2-D: P(r) = i + (nx+1) q with q = floor(r / nx)).  The ghost
// slots and the halo rows outside the grid hold zeros, so every neighbour of a row can be loaded
// unconditionally: an absent neighbour reads 0 and adds c * 0 = +-0 to the row sum, which leaves
// it unchanged (the arithmetic of a sequential CSR sum over the present entries).
__host__ __device__ inline int64_t cl_pad(int64_t r, int dim, int nx, int ny)
{
    const int64_t q = r >= 0 ? r / nx : -((-r + nx - 1) / nx);
    const int64_t i = r - q * nx;
    if (dim < 3) return i + (int64_t)(nx + 1) * q;
    const int64_t k = q >= 0 ? q / ny : -((-q + ny - 1) / ny);
    const int64_t j = q - k * ny;
    return i + (int64_t)(nx + 1) * (j + (int64_t)(ny + 1) * k);
}

// (A x)_r from the padded local copy (x[p] = x_r, neighbours at p +- 1, +- (nx+1), +- (ny+1)(nx+1)),
// ascending column order with separately rounded products (row_apply, small.cuh).  DC: dimension
// class 1, 2, 3 or 4 (2-D 9-point).
template <int DC>
__device__ __forceinline__ double cl_row(const StencilOp &S, const double *x, int p, int lx, int pl, double xc)
{
    double s = 0.0;
    if (DC == 3) s = __dadd_rn(s, __dmul_rn(S.c[5], x[p - pl]));
    if (DC == 4) s = __dadd_rn(s, __dmul_rn(S.c[7], x[p - lx - 1]));
    if (DC >= 2) s = __dadd_rn(s, __dmul_rn(S.c[3], x[p - lx]));
    if (DC == 4) s = __dadd_rn(s, __dmul_rn(S.c[8], x[p - lx + 1]));
    s = __dadd_rn(s, __dmul_rn(S.c[1], x[p - 1]));
    s = __dadd_rn(s, __dmul_rn(S.c[0], xc));               // x[p], held in a register
    s = __dadd_rn(s, __dmul_rn(S.c[2], x[p + 1]));
    if (DC == 4) s = __dadd_rn(s, __dmul_rn(S.c[9], x[p + lx - 1]));
    if (DC >= 2) s = __dadd_rn(s, __dmul_rn(S.c[4], x[p + lx]));
    if (DC == 4) s = __dadd_rn(s, __dmul_rn(S.c[10], x[p + lx + 1]));
    if (DC == 3) s = __dadd_rn(s, __dmul_rn(S.c[6], x[p + pl]));
    return s;
}

struct ClArgs {
    int64_t rpc;       // rows per CTA (the last CTA may have fewer, but at least `reach`)
    int reach;         // largest stencil offset: 1 (1-D), nx (+1 with corners), nx ny (3-D)
    int cs;            // CTAs in the cluster (= gridDim.x)
    int blen;          // doubles of the padded buffer (cl_buf_len)
};

// shared-memory doubles of the largest CTA buffer: padded rows [r0 - reach, r0 + rpc + reach) and the
// neighbours of its last row
inline int64_t cl_buf_len(const StencilOp &op, int64_t rpc, int reach, int cs)
{
    int64_t mx = 0;
    for (int c = 0; c < cs; c++) {
        const int64_t r0 = (int64_t)c * rpc;
        mx = std::max(mx, cl_pad(r0 + rpc + reach, op.dim, op.nx, op.ny) - cl_pad(r0 - reach, op.dim, op.nx, op.ny));
    }
    return mx + 2 * (op.nx + 1) + 8;
}

// Cluster sum, first half: the CTA total of one value per thread (warp shuffle tree, warps in order)
// and, with cs > 1, its push into slot `me` of every CTA's slot array.
template <int NT>
__device__ __forceinline__ void cl_send(double v, double *wred, double *slots, uint64_t *bar, int cs, uint32_t me)
{
    constexpr int NW = NT / 32;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    v = warp_sum(v);
    if (lane == 0) wred[warp] = v;
    __syncthreads();
    if (cs > 1 && warp == 0) {
        // lane l holds warp (l mod NW)'s total: the log2(NW)-level tree gives every lane the CTA total
        double p = wred[lane & (NW - 1)];
#pragma unroll
        for (int o = NW / 2; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
        if (lane < cs) cl_st_async(cl_mapa(cl_smem_u32(slots + me), lane), p, cl_mapa(cl_smem_u32(bar), lane));
    }
}

// Second half: the cluster total, identical in every thread of every CTA
template <int NT>
__device__ __forceinline__ double cl_recv(const double *wred, const double *slots, uint64_t *bar, uint32_t &par,
                                          int cs, bool &ok)
{
    constexpr int NW = NT / 32;
    if (cs == 1) {
        double p = wred[threadIdx.x & (NW - 1)];
#pragma unroll
        for (int o = NW / 2; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
        return p;
    }
    ok = cl_wait(bar, par) && ok;
    par ^= 1u;
    if (threadIdx.x == 0) cl_arm(bar, 8u * cs);          // the next phase (see the header)
    // fixed pairwise order over the 16 slots (slots >= cs hold zeros, set at kernel entry)
    double q[4];
#pragma unroll
    for (int g = 0; g < 4; g++) q[g] = (slots[4 * g] + slots[4 * g + 1]) + (slots[4 * g + 2] + slots[4 * g + 3]);
    return (q[0] + q[1]) + (q[2] + q[3]);
}

// The step loop is software-pipelined by one reduction: the norm ||v~_{j+1}||^2 of step j is sent at
// the end of step j and received after step j+1's raw SpMV u = A v~_{j+1} (which needs only v~_{j+1}
// and its halo), so the cluster round trip of the norm overlaps the SpMV.  y = sigma_{j+1} u - lz
// v~_j is then formed with exactly the arithmetic of the unpipelined step (sj * s, then the FMA).
template <int NT, int R, int DC>
__global__ void __launch_bounds__(NT, 1) krylov_cluster_lanczos_kernel(StencilOp op, SmallArgs a, ClArgs ca, Work wk)
{
    extern __shared__ __align__(16) double xs[];        // padded rows [r0 - reach, r0 + rows + reach)
    __shared__ double wred[2][NT / 32];
    __shared__ __align__(8) double slots[2][CLZ_MAXCS];
    __shared__ uint64_t rbar[2], hbar;
    const int t = threadIdx.x;
    const int cs = ca.cs;
    const uint32_t me = cs > 1 ? cl_rank() : 0u;
    const int64_t n = op.n;
    const int nx = op.nx;
    const int64_t r0 = (int64_t)me * ca.rpc;
    const int rows = (int)min(ca.rpc, n - r0);
    const int reach = ca.reach;
    const bool has_lo = me > 0, has_hi = (int)me < cs - 1;
    const uint32_t hbytes = 8u * reach * ((has_lo ? 1 : 0) + (has_hi ? 1 : 0));
    const int64_t pb = cl_pad(r0 - reach, op.dim, nx, op.ny);   // padded index of buffer slot 0
    const int lx = nx + 1, pl = (nx + 1) * (op.ny + 1);   // padded line / plane strides
    if (cs > 1) {
        if (t == 0) {
            cl_bar_init(&rbar[0]);
            cl_bar_init(&rbar[1]);
            cl_bar_init(&hbar);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            cl_arm(&rbar[0], 8u * cs);
            cl_arm(&rbar[1], 8u * cs);
            cl_arm(&hbar, hbytes);
        }
        cl_cluster_sync();
    }
    // zero the buffer (ghost slots, halo rows outside the grid), then load v~_{k0}
    for (int k = t; k < ca.blen; k += NT) xs[k] = 0.0;
    pdl_wait();
    __syncthreads();
    int pi[R];                                            // padded buffer slot of own row i
    double xv[R], zv[R];
    const double *vk = wk.V + (int64_t)a.k0 * wk.ldv;
#pragma unroll
    for (int i = 0; i < R; i++) {
        const int l = t + NT * i;
        xv[i] = zv[i] = 0.0;
        pi[i] = 0;
        if (l < rows) {
            pi[i] = (int)(cl_pad(r0 + l, op.dim, nx, op.ny) - pb);
            xv[i] = vk[r0 + l];
            if (a.k0 > 0) zv[i] = wk.V[(int64_t)(a.k0 - 1) * wk.ldv + r0 + l];
        }
    }
    {
        const int64_t lo = max((int64_t)0, r0 - reach), hi = min(n, r0 + rows + reach);
        for (int64_t r = lo + t; r < hi; r += NT) xs[cl_pad(r, op.dim, nx, op.ny) - pb] = vk[r];
    }
    double sj = wk.sigma[a.k0];
    double lz = wk.st->lz;
    int brk = wk.st->brk;
    uint32_t rpar[2] = {0u, 0u}, hpar = 0u;
    bool ok = true;
    // remote halo destinations: my first `reach` rows -> CTA me-1's upper halo, my last -> CTA me+1's
    // lower one; a row's slot there is its slot here shifted by the difference of the buffer origins
    const uint32_t xs_u = cl_smem_u32(xs);
    const int dlo = has_lo ? (int)(pb - cl_pad(r0 - ca.rpc - reach, op.dim, nx, op.ny)) : 0;
    const int dhi = has_hi ? (int)(pb - cl_pad(r0 + ca.rpc - reach, op.dim, nx, op.ny)) : 0;
    const uint32_t lo_dst = has_lo ? cl_mapa(xs_u, me - 1) : 0u;
    const uint32_t lo_bar = has_lo ? cl_mapa(cl_smem_u32(&hbar), me - 1) : 0u;
    const uint32_t hi_dst = has_hi ? cl_mapa(xs_u, me + 1) : 0u;
    const uint32_t hi_bar = has_hi ? cl_mapa(cl_smem_u32(&hbar), me + 1) : 0u;
    if (t < CLZ_MAXCS && t >= cs) slots[0][t] = slots[1][t] = 0.0;
    __syncthreads();
#ifdef CLZ_CLOCKS
    long long clz_prev = clock64(), clz_acc[6] = {0, 0, 0, 0, 0, 0};
#endif
    if (brk < 0) {
        for (int j = a.k0; j <= a.k1; j++) {
            const bool step = j < a.k1;                   // else: only receive step k1-1's norm
            if (step && j > a.k0 && hbytes) {             // halo of v~_j from the neighbours
                ok = cl_wait(&hbar, hpar) && ok;
                hpar ^= 1u;
                if (t == 0) cl_arm(&hbar, hbytes);
            }
            CLZ_STAMP(0)
            double u[R];
            if (step) {
#pragma unroll
                for (int i = 0; i < R; i++)
                    u[i] = (t + NT * i < rows) ? cl_row<DC>(op, xs, pi[i], lx, pl, xv[i]) : 0.0;
            }
            CLZ_STAMP(1)
            if (j > a.k0) {                               // step j-1's norm: h_{j,j-1}, sigma_j
                const double tot = cl_recv<NT>(wred[1], slots[1], &rbar[1], rpar[1], cs, ok);
                const double h = sqrt(tot);
                const double sn = 1.0 / h;
                const double lzn = h * sj;
                int b = -1;
                if (!isfinite(h)) b = j;
                else if (h <= a.bthr) b = j;
                if (t == 0 && me == 0) {
                    wk.H[j + (size_t)(j - 1) * wk.ldh] = h;
                    if (j < wk.hcols) wk.H[(j - 1) + (size_t)j * wk.ldh] = h;
                    wk.st->lz = lzn;
                    wk.sigma[j] = sn;
                    if (!isfinite(h)) wk.st->nonfinite = 1;
                    if (b >= 0) wk.st->brk = b;
                }
                sj = sn;
                lz = lzn;
                brk = b;
            }
            CLZ_STAMP(4)
            if (!step || brk >= 0 || !ok) break;
            double y[R];
            double dl = 0.0;
#pragma unroll
            for (int i = 0; i < R; i++) {
                y[i] = 0.0;
                if (t + NT * i < rows) {
                    y[i] = sj * u[i];
                    if (j > 0) y[i] = fma(-lz, zv[i], y[i]);
                }
                dl = fma(xv[i], y[i], dl);
            }
            // (every CTA sends this total after its SpMV: once the cluster total is in, no CTA reads
            // v~_j's halo any more, so the halo pushes of v~_{j+1} below cannot overwrite live data)
            cl_send<NT>(dl, wred[0], slots[0], &rbar[0], cs, me);
            const double d = cl_recv<NT>(wred[0], slots[0], &rbar[0], rpar[0], cs, ok);
            CLZ_STAMP(2)
            const double al = sj * d;                     // t_jj = sigma_j v~_j^T y
            const double g = al * sj;
            if (t == 0 && me == 0) {
                wk.H[j + (size_t)j * wk.ldh] = al;
                wk.g[0] = g;
            }
            const bool push = cs > 1 && j + 1 < a.k1;
            double wl = 0.0;
#pragma unroll
            for (int i = 0; i < R; i++) {
                const int l = t + NT * i;
                if (l < rows) {
                    const double w = fma(-g, xv[i], y[i]);   // v~_{j+1} = y - g v~_j
                    wk.V[(int64_t)(j + 1) * wk.ldv + r0 + l] = w;
                    xs[pi[i]] = w;                        // every local read of v~_j preceded the sum
                    wl = fma(w, w, wl);
                    if (push) {
                        if (has_lo && l < reach) cl_st_async(lo_dst + 8u * (uint32_t)(pi[i] + dlo), w, lo_bar);
                        if (has_hi && l >= rows - reach) cl_st_async(hi_dst + 8u * (uint32_t)(pi[i] + dhi), w, hi_bar);
                    }
                    zv[i] = xv[i];
                    xv[i] = w;
                }
            }
            CLZ_STAMP(3)
            cl_send<NT>(wl, wred[1], slots[1], &rbar[1], cs, me);
            CLZ_STAMP(5)
        }
    }
#ifdef CLZ_CLOCKS
    if (t == 0 && me == 0)
        for (int i = 0; i < 6; i++) clz_clk[i] = clz_acc[i];
#endif
    // every push into a CTA's shared memory was awaited by it (a breakdown is detected after the
    // next step's halo wait), so only a timed-out wait leaves the cluster out of step
    if (!ok) {
        if (t == 0) wk.st->aborted = 1;
        return;                                          // (a timed-out cluster cannot synchronise)
    }
    if (cs > 1) cl_cluster_sync();
}

} // namespace phipm
