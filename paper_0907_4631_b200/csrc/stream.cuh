// stream.cuh — the two n-sized kernels of a phipm step (sm_100a, fp64):
//
//   spmv_stream   y = s (A x) + sum_i c_i z_i ; d_k = v~_k^T y for a column range ; ||y||^2
//   axpy_stream   out = a0 base + sum_k c_k v~_k + sum_i e_i E_i ; ||out||^2
//
// Design (measured on this B200 with tools/stream_roof.cu: plain 16-B loads reach ~7.0 TB/s
// read-only, 1-D TMA bulk copies only do so with >= 16-32 KB per copy):
//   * Tiles of TILE = SNT * RPT rows (SNT = 1024 threads, one CTA per SM); each thread owns RPT rows
//     as RPT/2 double2 pairs (rows 2 tid + 2 SNT h, +1) and keeps its y values in registers from the
//     SpMV through the dot products, so y never round-trips through memory inside the kernel.
//   * Streamed Krylov columns are read with 16-B non-allocating loads, CU columns x RPT/2 pairs
//     in flight per thread (64-128 B/thread, one 1024-thread CTA per SM), which saturates HBM.
//   * Stencil operators stage their halo tile in shared memory with 1-D TMA (cp.async.bulk,
//     SASS UBLKCP): in 2-D/3-D the centre row range and the +-nx neighbour ranges are one
//     contiguous copy [r0 - nx, r0 + TILE + nx), the +-nx*ny ranges (3-D) two more; the next
//     tile's halo is issued as soon as the current one has been consumed, so the copy overlaps
//     the epilogue and the dot products.
//   * CSR rows are computed by groups of 2^glog lanes with 8 row groups in flight per lane.
// Both kernels end in the deterministic last-block grid reduction + finalize of kernels.cuh.
// All TMA sources are workspace vectors padded to ldv (a multiple of 32 doubles).
#pragma once

#include "kernels.cuh"

namespace phipm {

#ifndef PHIPM_SNT
#define PHIPM_SNT 1024
#endif
constexpr int SNT = PHIPM_SNT;          // threads per CTA: one 1024-thread CTA per SM (fewer partials
                                        // to reduce, less halo re-read per row than 4 x 256)
constexpr int SNW = SNT / 32;
constexpr int SMINB = 1024 / SNT;       // resident CTAs per SM the register budget is sized for
#ifndef PHIPM_CU
#define PHIPM_CU 4
#endif
constexpr int CU = PHIPM_CU;            // columns in flight per thread
// banded uniform-row CSR: x lives in a shared-memory ring of XRING doubles (x[c] at c mod XRING)
// that slides with the CTA's row range; each tile's 1-D bulk copy brings in only the new chunk
constexpr int XRING = 16384;
constexpr int MAXITEM = MAXD + MAXZ + 2;

// ---------------------------------------------------------------------------------------------
// mbarrier + bulk-copy primitives (PTX)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// 1-D TMA: global -> shared, completion counted on an mbarrier (bytes % 16 == 0, 16-B aligned)
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// bulk prefetch of [src, src + bytes) into L2 (TMA engine, no shared memory; 16-B granularity)
__device__ __forceinline__ void tma_prefetch_l2(const void *src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// L2 prefetch of rows [0, rows) of a vector (a tile segment); the bulk prefetch needs a 16-B aligned
// address and a multiple of 16 bytes: unaligned vectors are skipped, an odd last row is left out
__device__ __forceinline__ void prefetch_rows(const double *p, int rows)
{
    const uint32_t bytes = ((uint32_t)rows * 8u) & ~15u;
    if (((uintptr_t)p & 15) == 0 && bytes) tma_prefetch_l2(p, bytes);
}

// 16-B read-only load that does not allocate in L1 (streamed Krylov columns)
__device__ __forceinline__ double2 ld_stream2(const double *p)
{
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}

// ---------------------------------------------------------------------------------------------
// halo plan of a stencil tile: the x ranges the tile's rows read, rounded out to even indices,
// clamped to [0, ldx).  Segment 0 = centre (1-D: [r0-1, r0+rows+1); 2-D/3-D with nx <= TILE the
// union [r0-nx, r0+rows+nx)); with nx > TILE the y-/y+ ranges are separate segments; in 3-D the
// z-/z+ ranges follow.  off[k] is the segment's offset in the shared halo buffer (doubles).

struct HaloPlan {
    int nseg;
    int64_t start[5];
    uint32_t bytes[5];
    int off[5];
    int ylo, yhi, zlo, zhi;          // segment holding the y-, y+, z-, z+ neighbours
};

__host__ __device__ inline bool halo_union(int nx, int tile) { return nx <= tile; }

// capacity of the shared halo buffer (doubles) for a stencil with this geometry
__host__ __device__ inline int halo_capacity(int dim, int nx, int tile)
{
    if (dim == 1) return tile + 4;
    int c = halo_union(nx, tile) ? tile + 2 * nx + 8 : 3 * (tile + 8);     // (+-1 for 9-point corners)
    if (dim == 3) c += 2 * (tile + 4);
    return c;
}

__device__ __forceinline__ void seg_range(int64_t lo, int64_t hi, int64_t ldx, int64_t &start, uint32_t &bytes)
{
    lo = lo < 0 ? 0 : (lo & ~(int64_t)1);
    hi = hi > ldx ? ldx : ((hi + 1) & ~(int64_t)1);
    start = lo;
    bytes = hi > lo ? (uint32_t)((hi - lo) * 8) : 0u;
}

__device__ __forceinline__ void halo_plan(const StencilOp &S, int tile, int64_t r0, int rows, int64_t ldx, HaloPlan &h)
{
    int k = 0, off = 0;
    auto add = [&](int64_t lo, int64_t hi, int cap) {
        seg_range(lo, hi, ldx, h.start[k], h.bytes[k]);
        h.off[k] = off;
        off += cap;
        return k++;
    };
    if (S.dim == 1) {
        add(r0 - 1, r0 + rows + 1, tile + 4);
        h.ylo = h.yhi = 0;
    } else if (halo_union(S.nx, tile)) {
        const int d = S.diag ? 1 : 0;                       // corner neighbours x[r -+ nx -+ 1]
        h.ylo = h.yhi = add(r0 - S.nx - d, r0 + rows + S.nx + d, tile + 2 * S.nx + 8);
    } else {
        const int d = S.diag ? 1 : 0;
        add(r0 - 1, r0 + rows + 1, tile + 8);
        h.ylo = add(r0 - S.nx - d, r0 - S.nx + rows + d, tile + 8);
        h.yhi = add(r0 + S.nx - d, r0 + S.nx + rows + d, tile + 8);
    }
    h.zlo = h.zhi = 0;
    if (S.dim == 3) {
        const int64_t pl = (int64_t)S.nx * S.ny;
        h.zlo = add(r0 - pl, r0 - pl + rows, tile + 4);
        h.zhi = add(r0 + pl, r0 + pl + rows, tile + 4);
    }
    h.nseg = k;
}

__device__ __forceinline__ void halo_plan_ident(int64_t r0, int rows, int64_t ldx, HaloPlan &h)
{
    h.nseg = 1;
    h.off[0] = 0;
    h.ylo = h.yhi = h.zlo = h.zhi = 0;
    seg_range(r0, r0 + rows, ldx, h.start[0], h.bytes[0]);
}

// grid coordinates of row r (two 32-bit divisions)
__device__ __forceinline__ void grid_ijk(const StencilOp &S, int64_t r, int &i, int &jj, int &kk)
{
    const unsigned ur = (unsigned)r, unx = (unsigned)S.nx;
    const unsigned q = ur / unx;
    i = (int)(ur - q * unx);
    jj = 0;
    kk = 0;
    if (S.dim >= 2) {
        const unsigned uny = (unsigned)S.ny;
        const unsigned q2 = q / uny;
        jj = (int)(q - q2 * uny);
        kk = (int)q2;
    }
}

// CSR rows of a tile into ys: G = 2^glog lanes per row, U row groups in flight per lane (memory-
// level parallelism for the col -> x gather chain), rows longer than G strided, shuffle reduce.
// WIN: x is gathered from the tile's x window in shared memory (xs[c - xs0]) instead of global
// memory; `wait` is called once, after the first batch of row_ptr/col/val loads is in flight and
// before the first x access (it waits for the window's TMA copy).
template <bool WIN, class Wait>
__device__ __forceinline__ void csr_tile(const CsrOp &A, const double *__restrict__ x, const double *xs, int64_t xs0,
                                         int64_t r0, int rows, double *ys, Wait wait)
{
    constexpr int U = 8;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int G = 1 << A.glog;
    const int rpw = 32 >> A.glog;
    const int sub = lane >> A.glog, li = lane & (G - 1);
    const int stride = SNW * rpw;
    bool waited = false;
    auto X = [&](int c) -> double {
        if constexpr (WIN) return xs[c - xs0];
        else return __ldg(x + c);
    };
    for (int base = warp * rpw; base < rows; base += stride * U) {
        int q[U], e[U], e1[U];
        double acc[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            q[u] = base + u * stride + sub;
            const bool ok = q[u] < rows;
            e[u] = ok ? __ldg(A.rp + r0 + q[u]) + li : 0;
            e1[u] = ok ? __ldg(A.rp + r0 + q[u] + 1) : 0;
        }
        int cc[U];
        double vv[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const bool ok = e[u] < e1[u];
            cc[u] = ok ? __ldg(A.col + e[u]) : 0;
            vv[u] = ok ? ldg_stream(A.val + e[u]) : 0.0;
        }
        if (!waited) {
            wait();
            waited = true;
        }
#pragma unroll
        for (int u = 0; u < U; u++) acc[u] = (e[u] < e1[u]) ? vv[u] * X(cc[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < U; u++)
            for (int f = e[u] + G; f < e1[u]; f += G) acc[u] = fma(ldg_stream(A.val + f), X(__ldg(A.col + f)), acc[u]);
#pragma unroll
        for (int u = 0; u < U; u++) {
            for (int o = G >> 1; o > 0; o >>= 1) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
            if (q[u] < rows && li == 0) ys[q[u]] = acc[u];
        }
    }
    if (!waited) wait();
}

// Uniform-row-length CSR (row_ptr[r] = L r, L % 4 == 0): G = L/4 lanes per row, each lane loads 4
// consecutive entries with 16-B vector loads (val: 2 x double2, col: int4), U row groups in flight
// per lane; products summed in entry order per lane, then a log2(G)-level shuffle tree.
// XM: 0 gathers x from global memory, 1 from the tile's x window (xs[c - xs0]), 2 from the x ring
// (xs[c mod XRING])
template <int XM>
__device__ __forceinline__ void csr_tile_ell(const CsrOp &A, const double *__restrict__ x, const double *xs, int64_t xs0,
                                             int64_t r0, int rows, double *ys, double *amax = nullptr)
{
#ifndef PHIPM_ELL_U
#define PHIPM_ELL_U 3
#endif
    constexpr int U = PHIPM_ELL_U;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int G = A.ell >> 2;                 // lanes per row (power of two, <= 32)
    const int rpw = 32 / G;
    const int sub = lane / G, li = lane - sub * G;
    const int stride = SNW * rpw;
    auto X = [&](int c) -> double {
        if constexpr (XM == 1) return xs[c - xs0];
        else if constexpr (XM == 2) return xs[c & (XRING - 1)];
        else return __ldg(x + c);
    };
    for (int base = warp * rpw; base < rows; base += stride * U) {
        if constexpr (XM == 2) {
            // L2 prefetch (TMA engine) of the val / col rows pf ahead of this block of stride * U
            // rows, issued by the first thread, so the 16-B loads below hit L2
            if (A.pf > 0 && threadIdx.x == 0) {
                const int64_t pa = r0 + base + A.pf, pb = min(pa + (int64_t)stride * U, A.pf_end);
                if (pb > pa) {
                    tma_prefetch_l2(A.val + pa * A.ell, (uint32_t)((pb - pa) * A.ell * 8));
                    if (A.off16) tma_prefetch_l2(A.off16 + pa * A.ell, (uint32_t)((pb - pa) * A.ell * 2));
                    else tma_prefetch_l2(A.col + pa * A.ell, (uint32_t)((pb - pa) * A.ell * 4));
                }
            }
        }
        double2 va[U], vb[U];
        int4 cc[U];
        // column indices of all U groups first: the x lookups depend on them, the values only on
        // the products, so the index loads are the ones to put at the head of the queue
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int q = base + u * stride + sub;
            if (XM == 2 && A.off16) {
                // int16 offsets col - row: 8 B per lane instead of 16
                int2 o = q < rows ? __ldg(reinterpret_cast<const int2 *>(A.off16 + (r0 + q) * (int64_t)A.ell + 4 * li))
                                  : make_int2(0, 0);
                const int rr = (int)(r0 + q);
                cc[u] = make_int4(rr + (int)(short)(o.x & 0xffff), rr + (o.x >> 16), rr + (int)(short)(o.y & 0xffff),
                                  rr + (o.y >> 16));
                if (q >= rows) cc[u] = make_int4(0, 0, 0, 0);
            } else {
                cc[u] = q < rows ? __ldg(reinterpret_cast<const int4 *>(A.col + (r0 + q) * (int64_t)A.ell + 4 * li))
                                 : make_int4(0, 0, 0, 0);
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int q = base + u * stride + sub;
            if (q < rows) {
                const int64_t e = (r0 + q) * (int64_t)A.ell + 4 * li;
                va[u] = ldg_stream2(A.val + e);
                vb[u] = ldg_stream2(A.val + e + 2);
            } else {
                va[u] = vb[u] = make_double2(0.0, 0.0);
            }
        }
        double acc[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int q = base + u * stride + sub;
            double t = 0.0;
            if (q < rows) {
                t = va[u].x * X(cc[u].x);
                t = fma(va[u].y, X(cc[u].y), t);
                t = fma(vb[u].x, X(cc[u].z), t);
                t = fma(vb[u].y, X(cc[u].w), t);
            }
            acc[u] = t;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            for (int o = G >> 1; o > 0; o >>= 1) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
            const int q = base + u * stride + sub;
            if (q < rows && li == 0) ys[q] = acc[u];
        }
        if (amax) {
            // ||A||_inf: the row's |a| summed in entry order per lane, lanes by the same shuffle tree
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int q = base + u * stride + sub;
                double s = 0.0;
                if (q < rows) {
                    s = __dadd_rn(s, fabs(va[u].x));
                    s = __dadd_rn(s, fabs(va[u].y));
                    s = __dadd_rn(s, fabs(vb[u].x));
                    s = __dadd_rn(s, fabs(vb[u].y));
                }
                for (int o = G >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                *amax = fmax(*amax, s);
            }
        }
    }
}

// x-ring variant with the column indices software-pipelined one iteration ahead: the gathers of an
// iteration depend on its column loads (L2 latency even after the bulk prefetch; ncu: 13 % of the
// stall samples on the ring-index mask), so the next iteration's int4 column loads are issued before
// this iteration's gathers.  Same products and summation order as csr_tile_ell<2>.
template <int UP>
__device__ __forceinline__ void csr_tile_ell_ring_pipe(const CsrOp &A, const double *xs, int64_t r0, int rows,
                                                       double *ys, double *amax)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int G = A.ell >> 2;
    const int rpw = 32 / G;
    const int sub = lane / G, li = lane - sub * G;
    const int stride = SNW * rpw;
    auto ldc = [&](int q) -> int4 {
        return q < rows ? __ldg(reinterpret_cast<const int4 *>(A.col + (r0 + q) * (int64_t)A.ell + 4 * li))
                        : make_int4(0, 0, 0, 0);
    };
    int4 ccn[UP];
#pragma unroll
    for (int u = 0; u < UP; u++) ccn[u] = ldc(warp * rpw + u * stride + sub);
    for (int base = warp * rpw; base < rows; base += stride * UP) {
        if (A.pf > 0 && threadIdx.x == 0) {
            const int64_t pa = r0 + base + A.pf, pb = min(pa + (int64_t)stride * UP, A.pf_end);
            if (pb > pa) {
                tma_prefetch_l2(A.val + pa * A.ell, (uint32_t)((pb - pa) * A.ell * 8));
                tma_prefetch_l2(A.col + pa * A.ell, (uint32_t)((pb - pa) * A.ell * 4));
            }
        }
        int4 cc[UP];
        double2 va[UP], vb[UP];
#pragma unroll
        for (int u = 0; u < UP; u++) cc[u] = ccn[u];
#pragma unroll
        for (int u = 0; u < UP; u++) {
            const int q = base + u * stride + sub;
            if (q < rows) {
                const int64_t e = (r0 + q) * (int64_t)A.ell + 4 * li;
                va[u] = ldg_stream2(A.val + e);
                vb[u] = ldg_stream2(A.val + e + 2);
            } else {
                va[u] = vb[u] = make_double2(0.0, 0.0);
            }
        }
#pragma unroll
        for (int u = 0; u < UP; u++) ccn[u] = ldc(base + stride * UP + u * stride + sub);
        double acc[UP];
#pragma unroll
        for (int u = 0; u < UP; u++) {
            const int q = base + u * stride + sub;
            double t = 0.0;
            if (q < rows) {
                t = va[u].x * xs[cc[u].x & (XRING - 1)];
                t = fma(va[u].y, xs[cc[u].y & (XRING - 1)], t);
                t = fma(vb[u].x, xs[cc[u].z & (XRING - 1)], t);
                t = fma(vb[u].y, xs[cc[u].w & (XRING - 1)], t);
            }
            acc[u] = t;
        }
#pragma unroll
        for (int u = 0; u < UP; u++) {
            for (int o = G >> 1; o > 0; o >>= 1) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
            const int q = base + u * stride + sub;
            if (q < rows && li == 0) ys[q] = acc[u];
        }
        if (amax) {
#pragma unroll
            for (int u = 0; u < UP; u++) {
                const int q = base + u * stride + sub;
                double s = 0.0;
                if (q < rows) {
                    s = __dadd_rn(s, fabs(va[u].x));
                    s = __dadd_rn(s, fabs(va[u].y));
                    s = __dadd_rn(s, fabs(vb[u].x));
                    s = __dadd_rn(s, fabs(vb[u].y));
                }
                for (int o = G >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                *amax = fmax(*amax, s);
            }
        }
    }
}

// Issue the 1-D TMA copies of one stencil tile's halo x[hr0 - nx(ny), hr0 + hrows + nx(ny)) (thread
// 0 only): ho receives the tile-relative offsets of the centre, y-, y+, z-, z+ segments in hbuf.
template <int TILE_>
__device__ __forceinline__ void issue_halo_tile(const StencilOp &op, double *hbuf, const double *x, int64_t ldx,
                                                int64_t hr0, int hrows, int *ho, uint64_t *bar)
{
    HaloPlan h;
    halo_plan(op, TILE_, hr0, hrows, ldx, h);
    const int seg[5] = {0, h.ylo, h.yhi, h.zlo, h.zhi};
#pragma unroll
    for (int k = 0; k < 5; k++) ho[k] = h.off[seg[k]] - (int)(h.start[seg[k]] - hr0);
    uint32_t tot = 0;
    for (int k = 0; k < h.nseg; k++) tot += h.bytes[k];
    const uint64_t pol = policy_evict_last();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // prior generic reads of hbuf
    mbar_arrive_expect_tx(bar, tot);
    for (int k = 0; k < h.nseg; k++)
        if (h.bytes[k]) tma_load_1d(hbuf + h.off[k], x + h.start[k], h.bytes[k], bar, pol);
}

// A tile's halo plan, computed once per kernel (the segments' offsets relative to the source vector
// do not change from one Krylov column to the next): issuing a tile is then one expect_tx and
// nseg bulk copies, instead of the 64-bit plan arithmetic (local-memory arrays) on the issuing
// thread while its warp waits.
struct TilePlan {
    int64_t start[5];
    uint32_t bytes[5];
    int off[5];
    int ho[5];                       // tile-relative offsets of the centre, y-, y+, z-, z+ segments
    int nseg;
    uint32_t tot;
};

template <int TILE_>
__device__ __forceinline__ void tile_plan(const StencilOp &op, int64_t ldx, int64_t hr0, int hrows, TilePlan &tp)
{
    HaloPlan h;
    halo_plan(op, TILE_, hr0, hrows, ldx, h);
    const int seg[5] = {0, h.ylo, h.yhi, h.zlo, h.zhi};
    uint32_t tot = 0;
#pragma unroll
    for (int k = 0; k < 5; k++) {
        tp.ho[k] = h.off[seg[k]] - (int)(h.start[seg[k]] - hr0);
        tp.start[k] = h.start[k];
        tp.bytes[k] = k < h.nseg ? h.bytes[k] : 0u;
        tp.off[k] = h.off[k];
        tot += tp.bytes[k];
    }
    tp.nseg = h.nseg;
    tp.tot = tot;
}

// issue a planned tile's bulk copies of vector x into hbuf (one thread)
__device__ __forceinline__ void issue_planned_tile(const TilePlan &tp, double *hbuf, const double *x, uint64_t *bar,
                                                   uint64_t pol)
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // prior generic reads of hbuf
    mbar_arrive_expect_tx(bar, tp.tot);
    for (int k = 0; k < tp.nseg; k++)
        if (tp.bytes[k]) tma_load_1d(hbuf + tp.off[k], x + tp.start[k], tp.bytes[k], bar, pol);
}

// The raw rows (A x)_r of one stencil tile from its halo in shared memory (ho: tile-relative
// offsets of the centre, y-, y+, z-, z+ segments), for this thread's NP row pairs
// q = 2 tid + 2 SNT p, and the x values themselves (xr, for a dot with v_j = x).  Ascending column
// order with separately rounded products: bit-exact with a sequential CSR row sum.
// DIM is a template parameter; a pair of rows whose 2 DIM neighbours all lie inside the grid takes
// a branch-free path (the same operations in the same order), boundary pairs test each term.
// gc (optional): grid coordinates (i, j, k) of row r0 + 2 tid on entry, of the next tile's row
// r0 + TILE + 2 tid on return (callers walking consecutive tiles avoid the per-tile divisions)
template <int NP, int DIM, bool DG = false>
__device__ __forceinline__ void stencil_tile_d(const StencilOp &op, const double *hbuf, const int *ho, int64_t r0,
                                               int rows, int tid, double2 (&y)[NP], double2 (&xr)[NP],
                                               int3 *gc = nullptr)
{
    const double *pc = hbuf + ho[0];
    const double *pym = hbuf + ho[1], *pyp = hbuf + ho[2], *pzm = hbuf + ho[3], *pzp = hbuf + ho[4];
    const int nx = op.nx, ny = op.ny, nz = op.nz, pl = op.nx * op.ny;
    const double c0 = op.c[0], cxm = op.c[1], cxp = op.c[2], cym = op.c[3], cyp = op.c[4],
                 czm = op.c[5], czp = op.c[6];
    const double cmm = op.c[7], cpm = op.c[8], cmp = op.c[9], cpp = op.c[10];   // 9-point corners
    // grid coordinates of this thread's first row; later pairs are 2 SNT rows further on
    int i, jj = 0, kk = 0;
    if (gc) {
        i = gc->x;
        jj = gc->y;
        kk = gc->z;
    } else {
        const unsigned ur = (unsigned)(r0 + 2 * tid), unx = (unsigned)nx;
        const unsigned qy = ur / unx;
        i = (int)(ur - qy * unx);
        if (DIM >= 2) {
            const unsigned q2 = qy / (unsigned)ny;
            jj = (int)(qy - q2 * (unsigned)ny);
            kk = (int)q2;
        }
    }
    const int di = DIM >= 2 ? op.sdi : 2 * SNT, dj = DIM >= 2 ? op.sdj : 0;   // 2 SNT = dj nx + di
    // one term of the ascending-column sum, taken only where the neighbour exists: every lane
    // executes the same instructions (a warp spans boundary and interior rows, so per-row branches
    // would run both paths); absent neighbours read a clamped in-buffer index and are discarded
    auto term = [&](double s, bool on, double c, const double *nb, int q) -> double {
        const double v = *(on ? nb : pc + q);              // pc[q] (this row's own x) is always in the buffer
        const double t = __dadd_rn(s, __dmul_rn(c, v));
        return on ? t : s;
    };
    // v: the row exists (rows past the tile end compute row 0 with every neighbour off)
    auto row = [&](bool v, int q, int ii, int j2, int k2) -> double {
        double s = 0.0;
        if (DIM >= 3) s = term(s, v && k2 > 0, czm, pzm + (q - pl), q);
        if (DG) s = term(s, v && j2 > 0 && ii > 0, cmm, pym + (q - nx - 1), q);
        if (DIM >= 2) s = term(s, v && j2 > 0, cym, pym + (q - nx), q);
        if (DG) s = term(s, v && j2 > 0 && ii < nx - 1, cpm, pym + (q - nx + 1), q);
        s = term(s, v && ii > 0, cxm, pc + (q - 1), q);
        s = __dadd_rn(s, __dmul_rn(c0, pc[q]));
        s = term(s, v && ii < nx - 1, cxp, pc + (q + 1), q);
        if (DG) s = term(s, v && j2 < ny - 1 && ii > 0, cmp, pyp + (q + nx - 1), q);
        if (DIM >= 2) s = term(s, v && j2 < ny - 1, cyp, pyp + (q + nx), q);
        if (DG) s = term(s, v && j2 < ny - 1 && ii < nx - 1, cpp, pyp + (q + nx + 1), q);
        if (DIM >= 3) s = term(s, v && k2 < nz - 1, czp, pzp + (q + pl), q);
        return s;
    };
    // Fast pair path (nx even, 5/7-point or 1-D): both rows of a pair lie on one x-line at (i, i+1),
    // i even, and every halo segment offset is even, so the 2 DIM + 1 values each row reads come
    // from 16-B shared loads; when every pair of the warp is y/z-interior (warp-uniform branch) only
    // row a's x- and row b's x+ neighbour can be absent, and an absent value is replaced by 0 before
    // its product: s + c 0 = s exactly (s starts at +0 and can never become -0), so the sums are
    // bit-identical with the per-term path below.
    const bool fastok = !DG && (DIM == 1 || (nx & 1) == 0);
#pragma unroll
    for (int p = 0; p < NP; p++) {
        const int q = 2 * tid + 2 * SNT * p;
        const bool v0 = q < rows, v1 = q + 1 < rows;
        // which of the z-, z+, y-, y+ neighbours the pair has (bits 0..3); the fast path needs the
        // same set for every lane, so a boundary plane or line is skipped by a uniform branch
        int nbm = 0;
        if (DIM >= 2) nbm |= (jj > 0 ? 4 : 0) | (jj < ny - 1 ? 8 : 0);
        if (DIM >= 3) nbm |= (kk > 0 ? 1 : 0) | (kk < nz - 1 ? 2 : 0);
        const int nbm0 = __shfl_sync(0xffffffffu, nbm, 0);
        bool inner = v1 && nbm == nbm0;
        if (DIM == 1) inner = inner && i > 0 && i + 2 < nx;           // 1-D: every neighbour present
        if (!__any_sync(0xffffffffu, v0)) {
            // the whole warp's rows lie past the tile end (last, partial tile)
            xr[p] = make_double2(0.0, 0.0);
            y[p] = make_double2(0.0, 0.0);
        } else if (fastok && __all_sync(0xffffffffu, inner)) {
            auto ld2 = [](const double *a) { return *reinterpret_cast<const double2 *>(a); };
            const double2 xl = ld2(pc + q - 2), xc = ld2(pc + q), xh = ld2(pc + q + 2);
            const double am = (DIM == 1 || i > 0) ? xl.y : 0.0;        // x- of row a
            const double bp = (DIM == 1 || i + 2 < nx) ? xh.x : 0.0;   // x+ of row b
            double sa = 0.0, sb = 0.0;
            if (DIM >= 3 && (nbm0 & 1)) {
                const double2 zm = ld2(pzm + (q - pl));
                sa = __dadd_rn(sa, __dmul_rn(czm, zm.x));
                sb = __dadd_rn(sb, __dmul_rn(czm, zm.y));
            }
            if (DIM >= 2 && (nbm0 & 4)) {
                const double2 ym = ld2(pym + (q - nx));
                sa = __dadd_rn(sa, __dmul_rn(cym, ym.x));
                sb = __dadd_rn(sb, __dmul_rn(cym, ym.y));
            }
            sa = __dadd_rn(sa, __dmul_rn(cxm, am));
            sb = __dadd_rn(sb, __dmul_rn(cxm, xc.x));
            sa = __dadd_rn(sa, __dmul_rn(c0, xc.x));
            sb = __dadd_rn(sb, __dmul_rn(c0, xc.y));
            sa = __dadd_rn(sa, __dmul_rn(cxp, xc.y));
            sb = __dadd_rn(sb, __dmul_rn(cxp, bp));
            if (DIM >= 2 && (nbm0 & 8)) {
                const double2 yp = ld2(pyp + (q + nx));
                sa = __dadd_rn(sa, __dmul_rn(cyp, yp.x));
                sb = __dadd_rn(sb, __dmul_rn(cyp, yp.y));
            }
            if (DIM >= 3 && (nbm0 & 2)) {
                const double2 zp = ld2(pzp + (q + pl));
                sa = __dadd_rn(sa, __dmul_rn(czp, zp.x));
                sb = __dadd_rn(sb, __dmul_rn(czp, zp.y));
            }
            xr[p] = xc;
            y[p] = make_double2(sa, sb);
        } else {
        // second row of the pair: one step along x (wrapping to the next line / plane)
        int i1 = i + 1, j1 = jj, k1 = kk;
        if (i1 == nx) {
            i1 = 0;
            if (DIM >= 2) {
                j1++;
                if (j1 == ny) { j1 = 0; k1++; }
            }
        }
        const int qa = v0 ? q : 0, qb = v1 ? q + 1 : 0;     // rows past the tile: any valid index
        xr[p].x = v0 ? pc[qa] : 0.0;
        xr[p].y = v1 ? pc[qb] : 0.0;
        const double ya = row(v0, qa, i, jj, kk), yb = row(v1, qb, i1, j1, k1);
        y[p].x = v0 ? ya : 0.0;
        y[p].y = v1 ? yb : 0.0;
        }
        if (p + 1 < NP || gc) {
            i += di;
            if (DIM >= 2) {
                jj += dj;
                if (i >= nx) { i -= nx; jj++; }
                while (jj >= ny) { jj -= ny; kk++; }
            }
        }
    }
    if (gc) *gc = make_int3(i, jj, kk);
}

// grid coordinates of row r (divisions; once per kernel for callers that pass gc above)
__device__ __forceinline__ int3 grid_coords(const StencilOp &op, int64_t r)
{
    const unsigned ur = (unsigned)r, unx = (unsigned)op.nx;
    const unsigned qy = ur / unx;
    int3 g = make_int3((int)(ur - qy * unx), 0, 0);
    if (op.dim >= 2) {
        const unsigned q2 = qy / (unsigned)op.ny;
        g.y = (int)(qy - q2 * (unsigned)op.ny);
        g.z = (int)q2;
    }
    return g;
}

template <int NP>
__device__ __forceinline__ void stencil_tile(const StencilOp &op, const double *hbuf, const int *ho, int64_t r0, int rows,
                                             int tid, double2 (&y)[NP], double2 (&xr)[NP], int3 *gc = nullptr)
{
    if (op.dim == 3) stencil_tile_d<NP, 3>(op, hbuf, ho, r0, rows, tid, y, xr, gc);
    else if (op.dim == 2 && op.diag) stencil_tile_d<NP, 2, true>(op, hbuf, ho, r0, rows, tid, y, xr, gc);
    else if (op.dim == 2) stencil_tile_d<NP, 2>(op, hbuf, ho, r0, rows, tid, y, xr, gc);
    else stencil_tile_d<NP, 1>(op, hbuf, ho, r0, rows, tid, y, xr, gc);
}

// dynamic shared memory of spmv_stream (bytes): halo (or ys for CSR), CSR x window, per-warp dot
// partials
__host__ __device__ inline size_t spmv_smem_bytes(int halo_cap, int tile, int nd, int wcap = 0, int ring = 0)
{
    const int h = halo_cap > 0 ? halo_cap : tile;
    return ((size_t)((h + 15) & ~15) + (size_t)((wcap + 15) & ~15) + (size_t)(ring ? XRING : 0) +
            (size_t)nd * SNW) * sizeof(double);
}

// ---------------------------------------------------------------------------------------------
// spmv_stream

// CM = 2: the banded uniform-row CSR path with the x ring only (its own instantiation: its register
// budget is not shared with the other CSR paths); CM = 0: every other path
template <class Op, int RPT, int CM = 0>
__global__ void __launch_bounds__(SNT, SMINB) spmv_stream_kernel(Op op, SpmvArgs a, Work wk)
{
    constexpr int TILE_ = SNT * RPT;
    constexpr int NP = RPT / 2;                           // double2 pairs per thread
    constexpr bool IS_ST = std::is_same<Op, StencilOp>::value;
    constexpr bool HALO = !std::is_same<Op, CsrOp>::value;
#ifndef PHIPM_CUD_CSR
#define PHIPM_CUD_CSR 4
#endif
    constexpr int CUD = std::is_same<Op, CsrOp>::value ? PHIPM_CUD_CSR : CU;
    extern __shared__ __align__(128) double sm[];
    __shared__ uint64_t hbar;
    __shared__ int hofs[2][5];                            // tile-relative halo offsets per parity
    __shared__ double bsum[MAXD + 2];
    __shared__ double wsum[SNW];
    __shared__ int s_exit;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = op.n;
    const int64_t cs = (int64_t)blockIdx.x * a.rpc, ce = min(n, cs + a.rpc);   // this CTA's rows
    int hcap = TILE_;
    if constexpr (IS_ST) hcap = halo_capacity(op.dim, op.nx, TILE_);
    int wcap = 0;
    if constexpr (!HALO) wcap = (op.wtile == TILE_) ? op.wcap : 0;
    int ring = 0;
    if constexpr (!HALO) ring = op.ring;
    double *hbuf = sm;                                    // halo (stencil/ident) or ys (CSR)
    double *xwin = sm + ((hcap + 15) & ~15);             // CSR x window (wcap doubles)
    double *xring = xwin + ((wcap + 15) & ~15);          // CSR x ring (XRING doubles)
    double *lacc = xring + (ring ? XRING : 0);
    __shared__ uint64_t rbar[2];                          // x ring: tile t's chunk on rbar[t & 1]
    __shared__ int64_t s_wstart[2];
    // CSR: TMA the x window of tile tl (its [tlo, thi] column range) if it fits
    auto issue_window = [&](int64_t wr0, int wrows, uint32_t par) {
        if constexpr (!HALO) {
            // union of the column ranges of the global wtile-row tiles covering [wr0, wr0 + wrows)
            int lo = 0x7fffffff, hi = -1;
            for (int64_t tl = wr0 / op.wtile; tl <= (wr0 + wrows - 1) / op.wtile; tl++) {
                if (op.thi[tl] >= 0) {
                    lo = min(lo, op.tlo[tl]);
                    hi = max(hi, op.thi[tl]);
                }
            }
            int64_t st = 0;
            uint32_t by = 0;
            if (hi >= lo && hi - lo + 4 <= wcap) seg_range(lo, (int64_t)hi + 1, a.ldx, st, by);
            s_wstart[par] = by ? st : -1;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive_expect_tx(&hbar, by);
            if (by) tma_load_1d(xwin, a.x + st, by, &hbar, policy_evict_last());
        }
    };
    // x ring: copy x[lo, hi) (clamped to [0, ldx), even bounds) into ring slots lo mod XRING ..,
    // split where the ring wraps; one mbarrier phase per call
    auto issue_ring = [&](int64_t lo, int64_t hi, uint64_t *bar) {
        int64_t st = 0;
        uint32_t by = 0;
        seg_range(lo, hi, a.ldx, st, by);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // prior generic reads of the ring
        mbar_arrive_expect_tx(bar, by);
        const uint64_t pol = policy_evict_last();
        int64_t c0 = st;
        uint32_t left = by;
        while (left) {
            const int slot = (int)(c0 & (XRING - 1));
            const uint32_t chunk = min(left, (uint32_t)(XRING - slot) * 8u);
            tma_load_1d(xring + slot, a.x + c0, chunk, bar, pol);
            c0 += chunk / 8;
            left -= chunk;
        }
    };
    auto plan = [&](int64_t r0, int rows, HaloPlan &h) {
        if constexpr (IS_ST) halo_plan(op, TILE_, r0, rows, a.ldx, h);
        else halo_plan_ident(r0, rows, a.ldx, h);
    };
    auto issue_halo = [&](int64_t hr0, int hrows, uint32_t par) {
        HaloPlan h;
        plan(hr0, hrows, h);
        // x[hr0 + q + d] of direction k is hbuf[hofs[k] + q + d] (centre, y-, y+, z-, z+)
        const int seg[5] = {0, h.ylo, h.yhi, h.zlo, h.zhi};
#pragma unroll
        for (int k = 0; k < 5; k++) hofs[par][k] = h.off[seg[k]] - (int)(h.start[seg[k]] - hr0);
        uint32_t tot = 0;
        for (int k = 0; k < h.nseg; k++) tot += h.bytes[k];
        const uint64_t pol = policy_evict_last();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // prior generic reads of hbuf
        mbar_arrive_expect_tx(&hbar, tot);
        for (int k = 0; k < h.nseg; k++)
            if (h.bytes[k]) tma_load_1d(hbuf + h.off[k], a.x + h.start[k], h.bytes[k], &hbar, pol);
    };
    KSTAMP(0)
    pdl_wait();
    KSTAMP(1)
    if (tid == 0) {
        s_exit = a.check_brk ? (wk.st->brk >= 0) : 0;
        if constexpr (HALO) {
            if (!s_exit) {
                mbar_init(&hbar, 1);
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
                if (cs < ce) issue_halo(cs, (int)min((int64_t)TILE_, ce - cs), 0);
            }
        } else {
            if (!s_exit && ring) {
                mbar_init(&rbar[0], 1);
                mbar_init(&rbar[1], 1);
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
                if (cs < ce) issue_ring(cs - op.blo, cs + TILE_ + op.bhi, &rbar[0]);   // first tile's window
            }
            if (!s_exit && wcap > 0) {
                mbar_init(&hbar, 1);
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
                if (cs < ce) issue_window(cs, (int)min((int64_t)TILE_, ce - cs), 0);
            }
        }
    }
    const double sc = a.xscale ? *a.xscale : 1.0;
    double zc[MAXZ];
#pragma unroll
    for (int i = 0; i < MAXZ; i++) zc[i] = (i < a.nz) ? a.zc[i] * (a.zcd[i] ? *a.zcd[i] : 1.0) : 0.0;
    for (int i = tid; i < a.nd * SNW; i += SNT) lacc[i] = 0.0;
    __syncthreads();
    if (s_exit) return;

    double ysq = 0.0, xsq = 0.0, amax = 0.0;
    uint32_t ht = 0;
    int3 gcoord = make_int3(0, 0, 0);                      // stencil: grid coordinates of row r0 + 2 tid
    if constexpr (IS_ST) gcoord = grid_coords(op, cs + 2 * tid);
    for (int64_t r0 = cs; r0 < ce; r0 += TILE_) {
        const int rows = (int)min((int64_t)TILE_, ce - r0);
        const int64_t r1 = r0 + TILE_;                     // next tile of this CTA
        if (a.pfc && tid == 0) {
            // this tile's epilogue vectors and first dot columns into L2 during the SpMV phase
            for (int i = 0; i < a.nz; i++) prefetch_rows(a.z[i] + r0, rows);
            for (int k = 0; k < min(CUD, a.nd); k++)
                if (k != (HALO ? a.xcol : -1)) prefetch_rows(a.V + (int64_t)(a.d0 + k) * a.ldv + r0, rows);
        }
        double2 y[NP], xr[NP];
        // ---- phase 1: raw (A x) rows into registers (and x itself, for a dot with v_j = x)
        if constexpr (HALO) {
            mbar_wait(&hbar, ht & 1);
            if (r0 == cs) KSTAMP(2)
            const int *ho = hofs[ht & 1];
            ht++;
            const double *pc = hbuf + ho[0];
            if constexpr (IS_ST) {
                stencil_tile<NP>(op, hbuf, ho, r0, rows, tid, y, xr, &gcoord);
            } else {
#pragma unroll
                for (int p = 0; p < NP; p++) {
                    const int q = 2 * tid + 2 * SNT * p;
                    xr[p].x = q < rows ? pc[q] : 0.0;
                    xr[p].y = q + 1 < rows ? pc[q + 1] : 0.0;
                    y[p] = xr[p];
                }
            }
            __syncthreads();                               // halo consumed
            if (tid == 0 && r1 < ce) issue_halo(r1, (int)min((int64_t)TILE_, ce - r1), ht & 1);
        } else {
#pragma unroll
            for (int p = 0; p < NP; p++) xr[p] = make_double2(0.0, 0.0);
            if constexpr (CM == 2) {
                // this tile needs x[r0 - blo, r0 + TILE + bhi): its new chunk was requested one tile
                // ago (or in the prologue).  Request the next tile's chunk, whose ring slots held
                // x[r0 - TILE - blo, r0 - blo) (previous tile only; its gathers are complete).  Two
                // barriers: the one re-armed here was last waited on a tile ago, and every thread
                // has passed that wait (tile-end barrier), so no waiter can miss a phase.
                mbar_wait(&rbar[ht & 1], (ht >> 1) & 1);
                if (tid == 0 && r1 < ce) issue_ring(r1 + op.bhi, r1 + TILE_ + op.bhi, &rbar[(ht + 1) & 1]);
                ht++;
                {
                    CsrOp opf = op;
                    opf.pf_end = ce;
#ifndef PHIPM_RING_PIPE
#define PHIPM_RING_PIPE 1
#endif
                    if (PHIPM_RING_PIPE > 0 && !op.off16)
                        csr_tile_ell_ring_pipe<(PHIPM_RING_PIPE > 0 ? PHIPM_RING_PIPE : 1)>(opf, xring, r0, rows, hbuf,
                                                                                          a.anorm ? &amax : nullptr);
                    else
                        csr_tile_ell<2>(opf, a.x, xring, 0, r0, rows, hbuf, a.anorm ? &amax : nullptr);
                }
                __syncthreads();                           // ring reads done, ys complete
            } else {
                if (wcap > 0) {
                    const uint32_t par = ht & 1;
                    ht++;
                    // the window decision is uniform per tile; read it once the copy has landed
                    mbar_wait(&hbar, par);
                    const int64_t ws = s_wstart[par];
                    auto nowait = [] {};
                    if (op.ell) {
                        if (ws >= 0) csr_tile_ell<1>(op, a.x, xwin, ws, r0, rows, hbuf);
                        else csr_tile_ell<0>(op, a.x, xwin, 0, r0, rows, hbuf);
                    } else if (ws >= 0) csr_tile<true>(op, a.x, xwin, ws, r0, rows, hbuf, nowait);
                    else csr_tile<false>(op, a.x, xwin, 0, r0, rows, hbuf, nowait);
                    __syncthreads();                           // window consumed, ys complete
                    if (tid == 0 && r1 < ce) issue_window(r1, (int)min((int64_t)TILE_, ce - r1), ht & 1);
                } else {
                    if (op.ell) csr_tile_ell<0>(op, a.x, xwin, 0, r0, rows, hbuf);
                    else csr_tile<false>(op, a.x, xwin, 0, r0, rows, hbuf, [] {});
                    __syncthreads();
                }
            }
#pragma unroll
            for (int p = 0; p < NP; p++) {
                const int q = 2 * tid + 2 * SNT * p;
                y[p] = q + 1 < rows ? *reinterpret_cast<const double2 *>(hbuf + q)
                                    : make_double2(q < rows ? hbuf[q] : 0.0, 0.0);
            }
            __syncthreads();                               // ys consumed
        }
        // ---- phase 2: scale + epilogue, store y, ||y||^2
#pragma unroll
        for (int p = 0; p < NP; p++) {
            const int q = 2 * tid + 2 * SNT * p;
            const int64_t r = r0 + q;
            y[p].x *= sc;
            y[p].y *= sc;
#pragma unroll
            for (int i = 0; i < MAXZ; i++)
                if (i < a.nz) {
                    if (q < rows) y[p].x = fma(zc[i], __ldg(a.z[i] + r), y[p].x);
                    if (q + 1 < rows) y[p].y = fma(zc[i], __ldg(a.z[i] + r + 1), y[p].y);
                }
            if (a.y) {
                if (q + 1 < rows) *reinterpret_cast<double2 *>(a.y + r) = y[p];
                else if (q < rows) a.y[r] = y[p].x;
            }
            ysq = fma(y[p].x, y[p].x, ysq);
            ysq = fma(y[p].y, y[p].y, ysq);
        }
        // ---- phase 3: d_k = V_k^T y over the tile, CUD columns in flight (CSR: 3, its row loop holds more
        //      registers; measured c5 +1 %, stencils keep 4); the column equal to x
        //      (if any) is not re-read: its dot comes from the x tile values kept in registers
        if (a.xnorm) {
            // ||x||^2 over the tile: x values in registers (halo operators) or this thread's own rows
#pragma unroll
            for (int p = 0; p < NP; p++) {
                const int q = 2 * tid + 2 * SNT * p;
                double2 xv = xr[p];
                if constexpr (!HALO)
                    xv = q + 1 < rows ? ld_stream2(a.x + r0 + q) : make_double2(q < rows ? a.x[r0 + q] : 0.0, 0.0);
                xsq = fma(xv.x, xv.x, xsq);
                xsq = fma(xv.y, xv.y, xsq);
            }
        }
        int xc = -1;
        if constexpr (HALO) xc = a.xcol;
        if (xc >= 0 && xc < a.nd) {
            double d = 0.0;
#pragma unroll
            for (int p = 0; p < NP; p++) {
                d = fma(xr[p].x, y[p].x, d);
                d = fma(xr[p].y, y[p].y, d);
            }
            d = warp_sum(d);
            if (lane == 0) lacc[xc * SNW + warp] += d;
        }
        for (int k0 = 0; k0 < a.nd; k0 += CUD) {
            if (a.pfc && tid == 0) {
                // the tile segments of the next CUD columns into L2 while these are loaded
                for (int k = k0 + CUD; k < min(k0 + 2 * CUD, a.nd); k++)
                    if (k != xc) prefetch_rows(a.V + (int64_t)(a.d0 + k) * a.ldv + r0, rows);
            }
            double2 v[CUD][NP];
#pragma unroll
            for (int u = 0; u < CUD; u++) {
                const int k = k0 + u;
                const bool ld = k < a.nd && k != xc;
                const double *vc = a.V + (int64_t)(a.d0 + (k < a.nd ? k : k0)) * a.ldv + r0;
#pragma unroll
                for (int p = 0; p < NP; p++) {
                    const int q = 2 * tid + 2 * SNT * p;
                    v[u][p] = (ld && q < rows) ? ld_stream2(vc + q) : make_double2(0.0, 0.0);
                }
            }
#pragma unroll
            for (int u = 0; u < CUD; u++) {
                double d = 0.0;
#pragma unroll
                for (int p = 0; p < NP; p++) {
                    d = fma(v[u][p].x, y[p].x, d);
                    d = fma(v[u][p].y, y[p].y, d);
                }
                d = warp_sum(d);
                if (lane == 0 && k0 + u < a.nd && k0 + u != xc) lacc[(k0 + u) * SNW + warp] += d;
            }
        }
    }
    // ---- block totals (fixed order), grid reduction, finalize
    KSTAMP(3)
    __syncthreads();
    for (int k = tid; k < a.nd; k += SNT) {
        double t = 0.0;
        for (int w = 0; w < SNW; w++) t += lacc[k * SNW + w];
        bsum[k] = t;
    }
    if (a.ynorm) {
        const double v = warp_sum(ysq);
        if (lane == 0) wsum[warp] = v;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < SNW; w++) t += wsum[w];
            bsum[a.nd] = t;
        }
    }
    if (a.xnorm) {
        __syncthreads();
        const double v = warp_sum(xsq);
        if (lane == 0) wsum[warp] = v;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < SNW; w++) t += wsum[w];
            bsum[a.nd + (a.ynorm ? 1 : 0)] = t;
        }
    }
    if (a.anorm) {
        // ||A||_inf: CTA max, then one atomicMax on the non-negative double's bits (before the ticket
        // of publish_partials, whose release covers it)
        double m = amax;
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        __syncthreads();
        if (lane == 0) wsum[warp] = m;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < SNW; w++) t = fmax(t, wsum[w]);
            atomicMax(&wk.st->anorm_bits, (unsigned long long)__double_as_longlong(t));
        }
    }
    const int nv = a.nd + (a.ynorm ? 1 : 0) + (a.xnorm ? 1 : 0);
    __syncthreads();
    if (nv == 0 && !a.anorm) return;                      // (||A||_inf: the last CTA publishes it)
    if (a.defer) {
        // deferred finalize: the update kernel that follows sums these (deferred_finalize); its
        // griddepcontrol.wait orders them (kernel completion), so no ticket and no fence here
        for (int v = tid; v < nv; v += SNT) wk.part2[(size_t)v * wk.pstride + blockIdx.x] = bsum[v];
        KSTAMP(4)
        return;
    }
    const bool last = publish_partials(wk, bsum, nv);
    KSTAMP(4)
    if (!last) return;
    __shared__ double red[MAXD + 2];
    final_reduce(wk, nv, red);
    KSTAMP(5)
    if (a.anorm && tid == 0) {
        const double na = __longlong_as_double((long long)__ldcg(&wk.st->anorm_bits));
        wk.st->bthr_d = (double)n * 2.220446049250313080847e-16 * na;
        // publish to the host (tau_0 of Eq. tau_0): the value, a system-scope fence, the sequence
        a.anorm_pub[0] = na;
        __threadfence_system();
        *a.anorm_seq = a.anorm_seqv;
    }
    finalize(a.fin, a.j, a.nd, red, wk, a.bthr, 0);
    KSTAMP(6)
}

// ---------------------------------------------------------------------------------------------
// axpy_stream

template <int RPT>
__global__ void __launch_bounds__(SNT, SMINB) axpy_stream_kernel(int64_t n, AxpyArgs a, Work wk)
{
    constexpr int TILE_ = SNT * RPT;
    constexpr int NP = RPT / 2;
    __shared__ double coef[MAXITEM];
    __shared__ const double *src[MAXITEM];
    __shared__ double bsum[2];
    __shared__ double wsum[SNW];
    __shared__ int s_exit;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ double dred[MAXD + 2];                    // deferred finalize: the SpMV's totals,
    __shared__ double dg[MAXD + 1];                      // the update coefficients g_k
    __shared__ double s_a0s;                             // and the base vector's factor
    KSTAMP(0)
    pdl_wait();
    KSTAMP(1)
    int nc_ = a.nc;
    if (a.guard) {                                         // (uniform: every CTA reads the same words)
        if (__ldcg(a.guard) != a.guard_val) return;
        nc_ = __ldcg(a.guard + 1);
    }
    if (tid == 0) s_exit = a.check_brk ? (wk.st->brk >= 0) : 0;
    if (a.dfin) {
        // the preceding SpMV left its partials in wk.part2 (SpmvArgs.defer): reduce and finalize here
        __syncthreads();
        if (s_exit) return;                               // (that SpMV exited too: no partials)
        if (!deferred_finalize(a, wk, dred, dg, &s_a0s)) return;   // breakdown (FIN_ARNOLDI_LAG)
    }
    const int nbase = (a.a0h != 0.0) ? 1 : 0;
    const int nitem = nbase + nc_ + a.ne;
    for (int k = tid; k < nitem; k += SNT) {
        double c;
        const double *p;
        if (k < nbase) {
            c = a.a0h * (a.dfin == FIN_ARNOLDI_LAG ? s_a0s : (a.a0d ? *a.a0d : 1.0));   // (lag: a0d = &sigma_j)
            p = a.base;
        } else if (k < nbase + nc_) {
            const int kc = a.rev ? (nc_ - 1 - (k - nbase)) : (k - nbase);
            c = a.gsign * (a.dfin ? dg[kc] : a.g[kc]);
            p = a.V + (int64_t)(a.c0 + kc) * a.ldv;
        } else {
            const int i = k - nbase - nc_;
            c = a.ec[i] * (a.ecd ? a.ecd[i] : 1.0);
            p = a.e[i];
        }
        coef[k] = c;
        src[k] = p;
    }
    __syncthreads();
    if (s_exit) return;
    const int64_t cs = (int64_t)blockIdx.x * a.rpc, ce = min(n, cs + a.rpc);   // this CTA's rows
    double nrm = 0.0;
    for (int64_t r0 = cs; r0 < ce; r0 += TILE_) {
        const int rows = (int)min((int64_t)TILE_, ce - r0);
        double2 acc[NP];
#pragma unroll
        for (int p = 0; p < NP; p++) acc[p] = make_double2(0.0, 0.0);
        for (int k0 = 0; k0 < nitem; k0 += CU) {
            if (a.pfc && tid == 0) {
                // next group of this tile, or the first group of the next tile
                for (int k = k0 + CU; k < k0 + 2 * CU; k++) {
                    if (k < nitem) prefetch_rows(src[k] + r0, rows);
                    else if (r0 + TILE_ < ce && k - nitem < CU && k - nitem < nitem)
                        prefetch_rows(src[k - nitem] + r0 + TILE_, (int)min((int64_t)TILE_, ce - r0 - TILE_));
                }
                if (k0 == 0 && r0 == cs)
                    for (int k = 0; k < min(CU, nitem); k++) prefetch_rows(src[k] + r0, rows);
            }
            double2 v[CU][NP];
#pragma unroll
            for (int u = 0; u < CU; u++) {
                const int k = k0 + u;
                const double *sp = src[k < nitem ? k : k0] + r0;
#pragma unroll
                for (int p = 0; p < NP; p++) {
                    const int q = 2 * tid + 2 * SNT * p;
                    v[u][p] = (k < nitem && q < rows) ? ld_stream2(sp + q) : make_double2(0.0, 0.0);
                }
            }
#pragma unroll
            for (int u = 0; u < CU; u++) {
                const double c = (k0 + u < nitem) ? coef[k0 + u] : 0.0;
#pragma unroll
                for (int p = 0; p < NP; p++) {
                    acc[p].x = fma(c, v[u][p].x, acc[p].x);
                    acc[p].y = fma(c, v[u][p].y, acc[p].y);
                }
            }
        }
#pragma unroll
        for (int p = 0; p < NP; p++) {
            const int q = 2 * tid + 2 * SNT * p;
            double *o = a.out + r0 + q;
            if (q + 1 < rows) *reinterpret_cast<double2 *>(o) = acc[p];
            else if (q < rows) o[0] = acc[p].x;
            if (q < rows) nrm = fma(acc[p].x, acc[p].x, nrm);
            if (q + 1 < rows) nrm = fma(acc[p].y, acc[p].y, nrm);
        }
    }
    KSTAMP(3)
    if (!a.onorm) return;
    const double v = warp_sum(nrm);
    if (lane == 0) wsum[warp] = v;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < SNW; w++) t += wsum[w];
        bsum[0] = t;
    }
    __syncthreads();
    const bool last = publish_partials(wk, bsum, 1);
    KSTAMP(4)
    if (!last) return;
    __shared__ double red[2];
    final_reduce(wk, 1, red);
    KSTAMP(5)
    finalize(a.fin, a.j, 1, red, wk, a.bthr, a.lanczos);
    KSTAMP(6)
}

} // namespace phipm
