// stream.cuh — the two n-sized kernels of a phipm step, B200 style: persistent (one CTA per SM),
// one producer warp issuing 1-D TMA bulk copies (cp.async.bulk, SASS UBLKCP) of 8 KB vector
// segments into an mbarrier ring in shared memory, sixteen consumer warps doing the fp64 arithmetic
// from shared memory.  Stencil operators get their halo tiles (centre row range plus the +-nx and
// +-nx*ny neighbour ranges) the same way, double-buffered, so x is read from L2/HBM once per tile
// range rather than through per-thread gathers.
//
//   spmv_stream   y = s (A x) + sum_i c_i z_i ; d_k = v~_k^T y (k in a column range) ; ||y||^2
//   axpy_stream   out = sum over streamed sources (a0 base, -g_k v~_k or +c_k v~_k, e_i E_i) ; ||out||^2
//
// Both end in the deterministic last-block grid reduction + finalize of kernels.cuh.
// All TMA sources are workspace vectors padded to ldv (a multiple of 32 doubles), so every
// segment can be rounded out to 16-byte boundaries without leaving the allocation.
#pragma once

#include "kernels.cuh"

namespace phipm {

constexpr int NCW = 16;                 // consumer warps
constexpr int NCT = NCW * 32;           // consumer threads
constexpr int NTHR = NCT + 32;          // + producer warp
constexpr int MAXRING = 28;             // ring slots (TILE doubles = 8 KB each); runtime count fills smem
constexpr int HSEG = TILE + 8;          // halo segment capacity in doubles (alignment slack)
constexpr int MAXITEM = MAXD + MAXZ + 2;
static_assert(TILE == 2 * NCT, "2 rows (one double2) per consumer thread per slot");

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

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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

__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
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

__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(NCT) : "memory"); }

struct Pipe {
    uint64_t full[MAXRING], empty[MAXRING];
    uint64_t hfull[2], hempty[2];
};

__device__ __forceinline__ void pipe_init(Pipe &pp, int nring)
{
    for (int s = 0; s < nring; s++) {
        mbar_init(&pp.full[s], 1);
        mbar_init(&pp.empty[s], NCW);
    }
    for (int s = 0; s < 2; s++) {
        mbar_init(&pp.hfull[s], 1);
        mbar_init(&pp.hempty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// ---------------------------------------------------------------------------------------------
// halo plan: the x ranges a tile of stencil rows reads (centre [r0-1, r0+rows+1), y-/y+ ranges
// [r0 -+ nx, ... + rows), z-/z+ ranges [r0 -+ nx*ny, ... + rows)), rounded out to even indices
// and clamped to [0, ldv).

struct HaloPlan {
    int64_t start[5];
    uint32_t bytes[5];
};

template <class Op>
__device__ __forceinline__ int halo_nseg(const Op &) { return 0; }
template <>
__device__ __forceinline__ int halo_nseg<StencilOp>(const StencilOp &S) { return S.dim == 1 ? 1 : (S.dim == 2 ? 3 : 5); }
template <>
__device__ __forceinline__ int halo_nseg<IdentOp>(const IdentOp &) { return 1; }

__device__ __forceinline__ void seg_range(int64_t lo, int64_t hi, int64_t ldv, int64_t &start, uint32_t &bytes)
{
    lo = lo < 0 ? 0 : (lo & ~(int64_t)1);
    hi = hi > ldv ? ldv : ((hi + 1) & ~(int64_t)1);
    if (hi <= lo) { start = lo; bytes = 0; return; }
    start = lo;
    bytes = (uint32_t)((hi - lo) * 8);
}

__device__ __forceinline__ void halo_plan(const StencilOp &S, int64_t r0, int rows, int64_t ldv, HaloPlan &h)
{
    seg_range(r0 - 1, r0 + rows + 1, ldv, h.start[0], h.bytes[0]);
    if (S.dim >= 2) {
        seg_range(r0 - S.nx, r0 - S.nx + rows, ldv, h.start[1], h.bytes[1]);
        seg_range(r0 + S.nx, r0 + S.nx + rows, ldv, h.start[2], h.bytes[2]);
    }
    if (S.dim >= 3) {
        const int64_t pl = (int64_t)S.nx * S.ny;
        seg_range(r0 - pl, r0 - pl + rows, ldv, h.start[3], h.bytes[3]);
        seg_range(r0 + pl, r0 + pl + rows, ldv, h.start[4], h.bytes[4]);
    }
}

__device__ __forceinline__ void halo_plan(const IdentOp &, int64_t r0, int rows, int64_t ldv, HaloPlan &h)
{
    seg_range(r0, r0 + rows, ldv, h.start[0], h.bytes[0]);
}

__device__ __forceinline__ void halo_plan(const CsrOp &, int64_t, int, int64_t, HaloPlan &) {}

// Stencil row from the halo tile, summed in ascending column order with separately rounded
// products (no FMA): the same operations, in the same order, as a sequential CSR row sum, so y
// is bit-exact with it.
__device__ __forceinline__ double stencil_row_halo(const StencilOp &S, const double *hb, const HaloPlan &h, int64_t r)
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
    const double *c0 = hb + (r - h.start[0]);
    double s = 0.0;
    if (S.dim >= 3 && kk > 0) s = __dadd_rn(s, __dmul_rn(S.c[5], hb[3 * HSEG + (r - pl - h.start[3])]));
    if (S.dim >= 2 && jj > 0) s = __dadd_rn(s, __dmul_rn(S.c[3], hb[1 * HSEG + (r - S.nx - h.start[1])]));
    if (i > 0) s = __dadd_rn(s, __dmul_rn(S.c[1], c0[-1]));
    s = __dadd_rn(s, __dmul_rn(S.c[0], c0[0]));
    if (i < S.nx - 1) s = __dadd_rn(s, __dmul_rn(S.c[2], c0[1]));
    if (S.dim >= 2 && jj < S.ny - 1) s = __dadd_rn(s, __dmul_rn(S.c[4], hb[2 * HSEG + (r + S.nx - h.start[2])]));
    if (S.dim >= 3 && kk < S.nz - 1) s = __dadd_rn(s, __dmul_rn(S.c[6], hb[4 * HSEG + (r + pl - h.start[4])]));
    return s;
}

// CSR rows of a tile: G = 2^glog lanes per row, U row groups in flight per lane (memory-level
// parallelism for the col -> x gather chain), rows longer than G strided, shuffle reduction.
__device__ __forceinline__ void csr_tile(const CsrOp &A, const double *__restrict__ x, int64_t r0, int rows, double *ys,
                                         int ctid)
{
    constexpr int U = 8;
    const int lane = ctid & 31, warp = ctid >> 5;
    const int G = 1 << A.glog;
    const int rpw = 32 >> A.glog;
    const int sub = lane >> A.glog, li = lane & (G - 1);
    const int stride = NCW * rpw;
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
#pragma unroll
        for (int u = 0; u < U; u++) acc[u] = (e[u] < e1[u]) ? vv[u] * __ldg(x + cc[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < U; u++)
            for (int f = e[u] + G; f < e1[u]; f += G) acc[u] = fma(ldg_stream(A.val + f), __ldg(x + __ldg(A.col + f)), acc[u]);
#pragma unroll
        for (int u = 0; u < U; u++) {
            for (int o = G >> 1; o > 0; o >>= 1) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
            if (q[u] < rows && li == 0) ys[q[u]] = acc[u];
        }
    }
}

template <class Op>
__device__ __forceinline__ constexpr bool has_halo() { return true; }
template <>
__device__ __forceinline__ constexpr bool has_halo<CsrOp>() { return false; }

__device__ __forceinline__ uint32_t seg_bytes(int rows) { return (uint32_t)(((rows + 1) & ~1) * 8); }

// dynamic shared memory layout (doubles): halo (2 x nseg x HSEG) | ys | lacc | ring (nring x TILE)
__host__ __device__ inline size_t stream_fixed_doubles(int nseg, bool spmv)
{
    return (size_t)2 * nseg * HSEG + (spmv ? (size_t)TILE + (size_t)MAXD * NCW : 0);
}

// as many ring slots as fit in `budget` bytes of dynamic shared memory (>= 2)
__host__ __device__ inline int stream_nring(int nseg, bool spmv, size_t budget)
{
    const size_t fixed = stream_fixed_doubles(nseg, spmv) * sizeof(double);
    long r = budget > fixed ? (long)((budget - fixed) / (TILE * sizeof(double))) : 0;
    if (r > MAXRING) r = MAXRING;
    if (r < 2) r = 2;
    return (int)r;
}

__host__ __device__ inline size_t stream_smem_bytes(int nseg, bool spmv, int nring)
{
    return (stream_fixed_doubles(nseg, spmv) + (size_t)nring * TILE) * sizeof(double);
}

// ---------------------------------------------------------------------------------------------

template <class Op>
__global__ void __launch_bounds__(NTHR, 1) spmv_stream_kernel(Op op, SpmvArgs a, Work wk, int nring)
{
    extern __shared__ __align__(128) double sm[];
    __shared__ Pipe pp;
    __shared__ double bsum[MAXD + 2];
    __shared__ double wsum[NCW];
    __shared__ int s_exit;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        s_exit = a.check_brk ? (wk.st->brk >= 0) : 0;
        pipe_init(pp, nring);
    }
    __syncthreads();
    if (s_exit) return;
    const int nseg = halo_nseg(op);
    double *halo = sm;
    double *ys = halo + 2 * nseg * HSEG;
    double *lacc = ys + TILE;
    double *ring = lacc + MAXD * NCW;
    const int64_t n = op.n;
    const int64_t ntiles = (n + TILE - 1) / TILE;
    constexpr bool HALO = has_halo<Op>();

    if (warp == NCW) {
        // ------------------------------------------------------------------ producer
        if (lane == 0) {
            const uint64_t pol_v = policy_evict_first();
            const uint64_t pol_x = policy_evict_last();
            uint32_t it = 0, ht = 0;
            auto issue_halo = [&](int64_t tl) {
                const int64_t hr0 = tl * TILE;
                const int hrows = (int)min((int64_t)TILE, n - hr0);
                const int hb = ht & 1;
                if (ht >= 2) mbar_wait(&pp.hempty[hb], ((ht >> 1) - 1) & 1);
                HaloPlan h;
                halo_plan(op, hr0, hrows, a.ldx, h);
                uint32_t tot = 0;
                for (int k = 0; k < nseg; k++) tot += h.bytes[k];
                mbar_arrive_expect_tx(&pp.hfull[hb], tot);
                for (int k = 0; k < nseg; k++)
                    if (h.bytes[k])
                        tma_load_1d(halo + (hb * nseg + k) * HSEG, a.x + h.start[k], h.bytes[k], &pp.hfull[hb], pol_x);
                ht++;
            };
            if (HALO && (int64_t)blockIdx.x < ntiles) issue_halo(blockIdx.x);
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const int64_t r0 = tile * TILE;
                const int rows = (int)min((int64_t)TILE, n - r0);
                // prefetch the next tile's halo before this tile's column segments (double buffer)
                if (HALO && tile + gridDim.x < ntiles) issue_halo(tile + gridDim.x);
                const uint32_t by = seg_bytes(rows);
                for (int k = 0; k < a.nd; k++) {
                    const int s = it % nring;
                    const uint32_t r = it / nring;
                    if (r >= 1) mbar_wait(&pp.empty[s], (r - 1) & 1);
                    mbar_arrive_expect_tx(&pp.full[s], by);
                    tma_load_1d(ring + s * TILE, a.V + (int64_t)(a.d0 + k) * a.ldv + r0, by, &pp.full[s], pol_v);
                    it++;
                }
            }
        }
    } else {
        // ------------------------------------------------------------------ consumers
        const double sc = a.xscale ? *a.xscale : 1.0;
        double zc[MAXZ];
#pragma unroll
        for (int i = 0; i < MAXZ; i++) zc[i] = (i < a.nz) ? a.zc[i] * (a.zcd[i] ? *a.zcd[i] : 1.0) : 0.0;
        for (int i = tid; i < a.nd * NCW; i += NCT) lacc[i] = 0.0;
        double ysq = 0.0;
        uint32_t it = 0, ht = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int64_t r0 = tile * TILE;
            const int rows = (int)min((int64_t)TILE, n - r0);
            // phase 1+2: y rows into ys (and global)
            if constexpr (HALO) {
                const int hb = ht & 1;
                mbar_wait(&pp.hfull[hb], (ht >> 1) & 1);
                HaloPlan h;
                halo_plan(op, r0, rows, a.ldx, h);
                const double *hbuf = halo + hb * nseg * HSEG;
                for (int q = tid; q < rows; q += NCT) {
                    const int64_t r = r0 + q;
                    double y;
                    if constexpr (std::is_same<Op, StencilOp>::value) y = stencil_row_halo(op, hbuf, h, r);
                    else y = hbuf[r - h.start[0]];
                    y = sc * y;
#pragma unroll
                    for (int i = 0; i < MAXZ; i++)
                        if (i < a.nz) y = fma(zc[i], __ldg(a.z[i] + r), y);
                    ys[q] = y;
                    if (a.y) a.y[r] = y;
                    ysq = fma(y, y, ysq);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&pp.hempty[hb]);
                ht++;
            } else {
                csr_tile(op, a.x, r0, rows, ys, tid);
                consumer_sync();
                for (int q = tid; q < rows; q += NCT) {
                    const int64_t r = r0 + q;
                    double y = sc * ys[q];
#pragma unroll
                    for (int i = 0; i < MAXZ; i++)
                        if (i < a.nz) y = fma(zc[i], __ldg(a.z[i] + r), y);
                    ys[q] = y;
                    if (a.y) a.y[r] = y;
                    ysq = fma(y, y, ysq);
                }
            }
            consumer_sync();
            // phase 3: dot products of the tile with the streamed V column segments
            if (a.nd > 0) {
                const int qa = warp * 64 + 2 * lane;
                const double2 ya = *reinterpret_cast<const double2 *>(ys + qa);
                for (int k = 0; k < a.nd; k++) {
                    const int s = it % nring;
                    mbar_wait(&pp.full[s], (it / nring) & 1);
                    const double2 va = *reinterpret_cast<const double2 *>(ring + s * TILE + qa);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&pp.empty[s]);
                    double d = 0.0;
                    if (qa < rows) d = va.x * ya.x;
                    if (qa + 1 < rows) d = fma(va.y, ya.y, d);
                    d = warp_sum(d);
                    if (lane == 0) lacc[k * NCW + warp] += d;
                    it++;
                }
            }
            consumer_sync();
        }
        // block totals (fixed order)
        for (int k = tid; k < a.nd; k += NCT) {
            double t = 0.0;
            for (int w = 0; w < NCW; w++) t += lacc[k * NCW + w];
            bsum[k] = t;
        }
        if (a.ynorm) {
            const double v = warp_sum(ysq);
            if (lane == 0) wsum[warp] = v;
            consumer_sync();
            if (tid == 0) {
                double t = 0.0;
                for (int w = 0; w < NCW; w++) t += wsum[w];
                bsum[a.nd] = t;
            }
        }
    }
    const int nv = a.nd + (a.ynorm ? 1 : 0);
    __syncthreads();
    if (nv == 0) return;
    if (!publish_partials(wk, bsum, nv)) return;
    __shared__ double red[MAXD + 2];
    final_reduce(wk, nv, red);
    finalize(a.fin, a.j, a.nd, red, wk, 0.0, 0);
}

// ---------------------------------------------------------------------------------------------

struct AxpySrc {
    int nitem;
};

__device__ __forceinline__ const double *axpy_item(const AxpyArgs &a, int k)
{
    // item order: [base], V columns c0.., extras
    if (a.a0h != 0.0) {
        if (k == 0) return a.base;
        k--;
    }
    if (k < a.nc) return a.V + (int64_t)(a.c0 + k) * a.ldv;
    return a.e[k - a.nc];
}

__global__ void __launch_bounds__(NTHR, 1) axpy_stream_kernel(int64_t n, AxpyArgs a, Work wk, int nring)
{
    extern __shared__ __align__(128) double sm[];
    __shared__ Pipe pp;
    __shared__ double coef[MAXITEM];
    __shared__ double bsum[2];
    __shared__ double wsum[NCW];
    __shared__ int s_exit;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        s_exit = a.check_brk ? (wk.st->brk >= 0) : 0;
        pipe_init(pp, nring);
    }
    const int nbase = (a.a0h != 0.0) ? 1 : 0;
    const int nitem = nbase + a.nc + a.ne;
    for (int k = tid; k < nitem; k += NTHR) {
        double c;
        if (k < nbase) c = a.a0h * (a.a0d ? *a.a0d : 1.0);
        else if (k < nbase + a.nc) c = a.gsign * a.g[k - nbase];
        else c = a.ec[k - nbase - a.nc] * (a.ecd ? a.ecd[k - nbase - a.nc] : 1.0);
        coef[k] = c;
    }
    __syncthreads();
    if (s_exit) return;
    double *ring = sm;
    const int64_t ntiles = (n + TILE - 1) / TILE;
    double nrm = 0.0;
    if (warp == NCW) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            uint32_t it = 0;
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const int64_t r0 = tile * TILE;
                const int rows = (int)min((int64_t)TILE, n - r0);
                const uint32_t by = seg_bytes(rows);
                for (int k = 0; k < nitem; k++) {
                    const int s = it % nring;
                    const uint32_t r = it / nring;
                    if (r >= 1) mbar_wait(&pp.empty[s], (r - 1) & 1);
                    mbar_arrive_expect_tx(&pp.full[s], by);
                    tma_load_1d(ring + s * TILE, axpy_item(a, k) + r0, by, &pp.full[s], pol);
                    it++;
                }
            }
        }
    } else {
        uint32_t it = 0;
        const int qa = 2 * tid;                               // rows qa, qa+1 of the tile
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int64_t r0 = tile * TILE;
            const int rows = (int)min((int64_t)TILE, n - r0);
            double2 A = make_double2(0.0, 0.0);
            for (int k = 0; k < nitem; k++) {
                const int s = it % nring;
                mbar_wait(&pp.full[s], (it / nring) & 1);
                const double2 va = *reinterpret_cast<const double2 *>(ring + s * TILE + qa);
                __syncwarp();
                if (lane == 0) mbar_arrive(&pp.empty[s]);
                const double c = coef[k];
                A.x = fma(c, va.x, A.x);
                A.y = fma(c, va.y, A.y);
                it++;
            }
            double *o = a.out + r0;
            if (qa + 1 < rows) *reinterpret_cast<double2 *>(o + qa) = A;
            else if (qa < rows) o[qa] = A.x;
            if (qa < rows) nrm = fma(A.x, A.x, nrm);
            if (qa + 1 < rows) nrm = fma(A.y, A.y, nrm);
        }
        if (a.onorm) {
            const double v = warp_sum(nrm);
            if (lane == 0) wsum[warp] = v;
            consumer_sync();
            if (tid == 0) {
                double t = 0.0;
                for (int w = 0; w < NCW; w++) t += wsum[w];
                bsum[0] = t;
            }
        }
    }
    __syncthreads();
    if (!a.onorm) return;
    if (!publish_partials(wk, bsum, 1)) return;
    __shared__ double red[2];
    final_reduce(wk, 1, red);
    finalize(a.fin, a.j, 1, red, wk, a.bthr, a.lanczos);
}

} // namespace phipm
