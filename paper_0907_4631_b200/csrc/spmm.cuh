// spmm.cuh — the shared-operator block product of the block phipm solve:
//
//   Y_b = A X_b,  b = 0 .. nb-1     (nb <= SPMM_MAXB right-hand sides sharing the CSR matrix A)
//
// PAPER.md §2 (Eq. lincomb) motivates many phipm evaluations with one operator (the stages
// of an exponential integrator), and §5 the use inside such integrators.  For a CSR
// operator the val/col streams (12 B per nonzero) dominate an SpMV's traffic; here they are read
// once per block step for all nb vectors (SpMM shape: nb gathers and FMAs per loaded entry).
//
// Layout: one contiguous row range per CTA (rpc rows).  Uniform-row-length matrices (ell > 0,
// ell % 4 == 0) take the vectorised path of the streaming SpMV: ell/4 lanes per row, 4 entries per
// lane as int4 + 2 x double2 loads, val/col prefetched into L2 by the TMA engine `pf` rows ahead;
// x gathers go through L1 (__ldg: the band of a row block is re-read by its neighbours).  Other
// matrices: 2^glog lanes per row, entries strided over the lanes.  Per row and vector the products
// are summed per lane in entry order, then over the lanes by a shuffle tree.
#pragma once

#include "stream.cuh"

namespace phipm {

constexpr int SPMM_MAXB = 8;
constexpr int SPMM_NT = 512;

struct SpmmArgs {
    int nb;
    const double *x[SPMM_MAXB];
    double *y[SPMM_MAXB];
    int64_t rpc;               // rows per CTA
    const int *brk[SPMM_MAXB]; // optional: the problem's breakdown position (DevState::brk); >= 0 = skip
};

template <int NBT>
__device__ __forceinline__ void spmm_rows_ell(const CsrOp &A, const SpmmArgs &a, int64_t cs, int64_t ce,
                                              const bool *act)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = SPMM_NT / 32;
    const int G = A.ell >> 2, rpw = 32 / G;
    const int sub = lane / G, li = lane - sub * G;
    for (int64_t r = cs + (int64_t)warp * rpw + sub, blk = cs; blk < ce; blk += (int64_t)NW * rpw, r += (int64_t)NW * rpw) {
        if (A.pf > 0 && threadIdx.x == 0) {
            const int64_t pa = blk + A.pf, pb = min(pa + (int64_t)NW * rpw, ce);
            if (pb > pa) {
                tma_prefetch_l2(A.val + pa * A.ell, (uint32_t)((pb - pa) * A.ell * 8));
                tma_prefetch_l2(A.col + pa * A.ell, (uint32_t)((pb - pa) * A.ell * 4));
            }
        }
        const bool ok = r < ce;
        int4 cc = make_int4(0, 0, 0, 0);
        double2 va = make_double2(0.0, 0.0), vb = va;
        if (ok) {
            const int64_t e = r * (int64_t)A.ell + 4 * li;
            cc = __ldg(reinterpret_cast<const int4 *>(A.col + e));
            va = ldg_stream2(A.val + e);
            vb = ldg_stream2(A.val + e + 2);
        }
#pragma unroll
        for (int b = 0; b < NBT; b++) {
            if (b >= a.nb) break;
            double t = 0.0;
            if (ok && act[b]) {
                const double *x = a.x[b];
                t = va.x * __ldg(x + cc.x);
                t = fma(va.y, __ldg(x + cc.y), t);
                t = fma(vb.x, __ldg(x + cc.z), t);
                t = fma(vb.y, __ldg(x + cc.w), t);
            }
            for (int o = G >> 1; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (ok && li == 0 && act[b]) a.y[b][r] = t;
        }
    }
}

__device__ __forceinline__ void spmm_rows_gen(const CsrOp &A, const SpmmArgs &a, int64_t cs, int64_t ce,
                                              const bool *act)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = SPMM_NT / 32;
    const int G = 1 << A.glog, rpw = 32 / G;
    const int sub = lane / G, li = lane - sub * G;
    for (int64_t r = cs + (int64_t)warp * rpw + sub, blk = cs; blk < ce; blk += (int64_t)NW * rpw, r += (int64_t)NW * rpw) {
        const bool ok = r < ce;
        const int e0 = ok ? A.rp[r] : 0, e1 = ok ? A.rp[r + 1] : 0;
        double t[SPMM_MAXB];
#pragma unroll
        for (int b = 0; b < SPMM_MAXB; b++) t[b] = 0.0;
        for (int e = e0 + li; e < e1; e += G) {
            const double v = A.val[e];
            const int cidx = A.col[e];
#pragma unroll
            for (int b = 0; b < SPMM_MAXB; b++)
                if (b < a.nb && act[b]) t[b] = fma(v, __ldg(a.x[b] + cidx), t[b]);
        }
#pragma unroll
        for (int b = 0; b < SPMM_MAXB; b++) {
            if (b >= a.nb) break;
            double s = t[b];
            for (int o = G >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (ok && li == 0 && act[b]) a.y[b][r] = s;
        }
    }
}

__global__ void __launch_bounds__(SPMM_NT) spmm_csr_kernel(CsrOp A, SpmmArgs a)
{
    pdl_wait();
    bool act[SPMM_MAXB];
#pragma unroll
    for (int b = 0; b < SPMM_MAXB; b++) act[b] = b < a.nb && !(a.brk[b] && *a.brk[b] >= 0);
    const int64_t cs = (int64_t)blockIdx.x * a.rpc, ce = min(A.n, cs + a.rpc);
    if (A.ell > 0) {
        if (a.nb <= 2) spmm_rows_ell<2>(A, a, cs, ce, act);
        else if (a.nb <= 4) spmm_rows_ell<4>(A, a, cs, ce, act);
        else spmm_rows_ell<SPMM_MAXB>(A, a, cs, ce, act);
    } else {
        spmm_rows_gen(A, a, cs, ce, act);
    }
}

// ---------------------------------------------------------------------------------------------
// Banded uniform-row CSR: each vector's x lives in a shared-memory ring of R = 2 T + blo + bhi doubles
// (T rows per tile) that slides with the CTA's row range, as in the streaming SpMV's x ring
// (stream.cuh): the first tile's window [r0 - blo, r0 + T + bhi) in the prologue, then every tile
// requests the next tile's new T-row chunk, whose slots held the previous tile's lower window.  The
// gathers become shared-memory loads; x is read about once per vector.  nb R doubles must fit.

struct SpmmRing {
    int T, R;                  // tile rows, ring length (doubles, multiple of 32)
    int64_t ldx;               // x vectors are readable up to ldx (workspace columns)
};

template <int NBT>
__global__ void __launch_bounds__(SNT, 1) spmm_csr_ring_kernel(CsrOp A, SpmmArgs a, SpmmRing g)
{
    extern __shared__ __align__(128) double rs[];          // nb rings of R doubles
    __shared__ uint64_t rbar[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t cs = (int64_t)blockIdx.x * a.rpc, ce = min(A.n, cs + a.rpc);
    const int T = g.T, R = g.R;
    bool act[SPMM_MAXB];
#pragma unroll
    for (int b = 0; b < SPMM_MAXB; b++) act[b] = false;
    // copy x_b[lo, hi) (clamped, even bounds) into ring b slots lo mod R .., split where the ring wraps
    auto issue = [&](int64_t lo, int64_t hi, uint64_t *bar) {
        int64_t st = 0;
        uint32_t by = 0;
        seg_range(lo, hi, g.ldx, st, by);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        int na = 0;
        for (int b = 0; b < a.nb; b++) na += act[b];
        mbar_arrive_expect_tx(bar, by * (uint32_t)na);
        const uint64_t pol = policy_evict_last();
        for (int b = 0; b < a.nb; b++) {
            if (!act[b]) continue;
            int64_t c0 = st;
            uint32_t left = by;
            while (left) {
                const int slot = (int)(c0 % R);
                const uint32_t chunk = min(left, (uint32_t)(R - slot) * 8u);
                tma_load_1d(rs + (size_t)b * R + slot, a.x[b] + c0, chunk, bar, pol);
                c0 += chunk / 8;
                left -= chunk;
            }
        }
    };
    pdl_wait();
#pragma unroll
    for (int b = 0; b < SPMM_MAXB; b++) act[b] = b < a.nb && !(a.brk[b] && *a.brk[b] >= 0);
    if (tid == 0 && cs < ce) {
        mbar_init(&rbar[0], 1);
        mbar_init(&rbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        issue(cs - A.blo, cs + T + A.bhi, &rbar[0]);
    }
    __syncthreads();
    const int G = A.ell >> 2, rpw = 32 / G;
    const int sub = lane / G, li = lane - sub * G;
    uint32_t ht = 0;
    for (int64_t r0 = cs; r0 < ce; r0 += T) {
        const int rows = (int)min((int64_t)T, ce - r0);
        const int64_t r1 = r0 + T;
        mbar_wait(&rbar[ht & 1], (ht >> 1) & 1);
        if (tid == 0 && r1 < ce) issue(r1 + A.bhi, r1 + T + A.bhi, &rbar[(ht + 1) & 1]);
        ht++;
        // slot of column c: c - base, minus R if >= R (every column of the tile is in [r0 - blo, r0 + T + bhi))
        const int64_t lo = max((int64_t)0, r0 - A.blo);
        const int64_t base = lo - lo % R;
        for (int q0 = warp * rpw; q0 < rows; q0 += SNW * rpw) {
            if (A.pf > 0 && tid == 0) {
                const int64_t pa = r0 + q0 + A.pf, pb = min(pa + (int64_t)SNW * rpw, ce);
                if (pb > pa) {
                    tma_prefetch_l2(A.val + pa * A.ell, (uint32_t)((pb - pa) * A.ell * 8));
                    tma_prefetch_l2(A.col + pa * A.ell, (uint32_t)((pb - pa) * A.ell * 4));
                }
            }
            const int q = q0 + sub;
            const bool ok = q < rows;
            int4 cc = make_int4(0, 0, 0, 0);
            double2 va = make_double2(0.0, 0.0), vb = va;
            if (ok) {
                const int64_t e = (r0 + q) * (int64_t)A.ell + 4 * li;
                cc = __ldg(reinterpret_cast<const int4 *>(A.col + e));
                va = ldg_stream2(A.val + e);
                vb = ldg_stream2(A.val + e + 2);
            }
            int sl[4] = {(int)(cc.x - base), (int)(cc.y - base), (int)(cc.z - base), (int)(cc.w - base)};
#pragma unroll
            for (int i = 0; i < 4; i++) sl[i] -= sl[i] >= R ? R : 0;
#pragma unroll
            for (int b = 0; b < NBT; b++) {
                if (b >= a.nb) break;
                double t = 0.0;
                if (ok && act[b]) {
                    const double *x = rs + (size_t)b * R;
                    t = va.x * x[sl[0]];
                    t = fma(va.y, x[sl[1]], t);
                    t = fma(vb.x, x[sl[2]], t);
                    t = fma(vb.y, x[sl[3]], t);
                }
                for (int o = G >> 1; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
                if (ok && li == 0 && act[b]) a.y[b][r0 + q] = t;
            }
        }
        __syncthreads();                                  // ring reads of this tile done
    }
}

} // namespace phipm
