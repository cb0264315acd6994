// persist_tm.cuh — the persistent Lanczos extension (Alg. 2) with the CTA's
// row-resident vectors in TENSOR MEMORY instead of shared memory.
//
// krylov_persist_kernel (persist.cuh) keeps y (phase A -> phase B) and v~_{j-1} (-> the next
// step's three-term recurrence) of the CTA's ~14K rows in a 113 KB shared-memory slice, which
// leaves room for only one TMA halo tile: every tile waits for its own halo (ncu: ~15 % of the
// warp-stall samples at c4 on the mbarrier wait).  Nothing on this path issues an MMA, so the
// 256 KB of TMEM per SM is free: each thread owns 64 columns of its TMEM lane (8 warps share a
// 32-lane quarter of the 512 columns) and keeps there, per row pair of each tile,
//   slot A (cols  0..31): y     = sigma_j A v~_j - lz v~_{j-1}       (written in phase A)
//   slot B (cols 32..63): v~_j  = the x values of the thread's rows  (written in phase A)
// Phase B then needs no global loads at all (v~_{j+1} = y - alpha sigma_j v~_j from TMEM), and
// the next step's -lz v~_{j-1} term reads slot B before phase A overwrites it with v~_{j+1}.
// Shared memory holds two halo tiles, so tile t + 1's (and t + 2's) bulk copies fly while tile t
// is computed; the last warp to finish a halo buffer issues the next tile into it (no CTA barrier in
// the tile loop), and the next step's first two tiles are issued as soon as every CTA has arrived
// at the update phase's grid phase.  Arithmetic per row and the grid all-reduce are those of
// krylov_persist_kernel; the dot and ||y||^2 are accumulated per thread across tiles and reduced
// once per phase (block_sums), and every thread derives the phase-end scalars (alpha_j, sigma_j,
// the Lanczos coefficient, breakdown) from the all-reduced totals itself, without a CTA barrier.
// Requires ceil(rows per CTA / TILE) * NP <= 8 (c4: 14176 rows, 4 tiles).
#pragma once

#include "persist.cuh"

namespace phipm {

constexpr int TM_PAIRS = 8;          // row pairs per thread per slot (4 columns each)

// two consecutive pairs (8 columns) of this thread's TMEM lane <- registers
__device__ __forceinline__ void tm_st8(uint32_t ta, const double2 &a, const double2 &b)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(ta),
                 "r"(__double2loint(a.x)), "r"(__double2hiint(a.x)), "r"(__double2loint(a.y)),
                 "r"(__double2hiint(a.y)), "r"(__double2loint(b.x)), "r"(__double2hiint(b.x)),
                 "r"(__double2loint(b.y)), "r"(__double2hiint(b.y))
                 : "memory");
}

// registers <- two consecutive pairs of slot A and two of slot B; the wait is inside the same asm
// statement, so no use of the destination registers can be scheduled before the data arrived
__device__ __forceinline__ void tm_ld8x2(uint32_t ta, uint32_t tb, double2 (&a)[2], double2 (&b)[2])
{
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%16];\n"
                 "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%8, %9, %10, %11, %12, %13, %14, %15}, [%17];\n"
                 "tcgen05.wait::ld.sync.aligned;"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                   "=r"(r[15])
                 : "r"(ta), "r"(tb)
                 : "memory");
    a[0] = make_double2(__hiloint2double(r[1], r[0]), __hiloint2double(r[3], r[2]));
    a[1] = make_double2(__hiloint2double(r[5], r[4]), __hiloint2double(r[7], r[6]));
    b[0] = make_double2(__hiloint2double(r[9], r[8]), __hiloint2double(r[11], r[10]));
    b[1] = make_double2(__hiloint2double(r[13], r[12]), __hiloint2double(r[15], r[14]));
}

// four consecutive pairs (16 columns) of slot A and four of slot B, one wait
__device__ __forceinline__ void tm_ld16x2(uint32_t ta, uint32_t tb, double2 (&a)[4], double2 (&b)[4])
{
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%32];\n"
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%33];\n"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(ta), "r"(tb)
        : "memory");
#pragma unroll
    for (int i = 0; i < 4; i++) {
        a[i] = make_double2(__hiloint2double(r[4 * i + 1], r[4 * i]), __hiloint2double(r[4 * i + 3], r[4 * i + 2]));
        b[i] = make_double2(__hiloint2double(r[16 + 4 * i + 1], r[16 + 4 * i]),
                            __hiloint2double(r[16 + 4 * i + 3], r[16 + 4 * i + 2]));
    }
}

__device__ __forceinline__ void tm_ld8(uint32_t ta, double2 (&a)[2])
{
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 "tcgen05.wait::ld.sync.aligned;"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(ta)
                 : "memory");
    a[0] = make_double2(__hiloint2double(r[1], r[0]), __hiloint2double(r[3], r[2]));
    a[1] = make_double2(__hiloint2double(r[5], r[4]), __hiloint2double(r[7], r[6]));
}

__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// dynamic shared memory (bytes): two halo tiles
__host__ __device__ inline size_t persist_tm_smem_bytes(int halo_cap)
{
    return (size_t)2 * ((halo_cap + 15) & ~15) * sizeof(double);
}

// block sums of NV values per thread into out[0..NV) (visible to every thread on return): a shuffle
// tree per warp, then warp 0 reduces the SNW warp totals of each value with another shuffle tree.
// Two CTA barriers for all NV values (block_total below: two per value plus a serial 32-term loop).
// SYNC_OUT = false: out[] is only read by thread 0 afterwards (phase_allreduce's partials), which
// computed it, so the closing barrier is not needed
template <int NV, bool SYNC_OUT = true>
__device__ __forceinline__ void block_sums(const double (&v)[NV], double *wsum2, double *out)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; k++) {
        const double s = warp_sum(v[k]);
        if (lane == 0) wsum2[k * SNW + warp] = s;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < NV; k++) {
            const double s = warp_sum(lane < SNW ? wsum2[k * SNW + lane] : 0.0);
            if (lane == 0) out[k] = s;
        }
    }
    if (SYNC_OUT) __syncthreads();
}

// block sum of one value per thread (fixed order: shuffle tree, then warps in order by thread 0)
__device__ __forceinline__ double block_total(double v, double *wsum)
{
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < SNW; w++) t += wsum[w];
    __syncthreads();
    return t;                                              // valid in thread 0
}

template <int DIM>
__global__ void __launch_bounds__(SNT, 1) krylov_persist_tm_kernel(StencilOp op, PersistArgs a, Work wk)
{
    constexpr int RPT = 4;
    constexpr int TILE_ = SNT * RPT;
    constexpr int NP = RPT / 2;
    static_assert(NP == 2, "TMEM slots are moved two pairs (8 columns) at a time");
    extern __shared__ __align__(128) double sm[];
    __shared__ uint64_t hbar[2];
    __shared__ TilePlan tplan[TM_PAIRS / 2];
    __shared__ unsigned hcons[2];                      // warps done with each halo buffer (monotonic)
    __shared__ double bsum[2];
    __shared__ double red[MAXD + 2];
    __shared__ double wsum2[2 * SNW];
    __shared__ uint32_t s_tmem;
    __shared__ int s_stop;
    __shared__ double s_sig, s_lz;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int64_t n = op.n;
    const int64_t cs = (int64_t)blockIdx.x * a.rpc, ce = min(n, cs + a.rpc);
    const int hstride = (halo_capacity(op.dim, op.nx, TILE_) + 15) & ~15;
    const int64_t ldv = wk.ldv;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        mbar_init(&hbar[0], 1);
        mbar_init(&hbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    pdl_wait();                                            // the previous kernel's results from here on
    if (tid == 0) {
        s_stop = __ldcg(&wk.st->brk) >= 0;
        s_sig = __ldcg(wk.sigma + a.k0);
        s_lz = __ldcg(&wk.st->lz);
    }
    if (tid < 2) hcons[tid] = 0;
    if (tid < TM_PAIRS / 2) {
        const int64_t ru = cs + (int64_t)tid * TILE_;
        if (ru < ce) tile_plan<TILE_>(op, ldv, ru, (int)min((int64_t)TILE_, ce - ru), tplan[tid]);
    }
    const uint64_t pol = policy_evict_last();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    double sig = s_sig, lzc = s_lz;                        // sigma_j and the Lanczos coefficient, per thread
    bool stop = s_stop != 0;
    // this thread's 64 columns: lane quarter warp % 4, column block warp / 4
    const uint32_t tbase = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));
    const uint32_t slotA = tbase, slotB = tbase + 32;
    uint32_t ht = 0;
    unsigned phase = 0;
    const bool lead = blockIdx.x == 0;
    bool pre = false;                                      // the next SpMV phase's first tiles are in flight
    bool aborted = false;                                  // a grid phase timed out (no counter reset)
    auto issue_first = [&](const double *xj) {            // (one thread)
        for (int u = 0; u < 2; u++) {
            const int64_t ru = cs + (int64_t)u * TILE_;
            const uint32_t g = ht + u;
            if (ru < ce) issue_planned_tile(tplan[u], sm + (g & 1) * hstride, xj, &hbar[g & 1], pol);
        }
    };
    const int3 gc0 = grid_coords(op, cs + 2 * tid);
    for (int j = a.k0; j < a.k1; j++) {
        if (stop) break;                                   // breakdown (same decision in every CTA)
        const double *x = wk.V + (int64_t)j * ldv;
        const double sj = sig;
        const double *zv = j > 0 ? x - ldv : nullptr;      // v~_{j-1} (Alg. 2 line 3)
        const double lz = zv ? lzc : 0.0;
        const bool zs = j > a.k0;                          // v~_{j-1} of these rows is in slot B

        // ---------------- phase A: y = sigma_j A x - lz v~_{j-1}; d = x^T y; ||y||^2
        if (tid == 0 && !pre) issue_first(x);
        pre = false;
        double ysq = 0.0, dot = 0.0;
        int3 gcoord = gc0;
        int t = 0;
        for (int64_t r0 = cs; r0 < ce; r0 += TILE_, t++) {
            const int rows = (int)min((int64_t)TILE_, ce - r0);
            double2 zp[NP];
            if (zv && zs) {
                tm_ld8(slotB + 8 * t, zp);
            } else {
#pragma unroll
                for (int p = 0; p < NP; p++) {
                    const int q = 2 * tid + 2 * SNT * p;
                    zp[p].x = (zv && q < rows) ? __ldcg(zv + r0 + q) : 0.0;
                    zp[p].y = (zv && q + 1 < rows) ? __ldcg(zv + r0 + q + 1) : 0.0;
                }
            }
            const uint32_t g = ht++;
            double *hb = sm + (g & 1) * hstride;
            double2 y[NP], xr[NP];
            mbar_wait(&hbar[g & 1], (g >> 1) & 1);
            stencil_tile_d<NP, (DIM == 4 ? 2 : DIM), (DIM == 4)>(op, hb, tplan[t].ho, r0, rows, tid, y, xr, &gcoord);
            // halo buffer g & 1 consumed by this warp: no CTA barrier -- the last warp to finish it
            // (monotonic per-buffer counter: use g >> 1 ends at SNW ((g >> 1) + 1)) issues tile t + 2
            __syncwarp();
            if ((tid & 31) == 0) {
                unsigned old;
                asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                             : "=r"(old) : "r"(smem_u32(&hcons[g & 1])) : "memory");
                if (old == (unsigned)SNW * ((g >> 1) + 1) - 1 && r0 + 2 * TILE_ < ce)
                    issue_planned_tile(tplan[t + 2], hb, x, &hbar[g & 1], pol);
            }
#pragma unroll
            for (int p = 0; p < NP; p++) {
                const int q = 2 * tid + 2 * SNT * p;
                y[p].x *= sj;
                y[p].y *= sj;
                if (zv) {
                    if (q < rows) y[p].x = fma(-lz, zp[p].x, y[p].x);
                    if (q + 1 < rows) y[p].y = fma(-lz, zp[p].y, y[p].y);
                }
                ysq = fma(y[p].x, y[p].x, ysq);
                ysq = fma(y[p].y, y[p].y, ysq);
                dot = fma(xr[p].x, y[p].x, dot);
                dot = fma(xr[p].y, y[p].y, dot);
            }
            tm_st8(slotA + 8 * t, y[0], y[1]);
            tm_st8(slotB + 8 * t, xr[0], xr[1]);
        }
        tm_wait_st();
        {
            const double v2[2] = {dot, ysq};
            block_sums<2, false>(v2, wsum2, bsum);
        }
        if (!phase_allreduce(wk, bsum, 2, ++phase, a, red)) {
            aborted = true;
            break;
        }
        // finalize (FIN_LANCZOS): alpha_j = sigma_j d; update coefficient -alpha_j sigma_j -- derived by
        // every thread from the all-reduced totals (no CTA barrier); CTA 0 thread 0 writes H for the host
        const double al = sj * red[0];
        const double cf = -(al * sj);
        if (lead && tid == 0) {
            wk.H[j + (size_t)j * wk.ldh] = al;
            wk.g[0] = al * sj;
            wk.st->wnorm2 = red[1];
        }

        // ---------------- phase B: v~_{j+1} = y - alpha_j sigma_j v~_j (both from TMEM); ||v~_{j+1}||^2
        double *vn = wk.V + (int64_t)(j + 1) * ldv;
        double nrm = 0.0;
        // two tiles per TMEM load (16 columns of each slot, one wait)
        for (int64_t rp = cs; rp < ce; rp += 2 * TILE_) {
            const int tp = (int)((rp - cs) / TILE_);
            double2 yv[2 * NP], xv[2 * NP];
            tm_ld16x2(slotA + 8 * tp, slotB + 8 * tp, yv, xv);
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int64_t r0 = rp + (int64_t)h * TILE_;
                const int rows = (int)max((int64_t)0, min((int64_t)TILE_, ce - r0));
#pragma unroll
                for (int p = 0; p < NP; p++) {
                    const int q = 2 * tid + 2 * SNT * p;
                    double2 acc;
                    acc.x = fma(cf, xv[h * NP + p].x, yv[h * NP + p].x);
                    acc.y = fma(cf, xv[h * NP + p].y, yv[h * NP + p].y);
                    double *o = vn + r0 + q;
                    if (q + 1 < rows) *reinterpret_cast<double2 *>(o) = acc;
                    else if (q < rows) o[0] = acc.x;
                    if (q < rows) nrm = fma(acc.x, acc.x, nrm);
                    if (q + 1 < rows) nrm = fma(acc.y, acc.y, nrm);
                }
            }
        }
        {
            const double v1[1] = {nrm};
            block_sums<1, false>(v1, wsum2, bsum);
        }
        // v~_{j+1} is complete in every CTA once the phase's arrivals are in: the next step's first
        // halo tiles are issued then, while the partials are summed (drained below on breakdown)
        const bool more = j + 1 < a.k1;
        if (!phase_allreduce(wk, bsum, 1, ++phase, a, red, [&] {
                if (more) issue_first(x + ldv);
            })) {
            aborted = true;
            break;
        }
        pre = more;
        // finalize (FIN_NORM): h_{j+1,j}, sigma_{j+1}, the Lanczos coefficient, breakdown -- derived by
        // every thread from the all-reduced total (identical in every thread and CTA; no CTA barrier)
        {
            const double h = sqrt(red[0]);
            const double sn = 1.0 / h;
            const double lzn = h * sj;
            int brk = -1, nonfin = 0;
            if (!isfinite(h)) { nonfin = 1; brk = j + 1; }
            else if (h <= a.bthr) brk = j + 1;
            sig = sn;
            lzc = lzn;
            stop = brk >= 0;
            if (lead && tid == 0) {
                wk.H[(j + 1) + (size_t)j * wk.ldh] = h;
                if (j + 1 < wk.hcols) wk.H[j + (size_t)(j + 1) * wk.ldh] = h;
                wk.st->lz = lzn;
                wk.sigma[j + 1] = sn;
                if (nonfin) wk.st->nonfinite = 1;
                if (brk >= 0) wk.st->brk = brk;
            }
        }
    }
    // first tiles issued for a step that did not run (breakdown): land them before the CTA exits
    if (pre)
        for (int u = 0; u < 2; u++)
            if (cs + (int64_t)u * TILE_ < ce) mbar_wait(&hbar[(ht + u) & 1], ((ht + u) >> 1) & 1);
    // every warp's TMEM traffic is complete before warp 0 frees the columns
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem) : "memory");
    if (!aborted) coop_exit(a);
}

} // namespace phipm
