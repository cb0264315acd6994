// persist_brick.cuh — the persistent Lanczos extension (Alg. 2) of a 3-D 7-point
// stencil on 3-D BRICKS staged by tensor-map TMA (cp.async.bulk.tensor), y / v~_j in tensor memory.
//
// krylov_persist_tm_kernel (persist_tm.cuh) gives every CTA a contiguous row range (< one z-plane at
// c4) and stages, per 4096-row tile, five 1-D segments of x: each x value is read three times from L2
// (as a centre, a z- and a z+ neighbour), and ~70 % of the instructions it executes are row-coordinate
// bookkeeping, boundary predicates and halo-plan arithmetic (ncu, profiles/round2: DMUL+DADD+DFMA 16 %
// of the warp instructions; the kernel is issue-bound, not bandwidth-bound).  Here
//   * a CTA owns a brick: every x of `ylen` grid lines by `zlen` planes.  One 4-D tensor map over the
//     Krylov basis (x, y, z, column) describes it; plane s of the brick with its one-line / two-point
//     halo is ONE box copy (nx + 4) x (ylen + 2) x 1 x 1, and the TMA engine zero-fills what lies
//     outside the grid (negative or too large coordinates), so the stencil has NO boundary branches:
//     an absent neighbour contributes c * 0 = +-0, which leaves the ascending-column sum unchanged
//     bit for bit (the sum starts at +0 and +0 + -0 = +0).  Halo traffic: (ylen+2)(zlen+2)/(ylen zlen)
//     = 1.41 x at c4 instead of 3 x;
//   * a warp owns 64 consecutive x of one line and marches `ppg` <= 8 planes along z with the centre
//     values of planes z-1, z, z+1 in registers: per row pair and plane 3 16-byte and 2 8-byte shared
//     loads, 28 separately rounded multiply / adds, no index arithmetic beyond a plane stride;
//   * the whole brick (zlen + 2 planes) is resident in shared memory, one mbarrier per plane: all the
//     plane copies of the next step are issued the moment the grid phase of the update releases,
//     in the order the marching warps need them.
// y and v~_j of the thread's row pairs live in its TMEM columns exactly as in persist_tm.cuh (slot A /
// slot B, pair t = plane t of the warp), the update phase reads only TMEM, and the grid all-reduce,
// the finalize arithmetic and the breakdown rule are those of krylov_persist_tm_kernel.
#pragma once

#include <cuda.h>

#include "persist_tm.cuh"
#include "persist_wrec.cuh"

namespace phipm {

constexpr int BRICK_MAXPL = 36;      // staged planes per CTA (zlen + 2)

struct BrickGeom {
    int py, pz;        // bricks along y and z (grid = py pz)
    int ylen, zlen;    // lines / planes per brick (the last brick of a direction may hold fewer)
    int nseg;          // 64-point x segments per line
    int ncol;          // warp columns per CTA = nseg ylen (<= SNW)
    int ngrp;          // z groups per CTA = SNW / ncol
    int ppg;           // planes per z group (<= TM_PAIRS)
    int lstride;       // shared line stride (doubles) = nx + 4
    int pstride;       // shared plane stride (doubles), multiple of 16
};

__host__ __device__ inline size_t brick_smem_bytes(const BrickGeom &g)
{
    return (size_t)(g.zlen + 2) * g.pstride * sizeof(double);
}

// Host: the brick decomposition of an nx x ny x nz grid on at most `ctas` CTAs with the fewest planes
// per warp (the critical path), then the least staged volume.  false: no decomposition fits.
inline bool brick_geometry(int nx, int ny, int nz, int ctas, size_t smem_max, BrickGeom &best)
{
    if ((nx & 1) || nx < 2 || nx > 252) return false;
    const int nseg = (nx + 63) / 64;
    bool found = false;
    long long bcost = 0;
    for (int ylen = 1; ylen <= ny && nseg * ylen <= SNW; ylen++) {
        BrickGeom g;
        g.nseg = nseg;
        g.ylen = ylen;
        g.ncol = nseg * ylen;
        g.ngrp = SNW / g.ncol;
        g.py = (ny + ylen - 1) / ylen;
        g.lstride = nx + 4;
        g.pstride = ((ylen + 2) * g.lstride + 15) & ~15;
        for (int ppg = 1; ppg <= TM_PAIRS; ppg++) {
            g.ppg = ppg;
            g.zlen = g.ngrp * ppg < nz ? g.ngrp * ppg : nz;
            g.pz = (nz + g.zlen - 1) / g.zlen;
            if ((long long)g.py * g.pz > ctas) continue;
            if (g.zlen + 2 > BRICK_MAXPL || brick_smem_bytes(g) > smem_max) break;
            const long long cost = ((long long)ppg << 40) + (long long)g.py * g.pz * (g.zlen + 2) * g.pstride;
            if (!found || cost < bcost) {
                found = true;
                bcost = cost;
                best = g;
            }
            break;                                         // larger ppg only costs more
        }
    }
    return found;
}

// one box of the 4-D tensor map (x, y, z, column) -> shared memory, completion on an mbarrier
__device__ __forceinline__ void tma_load_box4(void *dst, const CUtensorMap *tm, int cx, int cy, int cz, int cc,
                                              uint64_t *bar, uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(dst)),
        "l"(tm), "r"(cx), "r"(cy), "r"(cz), "r"(cc), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// shared memory -> one box of the tensor map (bulk async-group; elements with out-of-range coordinates are
// not written)
__device__ __forceinline__ void tma_store_box4(const CUtensorMap *tm, int cx, int cy, int cz, int cc, const void *src)
{
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(tm),
                 "r"(cx), "r"(cy), "r"(cz), "r"(cc), "r"(smem_u32(src))
                 : "memory");
}

// one pair (4 columns) of this thread's TMEM lane <- registers
__device__ __forceinline__ void tm_st4(uint32_t ta, const double2 &a)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ta), "r"(__double2loint(a.x)),
                 "r"(__double2hiint(a.x)), "r"(__double2loint(a.y)), "r"(__double2hiint(a.y))
                 : "memory");
}

// registers <- one pair; the wait is a separate statement (tm_ld4_wait) so that the shared loads and
// the stencil arithmetic of the plane overlap the TMEM read
__device__ __forceinline__ void tm_ld4_issue(uint32_t ta, uint32_t (&r)[4])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(ta)
                 : "memory");
}

__device__ __forceinline__ double2 tm_ld4_wait(uint32_t (&r)[4])
{
    // the registers are operands of the wait: no use of them can be scheduled before it
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3])::"memory");
    return make_double2(__hiloint2double(r[1], r[0]), __hiloint2double(r[3], r[2]));
}

// RAGGED: nx is not a multiple of 64, so some lanes of a line's last segment hold no rows and their
// contributions are masked (compile-time: the full-line instantiation carries no selects)
template <bool RAGGED>
__global__ void __launch_bounds__(SNT, 1)
krylov_brick_tm_kernel(const __grid_constant__ CUtensorMap tmap, StencilOp op, BrickGeom g, PersistArgs a, Work wk)
{
    extern __shared__ __align__(128) double sm[];
    __shared__ uint64_t pbar[BRICK_MAXPL];
    __shared__ unsigned char porder[BRICK_MAXPL];
    __shared__ double bsum[2];
    __shared__ double red[MAXD + 2];
    __shared__ double wsum2[2 * SNW];
    __shared__ uint32_t s_tmem;
    __shared__ int s_stop;
    __shared__ double s_sig, s_lz;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nx = op.nx, ny = op.ny, nz = op.nz;
    const int64_t ldv = wk.ldv;
    // this CTA's brick and this warp's column of it
    const int by = blockIdx.x % g.py, bz = blockIdx.x / g.py;
    const int y0 = by * g.ylen, z0 = bz * g.zlen;
    const int zl = min(g.zlen, nz - z0);                   // planes of this brick
    const int col = warp % g.ncol, grp = warp / g.ncol;
    const int seg = col % g.nseg, yl = col / g.nseg;
    const int xi = seg * 64 + 2 * lane;                    // rows (xi, yy, z) and (xi + 1, yy, z)
    const int yy = y0 + yl;
    const int zb = grp * g.ppg;                            // first plane of the warp, brick-relative
    const int cnt = (grp < g.ngrp && yy < ny) ? max(0, min(g.ppg, zl - zb)) : 0;   // planes (warp-uniform)
    const bool act = xi < nx;                              // this lane holds a row pair
    const uint32_t plane_bytes = (uint32_t)(g.lstride * (g.ylen + 2)) * 8u;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid < zl + 2) mbar_init(&pbar[tid], 1);
    if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    pdl_wait();                                            // the previous kernel's results from here on
    if (tid == 0) {
        s_stop = __ldcg(&wk.st->brk) >= 0;
        s_sig = __ldcg(wk.sigma + a.k0);
        s_lz = __ldcg(&wk.st->lz);
    }
    const uint64_t pol = policy_evict_last();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    double sig = s_sig, lzc = s_lz;                        // sigma_j and the Lanczos coefficient, per thread
    bool stop = s_stop != 0;
    const uint32_t tbase = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));
    const uint32_t slotA = tbase, slotB = tbase + 32;
    unsigned phase = 0;
    const bool lead = blockIdx.x == 0;
    bool pre = false;                                      // the next step's planes are in flight
    bool aborted = false;
    uint32_t par = 0;                                      // mbarrier parity of the current step
    // the brick's planes in the order the marching warps reach them: plane t of every z group, t ascending
    // (planes ppg, ppg + 1 of a group are planes 0, 1 of the group above)
    if (tid == 0) {
        int o = 0;
        for (int t = 0; t < g.ppg + 2; t++)
            for (int gi = 0; gi < g.ngrp; gi++) {
                if (t >= g.ppg && gi + 1 < g.ngrp) continue;
                const int s = gi * g.ppg + t;
                if (s <= zl + 1) porder[o++] = (unsigned char)s;
            }
    }
    __syncthreads();
    // plane copies of Krylov column jc: lane 0 of warp w issues planes porder[w], porder[w + SNW], ... (one
    // thread issuing all zlen + 2 copies held the CTA for > 1 us at c4)
    auto issue_planes = [&](int jc) {
        if (lane == 0)
            for (int o = warp; o < zl + 2; o += SNW) {
                const int s = porder[o];
                mbar_arrive_expect_tx(&pbar[s], plane_bytes);
                tma_load_box4(sm + (size_t)s * g.pstride, &tmap, -2, y0 - 1, z0 - 1 + s, jc, &pbar[s], pol);
            }
    };
    const int xa = act ? xi : 0;                           // (idle lanes read a valid address)
    // shared address of the warp's centre pair in the plane below its first one; byte strides
    const uint32_t pa0 = smem_u32(sm + (yl + 1) * g.lstride + xa + 2 + zb * g.pstride);
    const uint32_t ps8 = (uint32_t)g.pstride * 8u, ls8 = (uint32_t)g.lstride * 8u;
    const uint32_t pb0 = smem_u32(&pbar[zb]);
    const int64_t row0 = xa + (int64_t)nx * (yy + (int64_t)ny * (z0 + zb));     // row of (xi, yy, z0 + zb)
    const int64_t pl = (int64_t)nx * ny;
    const double c0 = op.c[0], cxm = op.c[1], cxp = op.c[2], cym = op.c[3], cyp = op.c[4], czm = op.c[5],
                 czp = op.c[6];
    auto lds2 = [](uint32_t ad) {
        double2 r;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "r"(ad));
        return r;
    };
    auto lds1 = [](uint32_t ad) {
        double r;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(r) : "r"(ad));
        return r;
    };
    auto bar_wait = [](uint32_t bar, uint32_t parity) {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "WAIT_%=:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            "@!p bra WAIT_%=;\n"
            "}\n" ::"r"(bar),
            "r"(parity)
            : "memory");
    };
    for (int j = a.k0; j < a.k1; j++) {
        if (stop) break;                                   // breakdown (same decision in every CTA)
        const double sj = sig;
        const double *zv = j > 0 ? wk.V + (int64_t)(j - 1) * ldv : nullptr;     // v~_{j-1} (Alg. 2 line 3)
        const double lz = zv ? lzc : 0.0;

        // ---------------- phase A: y = sigma_j A x - lz v~_{j-1}; d = x^T y; ||y||^2
        if (!pre) {
            if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue_planes(j);
        }
        pre = false;
        double ysq = 0.0, dot = 0.0;
#ifdef BRICK_CLK
        unsigned long long ck0 = gtimer(), ck1 = 0, ck2 = 0, ck3 = 0, ckp[TM_PAIRS] = {};
        long long ckw = 0;
#endif
        if (cnt > 0) {
            // first step of the launch: v~_{j-1} of the warp's rows from global memory into slot B (zeros
            // for j = 0); afterwards phase A of the previous step left v~_j = this step's v~_{j-1} there
            if (j == a.k0) {
#pragma unroll
                for (int t = 0; t < TM_PAIRS; t++) {
                    if (t >= cnt) break;
                    const double2 z = (zv && act) ? ld_cg2(zv + row0 + t * pl) : make_double2(0.0, 0.0);
                    tm_st4(slotB + 4 * t, z);
                }
                tm_wait_st();
            }
            bar_wait(pb0, par);
            bar_wait(pb0 + 8, par);
#ifdef BRICK_CLK
            ck1 = gtimer();
#endif
            double2 zm = lds2(pa0), zc = lds2(pa0 + ps8);
            uint32_t pa = pa0 + ps8;                       // centre pair of the current plane
#pragma unroll
            for (int t = 0; t < TM_PAIRS; t++) {
                if (t >= cnt) break;
                uint32_t zr[4];
                tm_ld4_issue(slotB + 4 * t, zr);
#ifdef BRICK_CLK
                const long long cw0 = clock64();
#endif
                bar_wait(pb0 + 8 * (t + 2), par);
#ifdef BRICK_CLK
                ckw += clock64() - cw0;
#endif
                const uint32_t pn = pa + ps8;
                const double2 zn = lds2(pn);
                const double2 ym = lds2(pa - ls8), yp = lds2(pa + ls8);
                const double xl = lds1(pa - 8), xh = lds1(pa + 16);
                // ascending columns z-, y-, x-, centre, x+, y+, z+ (fused multiply-adds)
                double sa = czm * zm.x, sb = czm * zm.y;
                sa = fma(cym, ym.x, sa);
                sb = fma(cym, ym.y, sb);
                sa = fma(cxm, xl, sa);
                sb = fma(cxm, zc.x, sb);
                sa = fma(c0, zc.x, sa);
                sb = fma(c0, zc.y, sb);
                sa = fma(cxp, zc.y, sa);
                sb = fma(cxp, xh, sb);
                sa = fma(cyp, yp.x, sa);
                sb = fma(cyp, yp.y, sb);
                sa = fma(czp, zn.x, sa);
                sb = fma(czp, zn.y, sb);
                const double2 zq = tm_ld4_wait(zr);
                double2 y = make_double2(fma(-lz, zq.x, sa * sj), fma(-lz, zq.y, sb * sj));
                double2 xc = zc;
                if (RAGGED && !act) {
                    y = make_double2(0.0, 0.0);
                    xc = y;
                }
                ysq = fma(y.x, y.x, ysq);
                ysq = fma(y.y, y.y, ysq);
                dot = fma(xc.x, y.x, dot);
                dot = fma(xc.y, y.y, dot);
                tm_st4(slotA + 4 * t, y);
                tm_st4(slotB + 4 * t, xc);
                zm = zc;
                zc = zn;
                pa = pn;
#ifdef BRICK_CLK
                ckp[t] = gtimer();
#endif
            }
            tm_wait_st();
        }
#ifdef BRICK_CLK
        ck2 = gtimer();
#endif
        {
            const double v2[2] = {dot, ysq};
            block_sums<2, false>(v2, wsum2, bsum);
        }
#ifdef BRICK_CLK
        // (measurement build: where one CTA's SpMV phase goes, ns from the phase start of each warp)
        ck3 = gtimer();
        if (blockIdx.x == 37 && j == a.k0 + 4 && lane == 0)
            printf("w%02d A: start %llu planes01 +%llu p0 +%llu p1 +%llu p3 +%llu p5 +%llu march +%llu sums +%llu; plane waits %lld cycles\n", warp,
                   ck0 % 1000000, ck1 - ck0, ckp[0] - ck0, ckp[1] - ck0, ckp[3] - ck0, ckp[5] - ck0, ck2 - ck0, ck3 - ck0, ckw);
#endif
        if (!phase_allreduce(wk, bsum, 2, ++phase, a, red)) {
            aborted = true;
            break;
        }
        // finalize (FIN_LANCZOS): alpha_j = sigma_j d; update coefficient -alpha_j sigma_j
        const double al = sj * red[0];
        const double cf = -(al * sj);
        if (lead && tid == 0) {
            wk.H[j + (size_t)j * wk.ldh] = al;
            wk.g[0] = al * sj;
            wk.st->wnorm2 = red[1];
        }

        // ---------------- phase B: v~_{j+1} = y - alpha_j sigma_j v~_j (both from TMEM); ||v~_{j+1}||^2
        double *vn = wk.V + (int64_t)(j + 1) * ldv + row0;
        double nrm = 0.0;
#pragma unroll
        for (int h = 0; h < TM_PAIRS / 4; h++) {
            if (4 * h >= cnt) break;
            double2 yv[4], xv[4];
            tm_ld16x2(slotA + 16 * h, slotB + 16 * h, yv, xv);
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int t = 4 * h + u;
                if (t < cnt && act) {
                    double2 acc;
                    acc.x = fma(cf, xv[u].x, yv[u].x);
                    acc.y = fma(cf, xv[u].y, yv[u].y);
                    *reinterpret_cast<double2 *>(vn + t * pl) = acc;
                    nrm = fma(acc.x, acc.x, nrm);
                    nrm = fma(acc.y, acc.y, nrm);
                }
            }
        }
        {
            const double v1[1] = {nrm};
            block_sums<1, false>(v1, wsum2, bsum);
        }
        // v~_{j+1} is complete in every CTA once the phase's arrivals are in: the next step's planes are
        // issued then, while the partials are summed (drained below on breakdown)
        const bool more = j + 1 < a.k1;
        if (!phase_allreduce(wk, bsum, 1, ++phase, a, red, NoRelease{}, [&] {
                if (more) issue_planes(j + 1);
            })) {
            aborted = true;
            break;
        }
        pre = more;
        par ^= 1u;
        // finalize (FIN_NORM): h_{j+1,j}, sigma_{j+1}, the Lanczos coefficient, breakdown
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
    // planes issued for a step that did not run (breakdown): land them before the CTA exits
    if (pre && tid == 0)
        for (int s = 0; s < zl + 2; s++) mbar_wait(&pbar[s], par);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem) : "memory");
    if (!aborted) coop_exit(a);
}


// ---------------------------------------------------------------------------------------------
// krylov_brick_halo_kernel: the brick Lanczos extension with the brick's INTERIOR kept in shared memory from
// step to step.  krylov_brick_tm_kernel re-stages every plane of the brick (interior and halo, 1.41 x the
// vector) through the tensor map each step, so the update phase must have written ALL of v~_{j+1} to global
// memory before its grid phase releases: 16.8 MB through L2 on the critical path (~2.4 us at c4).  Here
//   * the update phase stores v~_{j+1} of the CTA's rows into its own shared-memory brick (the next SpMV
//     phase reads the interior from there) and the brick's planes go to global memory as tensor STORES
//     (cp.async.bulk.tensor shared -> global, one per plane, issued by lane 0 of the plane's warp and waited
//     for before the arrival): the threads issue no global stores at all.  (Measured first: per-thread
//     16-byte stores of the shell rows before the arrival and of the other rows after it did not shorten the
//     phase -- its length is the store issue itself, 128 KB per SM through the LSU, wherever it is placed;)
//   * only the halo is copied per step: the plane below and above the brick (two boxes nx x ylen x 1) and the
//     line before and after it on every plane (two boxes nx x 1 x zlen), four tensor copies and 49 KB instead
//     of 18 copies and 190 KB at c4, zero fill outside the grid in y and z as before;
//   * shared memory: planes 0 .. zlen + 1 of ylen dense lines (no y-halo lines inside a plane, no x pads) and
//     two y-halo arrays [zlen][nx]; a warp on the brick's first / last line reads its y neighbour from the array
//     (per-warp base and stride), every other warp from the adjacent interior line.  The lines
//     past the grid are zeroed once (nobody writes them).
// Arithmetic, TMEM use, reductions and finalize steps are those of krylov_brick_tm_kernel (bit-identical
// results); the first step of a launch loads the interior of column k0 from global memory.
// MEASURED SLOWER than krylov_brick_tm_kernel at c4 and therefore not the default (option brick_halo): the
// SpMV phase is unchanged (5.9 us: it is instruction-issue bound, not bound by the plane copies), and the
// update phase grows from 3.4 to 5.1 us (eight 16 KB tensor stores per CTA and their completion wait cost more
// than 8 16-byte stores per thread); 3320 vs 3500 solves/s.
// (lines are dense here: nx doubles, no pads -- tensor stores reject negative coordinates, so a box cannot
// start at x = -2; the x neighbour of a line's first / last point is removed by a zero coefficient instead)
__host__ __device__ inline int brick_halo_ps(const BrickGeom &g) { return (g.ylen * (g.lstride - 4) + 15) & ~15; }
__host__ __device__ inline int brick_halo_ys(const BrickGeom &g) { return (g.zlen * (g.lstride - 4) + 15) & ~15; }
__host__ __device__ inline size_t brick_halo_smem_bytes(const BrickGeom &g)
{
    // 16 doubles before and after the arrays: x - 1 of the first and x + 2 of the last element stay inside
    return ((size_t)(g.zlen + 2) * brick_halo_ps(g) + 2 * (size_t)brick_halo_ys(g) + 32) * sizeof(double);
}

template <bool RAGGED>
__global__ void __launch_bounds__(SNT, 1)
krylov_brick_halo_kernel(const __grid_constant__ CUtensorMap tmz, const __grid_constant__ CUtensorMap tmy, StencilOp op,
                         BrickGeom g, PersistArgs a, Work wk)
{
    extern __shared__ __align__(128) double sm_raw[];
    double *const sm = sm_raw + 16;
    __shared__ uint64_t hb[3];                             // z- plane, z+ plane, both y-halo arrays
    __shared__ double bsum[2];
    __shared__ double red[MAXD + 2];
    __shared__ double wsum2[2 * SNW];
    __shared__ uint32_t s_tmem;
    __shared__ int s_stop;
    __shared__ double s_sig, s_lz;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nx = op.nx, ny = op.ny, nz = op.nz;
    const int64_t ldv = wk.ldv;
    const int by = blockIdx.x % g.py, bz = blockIdx.x / g.py;
    const int y0 = by * g.ylen, z0 = bz * g.zlen;
    const int zl = min(g.zlen, nz - z0);                   // planes of this brick
    const int col = warp % g.ncol, grp = warp / g.ncol;
    const int seg = col % g.nseg, yl = col / g.nseg;
    const int xi = seg * 64 + 2 * lane;
    const int yy = y0 + yl;
    const int zb = grp * g.ppg;
    const int cnt = (grp < g.ngrp && yy < ny) ? max(0, min(g.ppg, zl - zb)) : 0;
    const bool act = xi < nx;
    const int ps = brick_halo_ps(g), ys = brick_halo_ys(g);
    double *const ymarr = sm + (size_t)(g.zlen + 2) * ps, *const yparr = ymarr + ys;
    const uint32_t zbytes = (uint32_t)(nx * g.ylen) * 8u, ybytes = (uint32_t)(nx * g.zlen) * 8u;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid < 3) mbar_init(&hb[tid], 1);
    if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // pads, lines past the grid, halo arrays: zero once
    for (int i = tid; i < (g.zlen + 2) * ps + 2 * ys + 32; i += SNT) sm_raw[i] = 0.0;
    pdl_wait();                                            // the previous kernel's results from here on
    if (tid == 0) {
        s_stop = __ldcg(&wk.st->brk) >= 0;
        s_sig = __ldcg(wk.sigma + a.k0);
        s_lz = __ldcg(&wk.st->lz);
    }
    const uint64_t pol = policy_evict_last();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    double sig = s_sig, lzc = s_lz;
    bool stop = s_stop != 0;
    const uint32_t tbase = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));
    const uint32_t slotA = tbase, slotB = tbase + 32;
    unsigned phase = 0;
    const bool lead = blockIdx.x == 0;
    bool pre = false;                                      // the next step's halo copies are in flight
    bool aborted = false;
    uint32_t par = 0;
    // halo copies of Krylov column jc: lane 0 of warps 0..3, one copy each
    auto issue_halo = [&](int jc) {
        if (lane == 0 && warp < 4) {
            if (warp == 0) {
                mbar_arrive_expect_tx(&hb[0], zbytes);
                tma_load_box4(sm, &tmz, 0, y0, z0 - 1, jc, &hb[0], pol);
            } else if (warp == 1) {
                mbar_arrive_expect_tx(&hb[1], zbytes);
                tma_load_box4(sm + (size_t)(zl + 1) * ps, &tmz, 0, y0, z0 + zl, jc, &hb[1], pol);
            } else if (warp == 2) {
                mbar_arrive_expect_tx(&hb[2], 2 * ybytes);
                tma_load_box4(ymarr, &tmy, 0, y0 - 1, z0, jc, &hb[2], pol);
            } else {
                tma_load_box4(yparr, &tmy, 0, y0 + g.ylen, z0, jc, &hb[2], pol);
            }
        }
    };
    const int xa = act ? xi : 0;
    const uint32_t ps8 = (uint32_t)ps * 8u, ls8 = (uint32_t)nx * 8u;
    // shared address of the warp's centre pair in the plane below its first one (plane index zb of the buffer)
    const uint32_t pa0 = smem_u32(sm + (size_t)zb * ps + yl * nx + xa);
    // y neighbours: the adjacent interior line, or the halo array on the brick's first / last line
    const bool ylo = yl == 0, yhi = yl == g.ylen - 1;
    const uint32_t ym0 = ylo ? smem_u32(ymarr + zb * nx + xa) : pa0 + ps8 - ls8;
    const uint32_t yp0 = yhi ? smem_u32(yparr + zb * nx + xa) : pa0 + ps8 + ls8;
    const uint32_t yms = ylo ? ls8 : ps8, yps = yhi ? ls8 : ps8;
    const uint32_t hb0 = smem_u32(&hb[0]);
    const int64_t row0 = xa + (int64_t)nx * (yy + (int64_t)ny * (z0 + zb));
    const int64_t pl = (int64_t)nx * ny;
    const double c0 = op.c[0], cxm = op.c[1], cxp = op.c[2], cym = op.c[3], cyp = op.c[4], czm = op.c[5],
                 czp = op.c[6];
    // the pair's outer x neighbours: absent at the ends of a line (dense lines: the value read there belongs to
    // the adjacent line), removed by a zero coefficient
    const double cxm_a = xi == 0 ? 0.0 : cxm, cxp_b = xi + 2 >= nx ? 0.0 : cxp;
    auto lds2 = [](uint32_t ad) {
        double2 r;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "r"(ad));
        return r;
    };
    auto lds1 = [](uint32_t ad) {
        double r;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(r) : "r"(ad));
        return r;
    };
    auto sts2 = [](uint32_t ad, const double2 &v) {
        asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(ad), "d"(v.x), "d"(v.y) : "memory");
    };
    auto bar_wait = [](uint32_t bar, uint32_t parity) {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "WAIT_%=:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            "@!p bra WAIT_%=;\n"
            "}\n" ::"r"(bar),
            "r"(parity)
            : "memory");
    };
    for (int j = a.k0; j < a.k1; j++) {
        if (stop) break;
        const double sj = sig;
        const double *zv = j > 0 ? wk.V + (int64_t)(j - 1) * ldv : nullptr;
        const double lz = zv ? lzc : 0.0;

        // ---------------- phase A: y = sigma_j A x - lz v~_{j-1}; d = x^T y; ||y||^2
        if (j == a.k0) {
            // first step of the launch: the interior of column k0 and v~_{k0-1} (slot B) from global memory
            const double *xg = wk.V + (int64_t)j * ldv + row0;
#pragma unroll
            for (int t = 0; t < TM_PAIRS; t++) {
                if (t >= cnt) break;
                double2 xv = make_double2(0.0, 0.0), z = xv;
                if (act) {
                    xv = ld_cg2(xg + t * pl);
                    if (zv) z = ld_cg2(zv + row0 + t * pl);
                    sts2(pa0 + (t + 1) * ps8, xv);
                }
                tm_st4(slotB + 4 * t, z);
            }
            if (cnt > 0) tm_wait_st();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // the zero fill, before the copies
            __syncthreads();                               // every warp's interior rows are in place
            issue_halo(j);
        }
        pre = false;
        double ysq = 0.0, dot = 0.0;
        if (cnt > 0) {
            if (zb == 0) bar_wait(hb0, par);               // the plane below the brick
            if (ylo || yhi) bar_wait(hb0 + 16, par);       // the lines before / after the brick
            double2 zm = lds2(pa0), zc = lds2(pa0 + ps8);
            uint32_t pa = pa0 + ps8, yma = ym0, ypa = yp0;
#pragma unroll
            for (int t = 0; t < TM_PAIRS; t++) {
                if (t >= cnt) break;
                uint32_t zr[4];
                tm_ld4_issue(slotB + 4 * t, zr);
                if (zb + t + 1 == zl) bar_wait(hb0 + 8, par);          // the plane above the brick
                const uint32_t pn = pa + ps8;
                const double2 zn = lds2(pn);
                const double2 ym = lds2(yma), yp = lds2(ypa);
                const double xl = lds1(pa - 8), xh = lds1(pa + 16);
                double sa = czm * zm.x, sb = czm * zm.y;
                sa = fma(cym, ym.x, sa);
                sb = fma(cym, ym.y, sb);
                sa = fma(cxm_a, xl, sa);
                sb = fma(cxm, zc.x, sb);
                sa = fma(c0, zc.x, sa);
                sb = fma(c0, zc.y, sb);
                sa = fma(cxp, zc.y, sa);
                sb = fma(cxp_b, xh, sb);
                sa = fma(cyp, yp.x, sa);
                sb = fma(cyp, yp.y, sb);
                sa = fma(czp, zn.x, sa);
                sb = fma(czp, zn.y, sb);
                const double2 zq = tm_ld4_wait(zr);
                double2 y = make_double2(fma(-lz, zq.x, sa * sj), fma(-lz, zq.y, sb * sj));
                double2 xc = zc;
                if (RAGGED && !act) {
                    y = make_double2(0.0, 0.0);
                    xc = y;
                }
                ysq = fma(y.x, y.x, ysq);
                ysq = fma(y.y, y.y, ysq);
                dot = fma(xc.x, y.x, dot);
                dot = fma(xc.y, y.y, dot);
                tm_st4(slotA + 4 * t, y);
                tm_st4(slotB + 4 * t, xc);
                zm = zc;
                zc = zn;
                pa = pn;
                yma += yms;
                ypa += yps;
            }
            tm_wait_st();
        }
        {
            const double v2[2] = {dot, ysq};
            block_sums<2, false>(v2, wsum2, bsum);
        }
        if (!phase_allreduce(wk, bsum, 2, ++phase, a, red)) {
            aborted = true;
            break;
        }
        const double al = sj * red[0];
        const double cf = -(al * sj);
        if (lead && tid == 0) {
            wk.H[j + (size_t)j * wk.ldh] = al;
            wk.g[0] = al * sj;
            wk.st->wnorm2 = red[1];
        }

        // ---------------- phase B: v~_{j+1} = y - alpha_j sigma_j v~_j (from TMEM) into the shared-memory brick;
        // shell rows to global memory now, the others after the arrival; ||v~_{j+1}||^2
        double nrm = 0.0;
#pragma unroll
        for (int h = 0; h < TM_PAIRS / 4; h++) {
            if (4 * h >= cnt) break;
            double2 yv[4], xv[4];
            tm_ld16x2(slotA + 16 * h, slotB + 16 * h, yv, xv);
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int t = 4 * h + u;
                if (t < cnt && act) {
                    double2 acc;
                    acc.x = fma(cf, xv[u].x, yv[u].x);
                    acc.y = fma(cf, xv[u].y, yv[u].y);
                    sts2(pa0 + (t + 1) * ps8, acc);
                    nrm = fma(acc.x, acc.x, nrm);
                    nrm = fma(acc.y, acc.y, nrm);
                }
            }
        }
        // the brick's planes of v~_{j+1}: shared memory -> global memory by tensor stores (lane 0 of warp q:
        // plane q; the pads and the lines past the grid have out-of-range coordinates and are not written),
        // complete before the CTA's arrival
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (lane == 0 && warp < zl) {
            for (int q = warp; q < zl; q += SNW)
                tma_store_box4(&tmz, 0, y0, z0 + q, j + 1, sm + (size_t)(q + 1) * ps);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        {
            const double v1[1] = {nrm};
            block_sums<1, false>(v1, wsum2, bsum);
        }
        const bool more = j + 1 < a.k1;
        if (!phase_allreduce(wk, bsum, 1, ++phase, a, red, NoRelease{}, [&] {
                if (more) issue_halo(j + 1);
            })) {
            aborted = true;
            break;
        }
        pre = more;
        par ^= 1u;
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
    // halo copies issued for a step that did not run (breakdown): land them before the CTA exits
    if (pre && tid == 0)
        for (int s = 0; s < 3; s++) mbar_wait(&hb[s], par);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem) : "memory");
    if (!aborted) coop_exit(a);
}

// ---------------------------------------------------------------------------------------------
// The w-recurrence of a step (Eq. wrecurrence; persist_wrec.cuh) on the same bricks:
//   w_0 = u_k ;  w_j = A w_{j-1} + sum_l t_k^l / l! u_{j+l}   (j = 1..p) ;  w_p -> V[:, 0], ||w_p||^2
// one cooperative kernel, p SpMV phases separated by grid phases.  Plane copies of w_{j-1} come from the
// tensor map of x_0 (j = 1: the caller's u_0 or its workspace copy) or of the context's W columns; the
// u-terms are read and w_j is written straight from / to global memory (a warp's 64 consecutive x of one
// line: coalesced 16-byte accesses).  The rows are the ascending-column sums with separately rounded
// products of every other SpMV of the library, then fma(c_l, u_{j+l}, y) in term order: w_1..w_p equal
// the streaming path's bit for bit (an absent neighbour adds c * 0, see above); ||w_p||^2 is summed in
// another order.  FIN_SEED as in wrec_persist_kernel.
__global__ void __launch_bounds__(SNT, 1)
wrec_brick_kernel(const __grid_constant__ CUtensorMap tmx0, const __grid_constant__ CUtensorMap tmw, StencilOp op,
                  BrickGeom g, WrecArgs w, PersistArgs a, Work wk)
{
    extern __shared__ __align__(128) double sm[];
    __shared__ uint64_t pbar[BRICK_MAXPL];
    __shared__ unsigned char porder[BRICK_MAXPL];
    __shared__ double bsum[2];
    __shared__ double red[MAXD + 2];
    __shared__ double wsum[SNW];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nx = op.nx, ny = op.ny, nz = op.nz;
    const int64_t ldv = wk.ldv;
    const int by = blockIdx.x % g.py, bz = blockIdx.x / g.py;
    const int y0 = by * g.ylen, z0 = bz * g.zlen;
    const int zl = min(g.zlen, nz - z0);
    const int col = warp % g.ncol, grp = warp / g.ncol;
    const int seg = col % g.nseg, yl = col / g.nseg;
    const int xi = seg * 64 + 2 * lane;
    const int yy = y0 + yl;
    const int zb = grp * g.ppg;
    const int cnt = (grp < g.ngrp && yy < ny) ? max(0, min(g.ppg, zl - zb)) : 0;
    const bool act = xi < nx;
    const uint32_t plane_bytes = (uint32_t)(g.lstride * (g.ylen + 2)) * 8u;
    if (tid < zl + 2) mbar_init(&pbar[tid], 1);
    if (tid == 0) {
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        int o = 0;
        for (int t = 0; t < g.ppg + 2; t++)
            for (int gi = 0; gi < g.ngrp; gi++) {
                if (t >= g.ppg && gi + 1 < g.ngrp) continue;
                const int s = gi * g.ppg + t;
                if (s <= zl + 1) porder[o++] = (unsigned char)s;
            }
    }
    const uint64_t pol = policy_evict_last();
    pdl_wait();
    __syncthreads();
    unsigned phase = 0;
    bool pre = false;
    uint32_t par = 0;
    auto issue_planes = [&](const CUtensorMap *tm, int jc) {
        if (lane == 0)
            for (int o = warp; o < zl + 2; o += SNW) {
                const int s = porder[o];
                mbar_arrive_expect_tx(&pbar[s], plane_bytes);
                tma_load_box4(sm + (size_t)s * g.pstride, tm, -2, y0 - 1, z0 - 1 + s, jc, &pbar[s], pol);
            }
    };
    const int xa = act ? xi : 0;
    const uint32_t pa0 = smem_u32(sm + (yl + 1) * g.lstride + xa + 2 + zb * g.pstride);
    const uint32_t ps8 = (uint32_t)g.pstride * 8u, ls8 = (uint32_t)g.lstride * 8u;
    const uint32_t pb0 = smem_u32(&pbar[zb]);
    const int64_t row0 = xa + (int64_t)nx * (yy + (int64_t)ny * (z0 + zb));
    const int64_t pl = (int64_t)nx * ny;
    const double c0 = op.c[0], cxm = op.c[1], cxp = op.c[2], cym = op.c[3], cyp = op.c[4], czm = op.c[5],
                 czp = op.c[6];
    auto lds2 = [](uint32_t ad) {
        double2 r;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "r"(ad));
        return r;
    };
    auto lds1 = [](uint32_t ad) {
        double r;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(r) : "r"(ad));
        return r;
    };
    auto bar_wait = [](uint32_t bar, uint32_t parity) {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "WAIT_%=:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            "@!p bra WAIT_%=;\n"
            "}\n" ::"r"(bar),
            "r"(parity)
            : "memory");
    };
    // L2 prefetch of the u-terms of pass jp for this brick: its ylen lines of a plane are contiguous, one
    // bulk prefetch per plane and term (warp t: plane t).  With one plane of register prefetch in the
    // marching loop the u loads were HBM-latency bound (16 KB in flight per SM: ~2 TB/s); from L2 the same
    // depth covers the latency
    const int ylines = min(g.ylen, ny - y0);
    auto prefetch_terms = [&](int jp) {
        if (lane == 0)
            for (int t = warp; t < zl; t += SNW)
                for (int i = 0; i < w.nz[jp - 1]; i++)
                    prefetch_rows(w.z[jp - 1][i] + (int64_t)nx * (y0 + (int64_t)ny * (z0 + t)), ylines * nx);
    };
    prefetch_terms(1);
    for (int j = 1; j <= w.p; j++) {
        double *y = ((j == w.p) ? wk.V : w.W + (int64_t)j * ldv) + row0;
        const int nzt = w.nz[j - 1];
        if (j < w.p) prefetch_terms(j + 1);
        if (!pre) {
            if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue_planes(j == 1 ? &tmx0 : &tmw, j == 1 ? 0 : j - 1);
        }
        pre = false;
        double ysq = 0.0;
#ifdef BRICK_CLK
        unsigned long long ck0 = gtimer(), ck1 = 0, ck2 = 0, ck3 = 0, ckp[TM_PAIRS] = {};
        long long ckw = 0;
#endif
        if (cnt > 0) {
            // the first u-term of the first plane is loaded before the plane wait (HBM latency)
            const double *z0p = nzt > 0 ? w.z[j - 1][0] + row0 : nullptr;
            double2 u0 = (z0p && act) ? ld_stream2(z0p) : make_double2(0.0, 0.0);
            bar_wait(pb0, par);
            bar_wait(pb0 + 8, par);
#ifdef BRICK_CLK
            ck1 = gtimer();
#endif
            double2 zm = lds2(pa0), zc = lds2(pa0 + ps8);
            uint32_t pa = pa0 + ps8;
#pragma unroll
            for (int t = 0; t < TM_PAIRS; t++) {
                if (t >= cnt) break;
                // the next plane's first u-term flies while this plane is computed
                double2 u1 = make_double2(0.0, 0.0);
                if (z0p && act && t + 1 < cnt) u1 = ld_stream2(z0p + (t + 1) * pl);
#ifdef BRICK_CLK
                const long long cw0 = clock64();
#endif
                bar_wait(pb0 + 8 * (t + 2), par);
#ifdef BRICK_CLK
                ckw += clock64() - cw0;
#endif
                const uint32_t pn = pa + ps8;
                const double2 zn = lds2(pn);
                const double2 ym = lds2(pa - ls8), yp = lds2(pa + ls8);
                const double xl = lds1(pa - 8), xh = lds1(pa + 16);
                double sa = 0.0, sb = 0.0;
                sa = __dadd_rn(sa, __dmul_rn(czm, zm.x));
                sb = __dadd_rn(sb, __dmul_rn(czm, zm.y));
                sa = __dadd_rn(sa, __dmul_rn(cym, ym.x));
                sb = __dadd_rn(sb, __dmul_rn(cym, ym.y));
                sa = __dadd_rn(sa, __dmul_rn(cxm, xl));
                sb = __dadd_rn(sb, __dmul_rn(cxm, zc.x));
                sa = __dadd_rn(sa, __dmul_rn(c0, zc.x));
                sb = __dadd_rn(sb, __dmul_rn(c0, zc.y));
                sa = __dadd_rn(sa, __dmul_rn(cxp, zc.y));
                sb = __dadd_rn(sb, __dmul_rn(cxp, xh));
                sa = __dadd_rn(sa, __dmul_rn(cyp, yp.x));
                sb = __dadd_rn(sb, __dmul_rn(cyp, yp.y));
                sa = __dadd_rn(sa, __dmul_rn(czp, zn.x));
                sb = __dadd_rn(sb, __dmul_rn(czp, zn.y));
                if (act) {
                    if (nzt > 0) {
                        const double cz0 = w.zc[j - 1][0];
                        sa = fma(cz0, u0.x, sa);
                        sb = fma(cz0, u0.y, sb);
                    }
#pragma unroll 1
                    for (int i = 1; i < nzt; i++) {
                        const double2 ui = ld_stream2(w.z[j - 1][i] + row0 + t * pl);
                        const double ci = w.zc[j - 1][i];
                        sa = fma(ci, ui.x, sa);
                        sb = fma(ci, ui.y, sb);
                    }
                    *reinterpret_cast<double2 *>(y + t * pl) = make_double2(sa, sb);
                    ysq = fma(sa, sa, ysq);
                    ysq = fma(sb, sb, ysq);
                }
                u0 = u1;
                zm = zc;
                zc = zn;
                pa = pn;
#ifdef BRICK_CLK
                ckp[t] = gtimer();
#endif
            }
        }
#ifdef BRICK_CLK
        ck2 = gtimer();
#endif
        {
            const double v1[1] = {j == w.p ? ysq : 0.0};
            block_sums<1, false>(v1, wsum, bsum);
        }
#ifdef BRICK_CLK
        ck3 = gtimer();
        if (blockIdx.x == 37 && lane == 0 && (warp & 7) == 0)
            printf("wrec j%d w%02d: start %llu planes01 +%llu p0 +%llu p1 +%llu p3 +%llu p5 +%llu march +%llu sums +%llu; plane waits %lld cycles\n",
                   j, warp, ck0 % 1000000, ck1 - ck0, ckp[0] - ck0, ckp[1] - ck0, ckp[3] - ck0, ckp[5] - ck0, ck2 - ck0,
                   ck3 - ck0, ckw);
#endif
        const bool more = j < w.p;
        if (!phase_allreduce(wk, bsum, 1, ++phase, a, red, NoRelease{}, [&] {
                if (more) issue_planes(&tmw, j);
            }))
            return;
        pre = more;
        par ^= 1u;
        if (j == w.p && blockIdx.x == 0 && tid == 0) {
            // FIN_SEED: beta = ||w_p||, sigma_0 = 1 / beta, breakdown / non-finite reset
            const double b = sqrt(red[0]);
            wk.st->beta = b;
            wk.sigma[0] = 1.0 / b;
            wk.st->brk = (b > 0.0 && isfinite(b)) ? -1 : 0;
            wk.st->nonfinite = isfinite(b) ? 0 : 1;
            wk.st->lz = 0.0;
        }
    }
    coop_exit(a);
}

} // namespace phipm
