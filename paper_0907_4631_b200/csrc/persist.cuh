// persist.cuh — the whole Krylov extension k0 -> k1 of a stencil operator in ONE cooperative kernel
// (Alg. 1 in CGS form / Alg. 2), one 1024-thread CTA per SM, for n > SMALL_N.
//
// Per step j the two-kernel path (spmv_stream + axpy_stream) pays two launch boundaries and the
// y round trip through L2.  Here every CTA keeps the y of its contiguous row range in shared
// memory between the SpMV phase and the update phase, and each phase ends in a grid all-reduce:
//   phase A  y = sigma_j A v~_j [- lz v~_{j-1}] (halo tiles by TMA), d_k = v~_k^T y, ||y||^2
//   phase B  v~_{j+1} = y - sum_k g_k v~_k (columns in descending order), ||v~_{j+1}||^2
// Phase end: every CTA publishes its partials, arrives on a monotonic counter (release) and, once
// all CTAs arrived (acquire), sums the partials itself in the fixed block order, so every CTA holds
// bit-identical totals and derives H, g, sigma and the breakdown decision locally; CTA 0 writes
// them to global memory for the exponential.  (A last-CTA reduction + flag release costs 3.3-4.5
// us per phase; the all-reduce 1.5 us, tools/kclock.py.)  Co-residency of all CTAs is guaranteed by
// the cooperative launch; a CTA that waits longer than timeout_ns sets an abort flag (every waiter
// then exits and the solve reports PHIPM_ECUDA) instead of hanging the GPU.
// The arithmetic per row, per thread, per warp and per block is that of spmv_stream/axpy_stream.
#pragma once

#include <type_traits>

#include "stream.cuh"

namespace phipm {

struct PersistArgs {
    int k0, k1;
    int symmetric;
    double bthr;
    int64_t rpc;                   // rows per CTA (balanced contiguous ranges, multiple of 32)
    unsigned *flag;                // arrival counter (CTAs x phases, monotonic within a launch)
    unsigned *abort;               // set by a CTA that timed out
    unsigned *exit_ctr;            // CTAs that left; the last one zeroes flag and exit_ctr for the next launch
    unsigned long long timeout_ns;
    unsigned long long *dbg;       // optional (PHIPM_KCLOCKS): per phase, per CTA: body end, release seen
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_u32(unsigned *p, unsigned v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// L2-coherent 16-B load (columns written earlier in this same kernel must not come from the
// non-coherent read-only path)
__device__ __forceinline__ double2 ld_cg2(const double *p)
{
    double2 r;
    asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}

// End of a grid phase as an all-reduce: every CTA writes its nv partials (buffer = phase parity,
// so a fast CTA's next partials never overwrite ones a slow CTA is still summing), arrives on the
// monotonic counter (release), waits until all gridDim.x CTAs of this phase arrived (acquire), and
// then sums the partials itself in block order: every CTA obtains bit-identical totals in red[]
// without a serialising last-CTA reduction and flag round trip.  Returns false on abort.
// End of a cooperative launch (normal exit): the last CTA to leave zeroes the arrival counter, so the
// next cooperative launch on the stream needs no memset node before it.  Every CTA has passed its last
// grid phase when it gets here, so no CTA can still be polling the counter.
__device__ __forceinline__ void coop_exit(const PersistArgs &a)
{
    if (threadIdx.x == 0) {
        const unsigned old = atomicAdd(a.exit_ctr, 1u);
        if (old == gridDim.x - 1) {
            *(volatile unsigned *)a.flag = 0u;
            *(volatile unsigned *)a.exit_ctr = 0u;
        }
    }
}

struct NoRelease {
    __device__ void operator()() const {}
};

// on_release: run by the last warp's lane 0 once every CTA has arrived, while warps 0.. nv-1 sum the
// partials (e.g. to issue the next phase's first bulk copies off the critical path)
// on_release_warps: run by lane 0 of EVERY warp at the same point (work that is spread over the warps,
// e.g. one bulk tensor copy each); both hooks run after a proxy fence for the other CTAs' writes
template <class OnRelease = NoRelease, class OnReleaseWarps = NoRelease>
__device__ __forceinline__ bool phase_allreduce(const Work &wk, const double *bsum, int nv, unsigned phase,
                                                const PersistArgs &a, double *red, OnRelease on_release = OnRelease{},
                                                OnReleaseWarps on_release_warps = OnReleaseWarps{})
{
    __shared__ int s_ok;
    const int nb = gridDim.x;
    const size_t half = (size_t)(phase & 1) * nb;
    if (a.dbg && threadIdx.x == 0) a.dbg[((size_t)(phase - 1) * gridDim.x + blockIdx.x) * 2] = gtimer();
    // (bsum is visible to every thread on entry) thread 0 writes the partials itself, so the release
    // that follows covers them in program order: no CTA barrier between the stores and the arrival
    if (threadIdx.x == 0) {
        for (int v = 0; v < nv; v++) wk.part[(size_t)v * wk.pstride + half + blockIdx.x] = bsum[v];
        int ok = 1;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.flag) : "memory");
        const unsigned target = phase * (unsigned)nb;
        const unsigned long long t0 = gtimer();
        // the abort flag and the clock are looked at every 16th poll only: a volatile load per
        // iteration doubles the poll period (two dependent L2 round trips)
        for (unsigned it = 1; ld_acquire_u32(a.flag) < target; it++) {
            if (it & 15) continue;
            if (*(volatile unsigned *)a.abort) { ok = 0; break; }
            if (gtimer() - t0 > a.timeout_ns) {
                atomicExch(a.abort, 1u);
                wk.st->aborted = 1;
                ok = 0;
                break;
            }
        }
        // the other CTAs' generic-proxy writes (acquired above) before this thread's TMA reads
        asm volatile("fence.proxy.async.global;" ::: "memory");
        s_ok = ok;
        if (a.dbg) a.dbg[((size_t)(phase - 1) * gridDim.x + blockIdx.x) * 2 + 1] = gtimer();
    }
    __syncthreads();
    if (!s_ok) return false;
    // fixed-order sum of the nb partials of each value (one warp per value, 8 loads in flight per lane)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (threadIdx.x == blockDim.x - 32) {
        // the other CTAs' generic-proxy writes were acquired by thread 0 and ordered for this thread by
        // the barrier above; its own bulk copies read them through the async proxy
        asm volatile("fence.proxy.async.global;" ::: "memory");
        on_release();
    }
    if constexpr (!std::is_same<OnReleaseWarps, NoRelease>::value) {
        if ((threadIdx.x & 31) == 0) {
            // (the shared-memory reads of the previous phase by this CTA's generic proxy, and the other
            // CTAs' global writes acquired by thread 0 and ordered by the barrier above)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        on_release_warps();
    }
    for (int v = warp; v < nv; v += nw) {
        const double *pv = wk.part + (size_t)v * wk.pstride + half;
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
        double t = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
        t = warp_sum(t);
        if (lane == 0) red[v] = t;
    }
    __syncthreads();
    return true;
}

// dynamic shared memory (bytes): halo tile, y of the CTA's rows, per-warp dot partials
__host__ __device__ inline size_t persist_smem_bytes(int halo_cap, int64_t rpc, int ndmax)
{
    return ((size_t)((halo_cap + 15) & ~15) + (size_t)((rpc + 15) & ~(int64_t)15) + (size_t)ndmax * SNW) *
           sizeof(double);
}

// LANC: Lanczos (symmetric) or Arnoldi; DIM: 1, 2, 3 or 4 (= 2-D 9-point) -- compile-time, so each
// instantiation carries only its own stencil and orthogonalisation code (registers, no spills)
template <int RPT, bool LANC, int DIM>
__global__ void __launch_bounds__(SNT, 1) krylov_persist_kernel(StencilOp op, PersistArgs a, Work wk)
{
    constexpr int TILE_ = SNT * RPT;
    constexpr int NP = RPT / 2;
    extern __shared__ __align__(128) double sm[];
    __shared__ uint64_t hbar;
    __shared__ int hofs[2][5];
    __shared__ double bsum[MAXD + 2];
    __shared__ double red[MAXD + 2];
    __shared__ double wsum[SNW];
    __shared__ double gco[MAXD + 2];
    __shared__ int s_stop;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = op.n;
    const int64_t cs = (int64_t)blockIdx.x * a.rpc, ce = min(n, cs + a.rpc);
    const int hcap = halo_capacity(op.dim, op.nx, TILE_);
    double *hbuf = sm;
    double *ys = sm + ((hcap + 15) & ~15);
    double *lacc = ys + ((a.rpc + 15) & ~(int64_t)15);
    const int64_t ldv = wk.ldv;
    if (tid == 0) {
        mbar_init(&hbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    pdl_wait();                                            // the previous kernel's results from here on
    __syncthreads();
    uint32_t ht = 0;
    unsigned phase = 0;
    // state carried between steps in shared memory (every CTA derives it from identical totals;
    // CTA 0 also writes it to global memory for the exponential and the next extension)
    __shared__ double s_sig, s_lz;
    if (tid == 0) {
        s_stop = __ldcg(&wk.st->brk) >= 0;
        s_sig = __ldcg(wk.sigma + a.k0);
        s_lz = __ldcg(&wk.st->lz);
    }
    __syncthreads();
    const bool lead = blockIdx.x == 0;
    const int3 gc0 = grid_coords(op, cs + 2 * tid);       // grid coordinates of this thread's first row
    bool pre = false;                                      // the next step's first halo tile is in flight
    double sig_r = s_sig, lz_r = s_lz;                     // per-thread copies of the carried state
    bool stop_r = s_stop != 0;
    for (int j = a.k0; j < a.k1; j++) {
        if (stop_r) break;                                 // breakdown (same decision in every CTA)
        const double *x = wk.V + (int64_t)j * ldv;
        const double sj = sig_r;                           // sigma_j
        constexpr bool lanc = LANC;
        const double *zv = (lanc && j > 0) ? x - ldv : nullptr;
        const double lz = zv ? lz_r : 0.0;
        const int c0 = lanc ? j : 0;
        const int nd = j - c0 + 1;                         // dot columns c0..j; column j is x

        // ---------------- phase A: y = sigma_j A x [- lz v~_{j-1}], dots, ||y||^2
        if (tid == 0 && cs < ce && !pre)
            issue_halo_tile<TILE_>(op, hbuf, x, ldv, cs, (int)min((int64_t)TILE_, ce - cs), hofs[ht & 1], &hbar);
        pre = false;
        for (int i = tid; i < nd * SNW; i += SNT) lacc[i] = 0.0;
        __syncthreads();
        double ysq = 0.0;
        int3 gcoord = gc0;
        for (int64_t r0 = cs; r0 < ce; r0 += TILE_) {
            const int rows = (int)min((int64_t)TILE_, ce - r0);
            const int64_t r1 = r0 + TILE_;
            double2 y[NP], xr[NP];
            mbar_wait(&hbar, ht & 1);
            const int *ho = hofs[ht & 1];
            ht++;
            stencil_tile_d<NP, (DIM == 4 ? 2 : DIM), (DIM == 4)>(op, hbuf, ho, r0, rows, tid, y, xr, &gcoord);
            __syncthreads();                               // halo consumed
            if (tid == 0 && r1 < ce)
                issue_halo_tile<TILE_>(op, hbuf, x, ldv, r1, (int)min((int64_t)TILE_, ce - r1), hofs[ht & 1], &hbar);
#pragma unroll
            for (int p = 0; p < NP; p++) {
                const int q = 2 * tid + 2 * SNT * p;
                const int64_t r = r0 + q;
                y[p].x *= sj;
                y[p].y *= sj;
                double *yp = ys + (r - cs);
                if (zv) {
                    // Lanczos: after the first step of this launch, v~_{j-1} of this thread's rows is
                    // in shared memory (kept by phase B of the previous step), not re-read from HBM
                    const bool zs = j > a.k0;
                    if (q < rows) y[p].x = fma(-lz, zs ? yp[0] : __ldcg(zv + r), y[p].x);
                    if (q + 1 < rows) y[p].y = fma(-lz, zs ? yp[1] : __ldcg(zv + r + 1), y[p].y);
                }
                if (q + 1 < rows) *reinterpret_cast<double2 *>(yp) = y[p];
                else if (q < rows) yp[0] = y[p].x;
                ysq = fma(y[p].x, y[p].x, ysq);
                ysq = fma(y[p].y, y[p].y, ysq);
            }
            // dot with v~_j = x from the tile values in registers
            {
                double d = 0.0;
#pragma unroll
                for (int p = 0; p < NP; p++) {
                    d = fma(xr[p].x, y[p].x, d);
                    d = fma(xr[p].y, y[p].y, d);
                }
                d = warp_sum(d);
                if (lane == 0) lacc[(nd - 1) * SNW + warp] += d;
            }
            // Arnoldi: the other columns 0..j-1, CU in flight, ascending
            for (int k0 = 0; k0 < nd - 1; k0 += CU) {
                double2 v[CU][NP];
#pragma unroll
                for (int u = 0; u < CU; u++) {
                    const int k = k0 + u;
                    const bool ld = k < nd - 1;
                    const double *vc = wk.V + (int64_t)(c0 + (ld ? k : k0)) * ldv + r0;
#pragma unroll
                    for (int p = 0; p < NP; p++) {
                        const int q = 2 * tid + 2 * SNT * p;
                        v[u][p] = (ld && q < rows) ? ld_cg2(vc + q) : make_double2(0.0, 0.0);
                    }
                }
#pragma unroll
                for (int u = 0; u < CU; u++) {
                    double d = 0.0;
#pragma unroll
                    for (int p = 0; p < NP; p++) {
                        d = fma(v[u][p].x, y[p].x, d);
                        d = fma(v[u][p].y, y[p].y, d);
                    }
                    d = warp_sum(d);
                    if (lane == 0 && k0 + u < nd - 1) lacc[(k0 + u) * SNW + warp] += d;
                }
            }
        }
        {
            // the dot partials per warp (lacc) and ||y||^2 per warp (wsum): warp k reduces value k with
            // a shuffle tree (all values in parallel, no serial 32-term loop)
            const double v = warp_sum(ysq);
            if (lane == 0) wsum[warp] = v;
            __syncthreads();
            for (int k = warp; k <= nd; k += SNW) {
                const double x = (lane < SNW) ? (k < nd ? lacc[k * SNW + lane] : wsum[lane]) : 0.0;
                const double t = warp_sum(x);
                if (lane == 0) bsum[k] = t;
            }
        }
        __syncthreads();
        if (!phase_allreduce(wk, bsum, nd + 1, ++phase, a, red)) return;
        // finalize (FIN_ARNOLDI / FIN_LANCZOS): h_k = sigma_k d_k, g_k = h_k sigma_k
        // (Lanczos: every thread derives the one coefficient from the all-reduced totals, no barrier)
        double cf_l = 0.0;
        if constexpr (LANC) {
            const double al = sj * red[0];
            cf_l = -(al * sj);
            if (lead && tid == 0) {
                wk.H[j + (size_t)j * wk.ldh] = al;
                wk.g[0] = al * sj;
                wk.st->wnorm2 = red[1];
            }
        } else {
            for (int k = tid; k < nd; k += SNT) {
                const double sk = (k == j) ? sj : __ldcg(wk.sigma + k);
                const double h = sk * red[k];
                gco[k] = -(h * sk);
                if (lead) {
                    wk.H[k + (size_t)j * wk.ldh] = h;
                    wk.g[k] = h * sk;
                }
            }
            if (lead && tid == 0) wk.st->wnorm2 = red[nd];
            __syncthreads();                               // gco[] of every column
        }

        // ---------------- phase B: v~_{j+1} = y - sum_k g_k v~_k, ||v~_{j+1}||^2
        double *vn = wk.V + (int64_t)(j + 1) * ldv;
        double nrm = 0.0;
        for (int64_t r0 = cs; r0 < ce; r0 += TILE_) {
            const int rows = (int)min((int64_t)TILE_, ce - r0);
            double2 acc[NP];
#pragma unroll
            for (int p = 0; p < NP; p++) {
                const int q = 2 * tid + 2 * SNT * p;
                const double *yp = ys + (r0 - cs) + q;
                acc[p] = q + 1 < rows ? *reinterpret_cast<const double2 *>(yp)
                                      : make_double2(q < rows ? yp[0] : 0.0, 0.0);
            }
            double2 vkeep[NP];                             // Lanczos: v~_j of these rows, for the next step
            if (lanc) {
                // one column (v~_j): no batching arithmetic
                const double cf = cf_l;
                const double *vc = wk.V + (int64_t)c0 * ldv + r0;
#pragma unroll
                for (int p = 0; p < NP; p++) {
                    const int q = 2 * tid + 2 * SNT * p;
                    vkeep[p] = q < rows ? ld_cg2(vc + q) : make_double2(0.0, 0.0);
                }
#pragma unroll
                for (int p = 0; p < NP; p++) {
                    acc[p].x = fma(cf, vkeep[p].x, acc[p].x);
                    acc[p].y = fma(cf, vkeep[p].y, acc[p].y);
                }
            }
            for (int i0 = 0; !lanc && i0 < nd; i0 += CU) {
                double2 v[CU][NP];
#pragma unroll
                for (int u = 0; u < CU; u++) {
                    const int it = i0 + u;
                    const int kc = nd - 1 - (it < nd ? it : i0);     // descending columns
                    const double *vc = wk.V + (int64_t)(c0 + kc) * ldv + r0;
#pragma unroll
                    for (int p = 0; p < NP; p++) {
                        const int q = 2 * tid + 2 * SNT * p;
                        v[u][p] = (it < nd && q < rows) ? ld_cg2(vc + q) : make_double2(0.0, 0.0);
                    }
                }
#pragma unroll
                for (int u = 0; u < CU; u++) {
                    const int it = i0 + u;
                    const double cf = it < nd ? gco[nd - 1 - it] : 0.0;
#pragma unroll
                    for (int p = 0; p < NP; p++) {
                        acc[p].x = fma(cf, v[u][p].x, acc[p].x);
                        acc[p].y = fma(cf, v[u][p].y, acc[p].y);
                    }
                }
            }
            if (lanc) {
                // y of these rows is consumed: keep v~_j (column j, the only Lanczos column) instead
#pragma unroll
                for (int p = 0; p < NP; p++) {
                    const int q = 2 * tid + 2 * SNT * p;
                    double *yp = ys + (r0 - cs) + q;
                    if (q + 1 < rows) *reinterpret_cast<double2 *>(yp) = vkeep[p];
                    else if (q < rows) yp[0] = vkeep[p].x;
                }
            }
#pragma unroll
            for (int p = 0; p < NP; p++) {
                const int q = 2 * tid + 2 * SNT * p;
                double *o = vn + r0 + q;
                if (q + 1 < rows) *reinterpret_cast<double2 *>(o) = acc[p];
                else if (q < rows) o[0] = acc[p].x;
                if (q < rows) nrm = fma(acc[p].x, acc[p].x, nrm);
                if (q + 1 < rows) nrm = fma(acc[p].y, acc[p].y, nrm);
            }
        }
        {
            const double v = warp_sum(nrm);
            if (lane == 0) wsum[warp] = v;
            __syncthreads();
            if (warp == 0) {
                const double t = warp_sum(lane < SNW ? wsum[lane] : 0.0);
                if (lane == 0) bsum[0] = t;
            }
            __syncthreads();
        }
        // the next step's first halo tile (the halo buffer is idle in this phase) is issued by the last
        // warp as soon as every CTA has published v~_{j+1}, while the partials are summed
        const bool more = j + 1 < a.k1 && cs < ce;
        if (!phase_allreduce(wk, bsum, 1, ++phase, a, red, [&] {
                if (more)
                    issue_halo_tile<TILE_>(op, hbuf, vn, ldv, cs, (int)min((int64_t)TILE_, ce - cs), hofs[ht & 1],
                                           &hbar);
            }))
            return;
        pre = more;
        // finalize (FIN_NORM): h_{j+1,j}, sigma_{j+1}, the Lanczos coefficient, breakdown -- derived by
        // every thread from the all-reduced total (no CTA barrier)
        {
            const double h = sqrt(red[0]);
            const double sn = 1.0 / h;
            const double lzn = h * sj;
            int brk = -1, nonfin = 0;
            if (!isfinite(h)) { nonfin = 1; brk = j + 1; }
            else if (h <= a.bthr) brk = j + 1;
            sig_r = sn;
            lz_r = lzn;
            stop_r = brk >= 0;
            if (lead && tid == 0) {
                wk.H[(j + 1) + (size_t)j * wk.ldh] = h;
                if (lanc) {
                    if (j + 1 < wk.hcols) wk.H[j + (size_t)(j + 1) * wk.ldh] = h;
                    wk.st->lz = lzn;
                }
                wk.sigma[j + 1] = sn;
                if (nonfin) wk.st->nonfinite = 1;
                if (brk >= 0) wk.st->brk = brk;
            }
        }
    }
    // a first tile issued for a step that did not run (breakdown): land it before the CTA exits
    if (pre) mbar_wait(&hbar, ht & 1);
    coop_exit(a);
}

} // namespace phipm
