// persist_wrec.cuh — the whole w-recurrence of a step (Eq. wrecurrence)
//
//   w_0 = u_k ;  w_j = A w_{j-1} + sum_l t_k^l / l! u_{j+l}   (j = 1..p) ;  w_p -> V[:, 0], ||w_p||^2
//
// for a stencil operator in ONE cooperative kernel (one 1024-thread CTA per SM).  The streaming
// path launches p spmv_stream kernels whose single halo buffer (3-D: ~200 KB per 8192-row tile)
// leaves every tile waiting for its own copy; here nothing else lives in shared memory, so two
// 4096-row halo tiles are double-buffered (tiles t+1 and t+2 fly while tile t is computed) and the
// SpMVs are separated by grid barriers instead of kernel boundaries.  The rows and the u-terms are
// those of spmv_stream (ascending-column stencil sums, then fma(c_l, u_{j+l}, y) in term order),
// so w_1..w_p equal the streaming path's bit for bit; ||w_p||^2 is summed in another order.  The
// last phase ends in an all-reduce of ||w_p||^2 whose FIN_SEED (beta, sigma_0 = 1 / beta,
// breakdown reset) CTA 0 writes, as the streaming path's last launch does.
#pragma once

#include "persist_tm.cuh"

namespace phipm {

constexpr int WREC_MAXP = 6;            // p <= p_max <= P_MAX_ABS = 6
constexpr int WREC_PLANS = 8;           // tiles per CTA with a precomputed halo plan

struct WrecArgs {
    int p;
    const double *x0;                   // w_0 = u_k (padded workspace vector, or the caller's u_0)
    int64_t ldx;                        // halo copies clamp to [0, ldx) (n when x0 is the caller's vector)
    double *W;                          // w_j at W + j ldv (j = 1..p-1); w_p goes to V column 0
    const double *z[WREC_MAXP][WREC_MAXP + 1];
    double zc[WREC_MAXP][WREC_MAXP + 1];
    int nz[WREC_MAXP];
};

__host__ __device__ inline size_t wrec_smem_bytes(int halo_cap) { return persist_tm_smem_bytes(halo_cap); }

template <int DIM>
__global__ void __launch_bounds__(SNT, 1) wrec_persist_kernel(StencilOp op, WrecArgs w, PersistArgs a, Work wk)
{
    constexpr int RPT = 4;
    constexpr int TILE_ = SNT * RPT;
    constexpr int NP = RPT / 2;
    extern __shared__ __align__(128) double sm[];
    __shared__ uint64_t hbar[2];
    __shared__ TilePlan tplan[WREC_PLANS];
    __shared__ int hofs[2][5];          // tiles beyond WREC_PLANS: offsets of the on-the-fly plan
    __shared__ double bsum[2];
    __shared__ double red[MAXD + 2];
    __shared__ double wsum[SNW];
    const int tid = threadIdx.x;
    const int64_t cs = (int64_t)blockIdx.x * a.rpc, ce = min(op.n, cs + a.rpc);
    const int hstride = (halo_capacity(op.dim, op.nx, TILE_) + 15) & ~15;
    const int64_t ldv = wk.ldv;
    const int nt = (int)((max((int64_t)0, ce - cs) + TILE_ - 1) / TILE_);
    if (tid == 0) {
        mbar_init(&hbar[0], 1);
        mbar_init(&hbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < WREC_PLANS && tid < nt) {
        const int64_t ru = cs + (int64_t)tid * TILE_;
        tile_plan<TILE_>(op, w.ldx, ru, (int)min((int64_t)TILE_, ce - ru), tplan[tid]);
    }
    const uint64_t pol = policy_evict_last();
    pdl_wait();
    __syncthreads();
    uint32_t ht = 0;
    unsigned phase = 0;
    bool pre = false;                   // the next SpMV's first tiles are in flight
    // tile u of the current vector into halo buffer g & 1 (one thread)
    auto issue = [&](int u, const double *x, uint32_t g) {
        double *hb = sm + (g & 1) * hstride;
        if (u < WREC_PLANS) {
            issue_planned_tile(tplan[u], hb, x, &hbar[g & 1], pol);
        } else {
            const int64_t ru = cs + (int64_t)u * TILE_;
            issue_halo_tile<TILE_>(op, hb, x, w.ldx, ru, (int)min((int64_t)TILE_, ce - ru), hofs[g & 1], &hbar[g & 1]);
        }
    };
    for (int j = 1; j <= w.p; j++) {
        const double *x = (j == 1) ? w.x0 : w.W + (int64_t)(j - 1) * ldv;
        double *y = (j == w.p) ? wk.V : w.W + (int64_t)j * ldv;
        const int nz = w.nz[j - 1];
        if (tid == 0 && !pre)
            for (int u = 0; u < 2 && u < nt; u++) issue(u, x, ht + u);
        pre = false;
        double ysq = 0.0;
        int3 gcoord = grid_coords(op, cs + 2 * tid);
        for (int t = 0; t < nt; t++) {
            const int64_t r0 = cs + (int64_t)t * TILE_;
            const int rows = (int)min((int64_t)TILE_, ce - r0);
            const uint32_t g = ht++;
            double2 yv[NP], xr[NP];
            // the first u-term of these rows (the only one on a step with t_k = 0) is loaded before
            // the halo wait, so its HBM latency overlaps the copy and the stencil rows
            double2 z0[NP];
#pragma unroll
            for (int p = 0; p < NP; p++) {
                const int q = 2 * tid + 2 * SNT * p;
                z0[p].x = (nz > 0 && q < rows) ? __ldg(w.z[j - 1][0] + r0 + q) : 0.0;
                z0[p].y = (nz > 0 && q + 1 < rows) ? __ldg(w.z[j - 1][0] + r0 + q + 1) : 0.0;
            }
            mbar_wait(&hbar[g & 1], (g >> 1) & 1);
            const int *ho = t < WREC_PLANS ? tplan[t].ho : hofs[g & 1];
            stencil_tile_d<NP, (DIM == 4 ? 2 : DIM), (DIM == 4)>(op, sm + (g & 1) * hstride, ho, r0, rows, tid, yv,
                                                                 xr, &gcoord);
            __syncthreads();                               // halo buffer g & 1 consumed
            if (tid == 0 && t + 2 < nt) issue(t + 2, x, g + 2);
#pragma unroll
            for (int p = 0; p < NP; p++) {
                const int q = 2 * tid + 2 * SNT * p;
                const int64_t r = r0 + q;
                if (nz > 0) {
                    const double c0 = w.zc[j - 1][0];
                    if (q < rows) yv[p].x = fma(c0, z0[p].x, yv[p].x);
                    if (q + 1 < rows) yv[p].y = fma(c0, z0[p].y, yv[p].y);
                }
                for (int i = 1; i < nz; i++) {
                    const double *zi = w.z[j - 1][i];
                    const double ci = w.zc[j - 1][i];
                    if (q < rows) yv[p].x = fma(ci, __ldg(zi + r), yv[p].x);
                    if (q + 1 < rows) yv[p].y = fma(ci, __ldg(zi + r + 1), yv[p].y);
                }
                double *o = y + r;
                if (q + 1 < rows) *reinterpret_cast<double2 *>(o) = yv[p];
                else if (q < rows) o[0] = yv[p].x;
                ysq = fma(yv[p].x, yv[p].x, ysq);
                ysq = fma(yv[p].y, yv[p].y, ysq);
            }
        }
        // grid phase: w_j visible to every CTA's next halo copies; after the last SpMV also ||w_p||^2
        {
            const double v1[1] = {j == w.p ? ysq : 0.0};
            block_sums<1, false>(v1, wsum, bsum);
        }
        // w_j is complete in every CTA once the arrivals are in: the next SpMV's first halo tiles are
        // issued by the last warp while the partials are summed
        const bool more = j < w.p;
        if (!phase_allreduce(wk, bsum, 1, ++phase, a, red, [&] {
                if (more)
                    for (int u = 0; u < 2 && u < nt; u++) issue(u, y, ht + u);
            }))
            return;
        pre = more;
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
