// mm_probe.cu — cycles per Kp x Kp fp64 DMMA product on one CTA (shared memory), the expm kernel's
// cta_matmul (2 x 2 tiles of 8 x 8 per warp task) against variants:
//   V1: split-K: every 2 x 2 block is computed by two warps over half of k each, summed through smem
//   V2: 2 x 2 blocks, k loop unrolled by two (two fragment sets in flight)
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_0907_4631_b200/csrc -Iinclude \
//        -o tools/mm_probe tools/mm_probe.cu
#include "expm.cuh"

#include <cstdio>

using namespace phipm;

#define DMMA(c0, c1, a, b) \
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b))

// 2 x 2 block (bi, bj) over k in [k0, k1): accumulators c
__device__ __forceinline__ void block_k(int Kp, int ld, const double *A, const double *B, int bi, int bj, int k0, int k1,
                                        double (&c)[2][2][2], bool unroll2)
{
    const int lane = threadIdx.x & 31, nt = Kp >> 3;
    const int ar = lane >> 2, ac = lane & 3;
    const int ti0 = 2 * bi, tj0 = 2 * bj;
    const bool ri = ti0 + 1 < nt, rj = tj0 + 1 < nt;
    const double *A0 = A + (ti0 * 8 + ar) + (size_t)ac * ld;
    const double *A1 = ri ? A0 + 8 : A0;
    const double *B0 = B + ac + (size_t)(tj0 * 8 + ar) * ld;
    const double *B1 = rj ? B0 + (size_t)8 * ld : B0;
    if (!unroll2) {
        double a0 = A0[(size_t)k0 * ld], a1 = A1[(size_t)k0 * ld], b0 = B0[k0], b1 = B1[k0];
        for (int k = k0; k < k1; k += 4) {
            double na0 = 0.0, na1 = 0.0, nb0 = 0.0, nb1 = 0.0;
            if (k + 4 < k1) {
                na0 = A0[(size_t)(k + 4) * ld];
                na1 = A1[(size_t)(k + 4) * ld];
                nb0 = B0[k + 4];
                nb1 = B1[k + 4];
            }
            DMMA(c[0][0][0], c[0][0][1], a0, b0);
            DMMA(c[0][1][0], c[0][1][1], a0, b1);
            DMMA(c[1][0][0], c[1][0][1], a1, b0);
            DMMA(c[1][1][0], c[1][1][1], a1, b1);
            a0 = na0; a1 = na1; b0 = nb0; b1 = nb1;
        }
    } else {
        int k = k0;
        for (; k + 8 <= k1; k += 8) {
            const double a0 = A0[(size_t)k * ld], a1 = A1[(size_t)k * ld], b0 = B0[k], b1 = B1[k];
            const double e0 = A0[(size_t)(k + 4) * ld], e1 = A1[(size_t)(k + 4) * ld], f0 = B0[k + 4], f1 = B1[k + 4];
            DMMA(c[0][0][0], c[0][0][1], a0, b0);
            DMMA(c[0][1][0], c[0][1][1], a0, b1);
            DMMA(c[1][0][0], c[1][0][1], a1, b0);
            DMMA(c[1][1][0], c[1][1][1], a1, b1);
            DMMA(c[0][0][0], c[0][0][1], e0, f0);
            DMMA(c[0][1][0], c[0][1][1], e0, f1);
            DMMA(c[1][0][0], c[1][0][1], e1, f0);
            DMMA(c[1][1][0], c[1][1][1], e1, f1);
        }
        for (; k < k1; k += 4) {
            const double a0 = A0[(size_t)k * ld], a1 = A1[(size_t)k * ld], b0 = B0[k], b1 = B1[k];
            DMMA(c[0][0][0], c[0][0][1], a0, b0);
            DMMA(c[0][1][0], c[0][1][1], a0, b1);
            DMMA(c[1][0][0], c[1][0][1], a1, b0);
            DMMA(c[1][1][0], c[1][1][1], a1, b1);
        }
    }
}

__device__ __forceinline__ void store_block(int Kp, int ld, double *C, int bi, int bj, const double (&c)[2][2][2])
{
    const int lane = threadIdx.x & 31, nt = Kp >> 3;
    const int ar = lane >> 2, ac = lane & 3;
    const int ti0 = 2 * bi, tj0 = 2 * bj;
    const bool ri = ti0 + 1 < nt, rj = tj0 + 1 < nt;
#pragma unroll
    for (int x = 0; x < 2; x++)
#pragma unroll
        for (int y = 0; y < 2; y++) {
            if ((x && !ri) || (y && !rj)) continue;
            const int row = (ti0 + x) * 8 + ar, col = (tj0 + y) * 8 + 2 * ac;
            C[row + (size_t)col * ld] = c[x][y][0];
            C[row + (size_t)(col + 1) * ld] = c[x][y][1];
        }
}

// V1: split-K over warp pairs (task t: block t/2, k half t%2); the second half's partials go through smem
__device__ void mm_splitk(int Kp, int ld, const double *A, const double *B, double *C, double *part)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int nt = Kp >> 3, nb = (nt + 1) >> 1, nblk = nb * nb;
    const int kh = ((Kp / 4 + 1) / 2) * 4;               // first half: k < kh
    for (int task = warp; task < 2 * nblk; task += nw) {
        const int bI = task >> 1, half = task & 1;
        const int bi = bI % nb, bj = bI / nb;
        double c[2][2][2] = {};
        block_k(Kp, ld, A, B, bi, bj, half ? kh : 0, half ? Kp : kh, c, false);
        if (half) {
            double *p = part + (size_t)bI * 256 + lane * 8;
#pragma unroll
            for (int x = 0; x < 2; x++)
#pragma unroll
                for (int y = 0; y < 2; y++) {
                    p[4 * x + 2 * y] = c[x][y][0];
                    p[4 * x + 2 * y + 1] = c[x][y][1];
                }
        }
        // partner warp of the same block is task ^ 1 = warp ^ 1 when nw is even (same round)
        asm volatile("bar.sync %0, 64;" ::"r"(1 + (warp >> 1)) : "memory");
        if (!half) {
            const double *p = part + (size_t)bI * 256 + lane * 8;
#pragma unroll
            for (int x = 0; x < 2; x++)
#pragma unroll
                for (int y = 0; y < 2; y++) {
                    c[x][y][0] += p[4 * x + 2 * y];
                    c[x][y][1] += p[4 * x + 2 * y + 1];
                }
            store_block(Kp, ld, C, bi, bj, c);
        }
        asm volatile("bar.sync %0, 64;" ::"r"(1 + (warp >> 1)) : "memory");
    }
    __syncthreads();
}

__device__ void mm_unroll2(int Kp, int ld, const double *A, const double *B, double *C)
{
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int nt = Kp >> 3, nb = (nt + 1) >> 1;
    for (int bI = warp; bI < nb * nb; bI += nw) {
        const int bi = bI % nb, bj = bI / nb;
        double c[2][2][2] = {};
        block_k(Kp, ld, A, B, bi, bj, 0, Kp, c, true);
        store_block(Kp, ld, C, bi, bj, c);
    }
    __syncthreads();
}

// V3/V4: tasks of 1 x TC tiles (TC = 2 or 1), task index column-major over (tile row, column group),
// dealt round-robin to the warps (warp w on sub-partition w mod 4)
template <int TC>
__device__ void mm_fine(int Kp, int ld, const double *A, const double *B, double *C)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int nt = Kp >> 3, ng = (nt + TC - 1) / TC;
    const int ar = lane >> 2, ac = lane & 3;
    for (int task = warp; task < nt * ng; task += nw) {
        const int ti = task % nt, cg = task / nt;
        const int tj0 = cg * TC;
        const bool rj = TC == 2 && tj0 + 1 < nt;
        const double *A0 = A + (ti * 8 + ar) + (size_t)ac * ld;
        const double *B0 = B + ac + (size_t)(tj0 * 8 + ar) * ld;
        const double *B1 = rj ? B0 + (size_t)8 * ld : B0;
        double c0 = 0, c1 = 0, d0 = 0, d1 = 0;
        double a0 = A0[0], b0 = B0[0], b1 = B1[0];
        for (int k = 0; k < Kp; k += 4) {
            double na0 = 0.0, nb0 = 0.0, nb1 = 0.0;
            if (k + 4 < Kp) {
                na0 = A0[(size_t)(k + 4) * ld];
                nb0 = B0[k + 4];
                if (TC == 2) nb1 = B1[k + 4];
            }
            DMMA(c0, c1, a0, b0);
            if (TC == 2) DMMA(d0, d1, a0, b1);
            a0 = na0; b0 = nb0; b1 = nb1;
        }
        const int row = ti * 8 + ar, col = tj0 * 8 + 2 * ac;
        C[row + (size_t)col * ld] = c0;
        C[row + (size_t)(col + 1) * ld] = c1;
        if (rj) {
            C[row + (size_t)(col + 8) * ld] = d0;
            C[row + (size_t)(col + 9) * ld] = d1;
        }
    }
    __syncthreads();
}

template <int V>
__global__ void __launch_bounds__(EXPM_NT, 1) prod_kernel(int Kp, int reps, long long *cyc, double *out)
{
    extern __shared__ double sm[];
    const int ld = expm_ld(Kp);
    double *A = sm, *C = sm + (size_t)ld * Kp, *part = C + (size_t)ld * Kp;
    for (int e = threadIdx.x; e < ld * Kp; e += blockDim.x) {
        const int r = e % ld, c = e / ld;
        A[e] = (r < Kp && c < Kp) ? 1.0 / (1.0 + r + 2 * c) : 0.0;
    }
    __syncthreads();
    const long long t0 = clock64();
    for (int q = 0; q < reps; q++) {
        if (V == 0) cta_matmul(Kp, ld, A, A, C);
        else if (V == 1) mm_splitk(Kp, ld, A, A, C, part);
        else if (V == 2) mm_unroll2(Kp, ld, A, A, C);
        else if (V == 3) mm_fine<2>(Kp, ld, A, A, C);
        else mm_fine<1>(Kp, ld, A, A, C);
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    for (int e = threadIdx.x; e < ld * Kp; e += blockDim.x) out[e] = C[e];
}

int main()
{
    long long *dc;
    double *dout;
    cudaMalloc(&dc, 8);
    cudaMalloc(&dout, 8 * 160 * 160);
    double *h0 = new double[160 * 160], *h1 = new double[160 * 160];
    for (int Kp : {40, 48, 56, 64}) {
        const int ld = expm_ld(Kp);
        const size_t smem = (2 * (size_t)ld * Kp + 64 * 256) * 8;
        long long c[5];
        void (*f[5])(int, int, long long *, double *) = {prod_kernel<0>, prod_kernel<1>, prod_kernel<2>,
                                                         prod_kernel<3>, prod_kernel<4>};
        double maxdiff = 0.0;
        for (int v = 0; v < 5; v++) {
            cudaFuncSetAttribute(f[v], cudaFuncAttributeMaxDynamicSharedMemorySize, 220000);
            f[v]<<<1, EXPM_NT, smem>>>(Kp, 50, dc, dout);
            f[v]<<<1, EXPM_NT, smem>>>(Kp, 50, dc, dout);
            cudaMemcpy(&c[v], dc, 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(v == 0 ? h0 : h1, dout, 8 * ld * Kp, cudaMemcpyDeviceToHost);
            if (v > 0)
                for (int e = 0; e < ld * Kp; e++) maxdiff = fmax(maxdiff, fabs(h0[e] - h1[e]) / (1e-300 + fabs(h0[e])));
        }
        printf("Kp=%3d: cta_matmul %6.0f  splitK %6.0f  unroll2 %6.0f  1x2 %6.0f  1x1 %6.0f cycles/product  (max rel diff %.1e, %s)\n", Kp,
               c[0] / 50.0, c[1] / 50.0, c[2] / 50.0, c[3] / 50.0, c[4] / 50.0, maxdiff, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
