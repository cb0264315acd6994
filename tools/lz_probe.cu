// lz_probe.cu — where do the cycles of one single-CTA Lanczos step go (c1: n = 1000, 1-D tridiagonal)?
// Variants of the step loop of krylov_small_lanczos_kernel, timed with clock64 over S steps:
//   NT threads, R = ceil(n / NT) rows per thread (r = t + NT i), two block sums per step,
//   SECOND: 0 full 5-level second stage, 1 log2(nwarps) levels
//   DIV: 0 IEEE sqrt + divide, 1 rsqrt-based (one Newton step on MUFU.RSQ64H)
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/lz_probe tools/lz_probe.cu
#include <cstdio>
#include <cmath>
#include <vector>

__device__ __forceinline__ double wsum(double v, int lv)
{
    for (int o = 16; o >= (32 >> lv); o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int NT, int R, int SECOND, int DIV>
__global__ void __launch_bounds__(NT) probe(const double *v0, double *V, int n, int S, double c0, double c1,
                                            long long *cyc, double *out)
{
    extern __shared__ double vs[];
    __shared__ double red[2][32];
    constexpr int NW = NT / 32;
    constexpr int L2 = (NW <= 1) ? 0 : (NW <= 2) ? 1 : (NW <= 4) ? 2 : (NW <= 8) ? 3 : (NW <= 16) ? 4 : 5;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    double zv[R];
    for (int i = 0; i < R; i++) {
        const int r = t + NT * i;
        zv[i] = 0.0;
        if (r < n) vs[r] = v0[r];
    }
    __syncthreads();
    double sj = 1.0, lz = 0.0;
    long long c_start = clock64();
    for (int j = 0; j < S; j++) {
        double y[R], xv[R];
        double dl = 0.0;
#pragma unroll
        for (int i = 0; i < R; i++) {
            const int r = t + NT * i;
            y[i] = 0.0;
            xv[i] = 0.0;
            if (r < n) {
                double s = 0.0;
                if (r > 0) s = __dadd_rn(s, __dmul_rn(c1, vs[r - 1]));
                s = __dadd_rn(s, __dmul_rn(c0, vs[r]));
                if (r < n - 1) s = __dadd_rn(s, __dmul_rn(c1, vs[r + 1]));
                y[i] = sj * s;
                xv[i] = vs[r];
                if (j > 0) y[i] = fma(-lz, zv[i], y[i]);
            }
            dl = fma(xv[i], y[i], dl);
        }
        double d;
        if (NW == 1) {
            d = wsum(dl, 5);
        } else {
            dl = wsum(dl, 5);
            if (lane == 0) red[0][warp] = dl;
            __syncthreads();
            d = SECOND ? wsum(lane < NW ? red[0][lane] : 0.0, L2) : wsum(lane < NW ? red[0][lane] : 0.0, 5);
        }
        const double al = sj * d;
        const double g = al * sj;
        double wl = 0.0;
#pragma unroll
        for (int i = 0; i < R; i++) {
            const int r = t + NT * i;
            if (r < n) {
                const double w = fma(-g, xv[i], y[i]);
                V[(long long)(j + 1) * 1024 + r] = w;
                vs[r] = w;
                wl = fma(w, w, wl);
            }
            zv[i] = xv[i];
        }
        if (NW == 1) __syncwarp();
        double tot;
        if (NW == 1) {
            tot = wsum(wl, 5);
        } else {
            wl = wsum(wl, 5);
            if (lane == 0) red[1][warp] = wl;
            __syncthreads();
            tot = SECOND ? wsum(lane < NW ? red[1][lane] : 0.0, L2) : wsum(lane < NW ? red[1][lane] : 0.0, 5);
        }
        double h, sn;
        if (DIV) {
            // sn = rsqrt(tot) refined once, h = tot * sn
            double r0;
            asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(tot));
            const double e = fma(-tot * r0, r0, 1.0);
            sn = fma(0.5 * r0, e, r0);
            h = tot * sn;
        } else {
            h = sqrt(tot);
            sn = 1.0 / h;
        }
        const double lzn = h * sj;
        if (t == 0) out[j] = al + h;
        sj = sn;
        lz = lzn;
    }
    long long c_end = clock64();
    if (t == 0) cyc[0] = c_end - c_start;
}

template <int NT, int SECOND, int DIV>
void run(const char *name, const double *dv, double *dV, int n, int S, long long *dc, double *dout)
{
    constexpr int R = (1000 + NT - 1) / NT;
    probe<NT, R, SECOND, DIV><<<1, NT, n * 8>>>(dv, dV, n, S, -2.0, 1.0, dc, dout);
    cudaDeviceSynchronize();
    long long best = 1LL << 60;
    for (int rep = 0; rep < 5; rep++) {
        probe<NT, R, SECOND, DIV><<<1, NT, n * 8>>>(dv, dV, n, S, -2.0, 1.0, dc, dout);
        long long c;
        cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        if (c < best) best = c;
    }
    printf("%-28s NT=%4d R=%2d second=%d div=%d : %7.0f cycles/step\n", name, NT, R, SECOND, DIV, (double)best / S);
}

int main()
{
    const int n = 1000, S = 64;
    std::vector<double> h(n);
    for (int i = 0; i < n; i++) h[i] = sin(0.01 * i) + 1.0;
    double *dv, *dV, *dout;
    long long *dc;
    cudaMalloc(&dv, n * 8);
    cudaMalloc(&dV, 1024 * 8 * (S + 2));
    cudaMalloc(&dout, 8 * S);
    cudaMalloc(&dc, 8);
    cudaMemcpy(dv, h.data(), n * 8, cudaMemcpyHostToDevice);
    run<256, 0, 0>("current (SLZ)", dv, dV, n, S, dc, dout);
    run<256, 1, 0>("short 2nd stage", dv, dV, n, S, dc, dout);
    run<256, 1, 1>("short + rsqrt", dv, dV, n, S, dc, dout);
    run<128, 1, 1>("", dv, dV, n, S, dc, dout);
    run<64, 1, 1>("", dv, dV, n, S, dc, dout);
    run<32, 1, 1>("one warp", dv, dV, n, S, dc, dout);
    run<32, 1, 0>("one warp ieee", dv, dV, n, S, dc, dout);
    run<512, 1, 1>("", dv, dV, n, S, dc, dout);
    run<1024, 1, 1>("", dv, dV, n, S, dc, dout);
    run<1024, 0, 0>("1024 current", dv, dV, n, S, dc, dout);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
