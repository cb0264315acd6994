// fp64 CUDA-core latency / throughput probe (DFMA dependent chain, independent chains, 1-32 warps per SM)
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void dfma_kernel(double *out, long long *cyc, int iters, double a, double b)
{
    double x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; i++) x[i] = threadIdx.x * 1e-3 + i;
    __syncthreads();
    long long t0 = clock64();
    for (int k = 0; k < iters; k++) {
#pragma unroll
        for (int i = 0; i < ILP; i++) x[i] = fma(x[i], a, b);
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; i++) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void ffma_kernel(float *out, long long *cyc, int iters, float a, float b)
{
    float x[8];
    for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 1e-3f + i;
    __syncthreads();
    long long t0 = clock64();
    for (int k = 0; k < iters; k++)
#pragma unroll
        for (int i = 0; i < 8; i++) x[i] = fmaf(x[i], a, b);
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; i++) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main()
{
    double *out;
    float *outf;
    long long *cyc, h;
    cudaMalloc(&out, 1 << 20);
    cudaMalloc(&outf, 1 << 20);
    cudaMalloc(&cyc, 1024);
    const int iters = 4096;
    for (int warps : {1, 4, 8, 16, 32}) {
        dfma_kernel<1><<<1, 32 * warps>>>(out, cyc, iters, 0.999, 1e-3);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("DFMA chain ILP1 warps=%2d: %.2f cycles per dependent DFMA\n", warps, (double)h / iters);
        dfma_kernel<8><<<1, 32 * warps>>>(out, cyc, iters, 0.999, 1e-3);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("DFMA ILP8       warps=%2d: %.2f cycles per 8 DFMA per warp -> %.2f DFMA lanes/clk/SM\n", warps,
               (double)h / iters, 8.0 * 32 * warps * iters / (double)h);
        ffma_kernel<<<1, 32 * warps>>>(outf, cyc, iters, 0.999f, 1e-3f);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("FFMA ILP8       warps=%2d: %.2f cycles per 8 FFMA per warp -> %.2f FFMA lanes/clk/SM\n", warps,
               (double)h / iters, 8.0 * 32 * warps * iters / (double)h);
    }
    return 0;
}
