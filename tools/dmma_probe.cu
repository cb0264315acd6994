// dmma_probe.cu — measurement tool: fp64 mma.sync (DMMA) latency/throughput, barrier and smem
// round-trip costs inside one CTA on this B200 (guides the single-CTA expm design).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(long long *out, int iters)
{
    __shared__ double sm[4096];
    const int t = threadIdx.x, lane = t & 31;
    for (int i = t; i < 4096; i += blockDim.x) sm[i] = 1.0 + 1e-9 * i;
    __syncthreads();
    double c0 = 0, c1 = 0, d0 = 0, d1 = 0, e0 = 0, e1 = 0, f0 = 0, f1 = 0;
    const double a = sm[lane], b = sm[lane + 32];
    long long t0 = clock64();
    // 1) dependent DMMA chain (latency)
    for (int i = 0; i < iters; i++)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    long long t1 = clock64();
    // 2) four independent chains (throughput per warp)
    for (int i = 0; i < iters; i++) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(e0), "+d"(e1) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(f0), "+d"(f1) : "d"(a), "d"(b));
    }
    long long t2 = clock64();
    // 3) barrier cost
    for (int i = 0; i < iters; i++) __syncthreads();
    long long t3 = clock64();
    // 4) dependent shared-memory round trips
    int idx = lane;
    for (int i = 0; i < iters; i++) idx = (int)sm[idx & 4095] & 31;
    long long t4 = clock64();
    // 5) fp64 division latency
    double q = 1.2345;
    for (int i = 0; i < iters; i++) q = 1.0 / (q + 1.0);
    long long t5 = clock64();
    if (t == 0) {
        out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4;
    }
    if (c0 + d0 + e0 + f0 + c1 + d1 + e1 + f1 + idx + q == 12345.678) out[7] = 1;
}

int main()
{
    long long *d, h[8];
    cudaMalloc(&d, 64);
    const int iters = 256;
    for (int nt : {32, 256, 1024}) {
        probe<<<1, nt>>>(d, iters);
        probe<<<1, nt>>>(d, iters);
        cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
        printf("threads %4d: DMMA dep-chain %6.1f cyc/op | DMMA 4 chains %6.1f cyc/op-per-warp | __syncthreads %6.1f cyc | "
               "smem dep load %5.1f cyc | fp64 div %5.1f cyc\n",
               nt, (double)h[0] / iters, (double)h[1] / (4.0 * iters), (double)h[2] / iters, (double)h[3] / iters,
               (double)h[4] / iters);
    }
    return 0;
}
