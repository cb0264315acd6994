// barrier_probe.cu — measurement tool: latency of a grid-wide all-reduce of nv doubles between the
// 148 co-resident CTAs of a cooperative launch, two ways:
//   (a) counter: partials to global, red.release on one counter, ld.acquire poll, load partials
//       (the scheme of persist.cuh: phase_allreduce);
//   (b) inbox: every CTA stores its partial, as {tag, 32-bit half} 8-byte words, into every CTA's
//       own inbox; each CTA polls only its inbox (one warp), then sums in block order;
//   (c) lean counter: warp 0 alone publishes, polls, loads and sums (one CTA barrier per phase).
// Measured on this pool: (a) 2.2 us, (b) 6.5-10.8 us, (c) 2.1 us (nv = 1) per phase.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier_probe tools/barrier_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ double warp_sum(double v)
{
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void probe_counter(unsigned *flag, double *part, int iters, int nv, double *out, long long *cyc)
{
    __shared__ double red[8];
    const int nb = gridDim.x;
    long long t0 = clock64();
    for (int it = 1; it <= iters; it++) {
        const size_t half = (size_t)(it & 1) * nb * 8;
        if (threadIdx.x < nv) part[half + (size_t)threadIdx.x * nb + blockIdx.x] = blockIdx.x + it + threadIdx.x;
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(flag) : "memory");
            while (ld_acq(flag) < (unsigned)(it * nb)) {
            }
        }
        __syncthreads();
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (warp < nv) {
            double acc = 0.0;
            for (int b = lane; b < nb; b += 32) acc += __ldcg(part + half + (size_t)warp * nb + b);
            acc = warp_sum(acc);
            if (lane == 0) red[warp] = acc;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        cyc[blockIdx.x] = clock64() - t0;
        out[blockIdx.x] = red[0];
    }
}

// (c) counter, lean: warp 0 alone publishes (lane 0: partials + red.release), polls, loads and sums
// the partials; one CTA barrier per phase instead of three
__global__ void probe_lean(unsigned *flag, double *part, int iters, int nv, double *out, long long *cyc)
{
    __shared__ double red[8];
    const int nb = gridDim.x;
    long long t0 = clock64();
    for (int it = 1; it <= iters; it++) {
        const size_t half = (size_t)(it & 1) * nb * 8;
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            if (lane == 0) {
                for (int v = 0; v < nv; v++) part[half + (size_t)v * nb + blockIdx.x] = blockIdx.x + it + v;
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(flag) : "memory");
                while (ld_acq(flag) < (unsigned)(it * nb)) {
                }
            }
            __syncwarp();
            for (int v = 0; v < nv; v++) {
                double acc = 0.0;
                for (int b = lane; b < nb; b += 32) acc += __ldcg(part + half + (size_t)v * nb + b);
                acc = warp_sum(acc);
                if (lane == 0) red[v] = acc;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        cyc[blockIdx.x] = clock64() - t0;
        out[blockIdx.x] = red[0];
    }
}

// inbox[b] of CTA b: parity x nb x (2 nv) words
__global__ void probe_inbox(unsigned long long *inbox, int iters, int nv, double *out, long long *cyc)
{
    __shared__ unsigned st32[8 * 2 * 160];
    __shared__ double red[8];
    const int nb = gridDim.x, W = 2 * nv;
    const size_t per = (size_t)nb * W;                   // words per inbox per parity
    long long t0 = clock64();
    for (int it = 1; it <= iters; it++) {
        const unsigned long long tag = (unsigned long long)(unsigned)it << 32;
        const size_t par = (size_t)(it & 1) * nb * per;
        // writers: warp 1; lane l stores to inboxes l, l+32, ... this CTA's W words each
        if ((threadIdx.x >> 5) == 1) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            for (int dst = threadIdx.x & 31; dst < nb; dst += 32)
                for (int k = 0; k < W; k++) {
                    const double v = (double)(blockIdx.x + it + (k >> 1));
                    const unsigned pay = (k & 1) ? (unsigned)__double2hiint(v) : (unsigned)__double2loint(v);
                    unsigned long long *p = inbox + par + (size_t)dst * per + (size_t)blockIdx.x * W + k;
                    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(tag | pay) : "memory");
                }
        }
        // reader: warp 0 polls this CTA's inbox
        if ((threadIdx.x >> 5) == 0) {
            const unsigned long long *my = inbox + par + (size_t)blockIdx.x * per;
            for (int i = threadIdx.x; i < (int)per; i += 32) {
                unsigned long long x;
                do {
                    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(my + i) : "memory");
                } while ((x & 0xffffffff00000000ull) != tag);
                const int b = i / W, k = i - b * W;
                st32[k * nb + b] = (unsigned)x;
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        __syncthreads();
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (warp < nv) {
            double acc = 0.0;
            for (int b = lane; b < nb; b += 32)
                acc += __hiloint2double((int)st32[(2 * warp + 1) * nb + b], (int)st32[(2 * warp) * nb + b]);
            acc = warp_sum(acc);
            if (lane == 0) red[warp] = acc;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        cyc[blockIdx.x] = clock64() - t0;
        out[blockIdx.x] = red[0];
    }
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 2000;
    unsigned *flag;
    double *part, *out;
    long long *cyc;
    unsigned long long *inbox;
    cudaMalloc(&flag, 64);
    cudaMalloc(&part, sizeof(double) * 2 * 8 * 256);
    cudaMalloc(&out, sizeof(double) * 256);
    cudaMalloc(&cyc, sizeof(long long) * 256);
    const size_t inbox_words = (size_t)2 * sms * sms * 16;
    cudaMalloc(&inbox, inbox_words * 8);
    for (int nv : {1, 2}) {
        for (int rep = 0; rep < 2; rep++) {
            cudaMemset(flag, 0, 64);
            cudaMemset(inbox, 0, inbox_words * 8);
            int nvv = nv, it = iters;
            void *a1[] = {&flag, &part, &it, &nvv, &out, &cyc};
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            cudaLaunchCooperativeKernel((void *)probe_counter, sms, 1024, a1, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms1;
            cudaEventElapsedTime(&ms1, e0, e1);
            void *a2[] = {&inbox, &it, &nvv, &out, &cyc};
            cudaEventRecord(e0);
            cudaLaunchCooperativeKernel((void *)probe_inbox, sms, 1024, a2, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms2;
            cudaEventElapsedTime(&ms2, e0, e1);
            cudaMemset(flag, 0, 64);
            cudaEventRecord(e0);
            cudaLaunchCooperativeKernel((void *)probe_lean, sms, 1024, a1, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms3;
            cudaEventElapsedTime(&ms3, e0, e1);
            cudaError_t err = cudaGetLastError();
            printf("nv=%d: counter all-reduce %.3f us per phase | inbox %.3f us | lean counter %.3f us  (%s)\n", nv,
                   1e3 * ms1 / iters, 1e3 * ms2 / iters, 1e3 * ms3 / iters, cudaGetErrorString(err));
        }
    }
    return 0;
}
