// stream_roof.cu — read/copy bandwidth roofs on this B200 (measurement tool, not product code).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_roof tools/stream_roof.cu
// Measures (CUDA events, best of 10, 1 GiB buffers):
//   copy_ld      : y = x with 16-B vector loads/stores, grid-stride (read+write bytes)
//   read_ld      : sum(x) with 16-B loads, U loads in flight per thread, many CTAs
//   read_tma     : sum(x) through a 1-D TMA (cp.async.bulk) mbarrier ring, 1 CTA/SM,
//                  segment size and ring depth varied
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void copy_ld(const double2 *__restrict__ x, double2 *__restrict__ y, size_t n2)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) y[i] = x[i];
}

template <int U>
__global__ void read_ld(const double2 *__restrict__ x, size_t n2, double *out)
{
    double s = 0;
    size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n2; i += U * stride) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; u++) v[u] = __ldcs(x + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; u++) s += v[u].x + v[u].y;
    }
    for (; i < n2; i += stride) { double2 v = x[i]; s += v.x + v.y; }
    if (s == 1.2345) *out = s;
}

__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void read_tma(const double *__restrict__ x, size_t n, int seg, int nring, int nconsumer_warps, double *out)
{
    extern __shared__ __align__(128) double sm[];
    __shared__ uint64_t full[64], empty[64];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < nring; s++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&empty[s])), "r"(nconsumer_warps));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const size_t nseg = n / seg;
    double acc = 0;
    if (warp == nconsumer_warps) {
        if (lane == 0) {
            uint32_t it = 0;
            for (size_t g = blockIdx.x; g < nseg; g += gridDim.x, it++) {
                int s = it % nring; uint32_t r = it / nring;
                if (r >= 1) {
                    asm volatile("{.reg .pred p; W1: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W1;}" ::"r"(su(&empty[s])), "r"((r - 1) & 1));
                }
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(seg * 8));
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(sm + (size_t)s * seg)), "l"(x + g * seg), "r"(seg * 8), "r"(su(&full[s])) : "memory");
            }
        }
    } else {
        uint32_t it = 0;
        for (size_t g = blockIdx.x; g < nseg; g += gridDim.x, it++) {
            int s = it % nring;
            asm volatile("{.reg .pred p; W2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W2;}" ::"r"(su(&full[s])), "r"((it / nring) & 1) : "memory");
            const double *sl = sm + (size_t)s * seg;
            for (int q = tid; q < seg; q += nconsumer_warps * 32) acc += sl[q];
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
        }
    }
    if (acc == 1.2345) *out = acc;
}

int main()
{
    const size_t n = (size_t)1 << 27;      // 128 Mi doubles = 1 GiB
    double *x, *y, *out;
    CK(cudaMalloc(&x, n * 8));
    CK(cudaMalloc(&y, n * 8));
    CK(cudaMalloc(&out, 8));
    CK(cudaMemset(x, 0, n * 8));
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto best = [&](auto launch, double bytes, const char *name) {
        float bms = 1e9;
        for (int r = 0; r < 10; r++) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r > 0 && ms < bms) bms = ms;
        }
        cudaError_t e = cudaGetLastError();
        printf("%-44s %8.1f GB/s  %s\n", name, bytes / (bms * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    best([&] { copy_ld<<<sms * 8, 256>>>((double2 *)x, (double2 *)y, n / 2); }, 16.0 * n, "copy_ld (read+write)");
    best([&] { read_ld<4><<<sms * 8, 256>>>((double2 *)x, n / 2, out); }, 8.0 * n, "read_ld U=4, 8 CTA/SM x 256");
    best([&] { read_ld<8><<<sms * 8, 256>>>((double2 *)x, n / 2, out); }, 8.0 * n, "read_ld U=8, 8 CTA/SM x 256");
    best([&] { read_ld<8><<<sms * 4, 256>>>((double2 *)x, n / 2, out); }, 8.0 * n, "read_ld U=8, 4 CTA/SM x 256");
    int segs[] = {1024, 2048, 4096, 8192};
    for (int seg : segs)
        for (int depth_kb : {64, 128, 192}) {
            int nring = depth_kb * 1024 / (seg * 8);
            if (nring < 2 || nring > 64) continue;
            for (int cw : {4, 16}) {
                size_t smem = (size_t)nring * seg * 8;
                cudaFuncSetAttribute(read_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                char name[128];
                snprintf(name, sizeof(name), "read_tma seg=%d B ring=%d (%d KB) cw=%d", seg * 8, nring, depth_kb, cw);
                best([&] { read_tma<<<sms, (cw + 1) * 32, smem>>>(x, n, seg, nring, cw, out); }, 8.0 * n, name);
            }
        }
    // two CTAs per SM
    for (int seg : {1024, 4096}) {
        int nring = 96 * 1024 / (seg * 8);
        size_t smem = (size_t)nring * seg * 8;
        cudaFuncSetAttribute(read_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        char name[128];
        snprintf(name, sizeof(name), "read_tma 2 CTA/SM seg=%d B ring=%d", seg * 8, nring);
        best([&] { read_tma<<<sms * 2, 8 * 32 + 32, smem>>>(x, n, seg, nring, 8, out); }, 8.0 * n, name);
    }
    return 0;
}
