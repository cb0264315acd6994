// Probe: tensor-map TMA store (shared -> global) of a 4-D box with out-of-range coordinates (clipping).
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tma_store_probe tools/tma_store_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tm, int cx, int cy, int cz, int cc, int n)
{
    extern __shared__ __align__(128) double sm[];
    for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = 1000.0 + i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(&tm),
                     "r"(cx), "r"(cy), "r"(cz), "r"(cc), "r"(smem_u32(sm))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

int main()
{
    const int nx = 12, ny = 6, nz = 5, nc = 3, ylen = 4;
    const int64_t ld = 512;
    double *d;
    cudaMalloc(&d, ld * nc * 8);
    cudaMemset(d, 0, ld * nc * 8);
    typedef CUresult (*Enc)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                            const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void *fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    CUtensorMap tm;
    const cuuint64_t gdim[4] = {nx, ny, nz, nc};
    const cuuint64_t gstr[3] = {nx * 8, nx * ny * 8, (cuuint64_t)ld * 8};
    const cuuint32_t box[4] = {nx + 4, ylen, 1, 1}, est[4] = {1, 1, 1, 1};
    CUresult r = ((Enc)fp)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, gdim, gstr, box, est, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    const int cases[3][4] = {{0, 4, 2, 1}, {0, 0, 4, 2}, {-2, 0, 1, 2}};
    for (auto &c : cases) {
        cudaMemset(d, 0, ld * nc * 8);
        probe<<<1, 128, (nx + 4) * ylen * 8>>>(tm, c[0], c[1], c[2], c[3], (nx + 4) * ylen);
        cudaError_t e = cudaDeviceSynchronize();
        printf("coords (%d,%d,%d,%d): %s\n", c[0], c[1], c[2], c[3], cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
        std::vector<double> h(ld * nc);
        cudaMemcpy(h.data(), d, ld * nc * 8, cudaMemcpyDeviceToHost);
        int nzc = 0;
        for (int i = 0; i < ld * nc; i++)
            if (h[i] != 0.0) {
                if (nzc < 6) printf("  [%d] = %g\n", i, h[i]);
                nzc++;
            }
        printf("  nonzeros %d\n", nzc);
    }
    return 0;
}
