// clz_probe.cu — phase cycles of the cluster Lanczos kernel (csrc/persist_cl.cuh) on c2's operator
// (2-D Laplacian 256 x 256), CTA 0 / thread 0 clock64 stamps (CLZ_CLOCKS), plus event time per step.
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_0907_4631_b200/csrc -Iinclude \
//        -o tools/clz_probe tools/clz_probe.cu
#define CLZ_CLOCKS 1
#include "persist_cl.cuh"

#include <cmath>
#include <cstdio>
#include <vector>

using namespace phipm;

int main(int argc, char **argv)
{
    const int nx = argc > 1 ? atoi(argv[1]) : 256, cs = argc > 2 ? atoi(argv[2]) : 16;
    const int nt = argc > 3 ? atoi(argv[3]) : 1024;
    const int m = argc > 4 ? atoi(argv[4]) : 40;
    const int64_t n = (int64_t)nx * nx;
    StencilOp op{};
    op.dim = 2;
    op.nx = op.ny = nx;
    op.nz = 1;
    op.n = n;
    const double h2 = (nx + 1.0) * (nx + 1.0);
    op.c[0] = -4 * h2;
    op.c[1] = op.c[2] = op.c[3] = op.c[4] = h2;
    double *V, *H, *sigma, *g;
    DevState *st;
    cudaMalloc(&V, n * 8 * (m + 2));
    cudaMalloc(&H, 8 * (m + 1) * (m + 1));
    cudaMalloc(&sigma, 8 * (m + 2));
    cudaMalloc(&g, 8 * 130);
    cudaMalloc(&st, sizeof(DevState));
    std::vector<double> v(n);
    double s2 = 0;
    for (int64_t i = 0; i < n; i++) {
        v[i] = sin(0.37 * i) + 0.1 * cos(0.011 * i);
        s2 += v[i] * v[i];
    }
    cudaMemcpy(V, v.data(), n * 8, cudaMemcpyHostToDevice);
    const double s0 = 1.0 / sqrt(s2);
    cudaMemcpy(sigma, &s0, 8, cudaMemcpyHostToDevice);
    DevState hs{};
    hs.brk = -1;
    Work wk{};
    wk.V = V;
    wk.ldv = n;
    wk.H = H;
    wk.ldh = m + 1;
    wk.hcols = m;
    wk.sigma = sigma;
    wk.g = g;
    wk.st = st;
    SmallArgs sa;
    sa.k0 = 0;
    sa.k1 = m;
    sa.symmetric = 1;
    sa.orth = 0;
    sa.bthr = 0.0;
    ClArgs ca;
    ca.cs = cs;
    ca.rpc = (n + cs - 1) / cs;
    ca.reach = nx;
    void (*kfn)(StencilOp, SmallArgs, ClArgs, Work) = nt == 1024 ? krylov_cluster_lanczos_kernel<1024, 4, 2>
                                                      : nt == 512 ? krylov_cluster_lanczos_kernel<512, 8, 2>
                                                                  : krylov_cluster_lanczos_kernel<256, 16, 2>;
    ca.blen = (int)cl_buf_len(op, ca.rpc, ca.reach, cs);
    const size_t smem = ca.blen * 8;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    long long zero[16] = {0};
    long long clk[16];
    for (int rep = 0; rep < 10; rep++) {
        cudaMemcpy(st, &hs, sizeof(hs), cudaMemcpyHostToDevice);
        cudaMemcpyToSymbol(clz_clk, zero, sizeof(zero));
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, kfn, op, sa, ca, wk);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) {
            best = ms;
            cudaMemcpyFromSymbol(clk, clz_clk, sizeof(clk));
        }
    }
    printf("nt=%d nx=%d cs=%d rpc=%lld: %s, kernel %.1f us for %d steps (%.3f us/step)\n", nt, nx, cs, (long long)ca.rpc,
           cudaGetErrorString(cudaGetLastError()), best * 1e3, m, best * 1e3 / m);
    const char *nm[6] = {"halo wait", "raw spmv", "y,dot,red1", "update+push", "recv norm", "send norm"};
    long long tot = 0;
    for (int i = 0; i < 6; i++) tot += clk[i];
    for (int i = 0; i < 6; i++) printf("  %-12s %7.0f cycles/step\n", nm[i], (double)clk[i] / m);
    printf("  total        %7.0f cycles/step\n", (double)tot / m);
    return 0;
}
