// phipm.cu — host side of libphipm: context/workspace, kernel launches, the step-size and
// Krylov-dimension controller (Sec. 3.3-3.4, Algorithms 3-4), and the C ABI of
// include/phipm.h.
//
// The controller reads back one small result block per attempt (mapped pinned memory written
// by the expm kernel); everything n-sized runs in the kernels of kernels.cuh / expm.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <functional>
#include <mutex>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "phipm.h"
#include "kernels.cuh"
#include "expm.cuh"
#include "stream.cuh"
#include "small.cuh"
#include "persist.cuh"
#include "persist_tm.cuh"
#include "persist_brick.cuh"
#include "persist_wrec.cuh"
#include "phicheb.cuh"
#include "spmm.cuh"
#include "persist_cl.cuh"
#include "ctl.cuh"
#include "solve_small.cuh"

using namespace phipm;

namespace {

constexpr int P_MAX_ABS = 6;          // MAXZ bounds the epilogue vector count
constexpr double EPS_MACH = 2.220446049250313080847e-16;

constexpr int KCLK_MAXL = 512, KCLK_GRID = 1024;     // PHIPM_KCLOCKS capacity (launches, CTAs)
constexpr size_t PCLK_CAP = (size_t)1 << 22;           // persistent-kernel stamps (u64)

enum ProfClass { PC_SPMV = 0, PC_ORTH, PC_EXPM, PC_COMBINE, PC_OTHER, PC_N };

struct ProfRec {
    cudaEvent_t a, b;
    int cls;
    int ncols;
    double bytes;
};

} // namespace

struct GraphRec {
    std::vector<unsigned char> key;
    cudaGraphExec_t exec = nullptr;
    int64_t nlaunch = 0;
};

struct BrickMap {
    CUtensorMap map;
    const double *base = nullptr;           // nullptr: none
    int nx = 0, ny = 0, nz = 0, ylen = 0, zlen = 0, xlen = 0;    // grid and box (lines, planes, points)
};

struct phipm_ctx {
    int dev = 0;
    cudaStream_t stream = nullptr;
    int64_t n_max = 0, ldv = 0;
    int m_max = 0, p_max = 0, kmax = 0;
    int sm_count = 0, occ_spmv = 1, occ_axpy = 1;
    int pstride = 0;
    size_t expm_smem_limit = 0, stream_smem_budget = 0, smem_optin = 0;
    struct OccEntry { const void *fn; size_t smem; int occ; };
    std::vector<OccEntry> occ_cache;
    // device workspace
    double *V = nullptr, *W = nullptr, *Y = nullptr, *U = nullptr, *H = nullptr, *sigma = nullptr, *g = nullptr;
    double *part2 = nullptr;                         // partials of a deferred-finalize SpMV (PHIPM_OPT_DEFER)
    int defer_nb = 0;                                // grid of the last SpMV launched with SpmvArgs.defer
    double *part = nullptr, *comb = nullptr, *combd = nullptr, *scratch = nullptr, *raw = nullptr;
    unsigned *counter = nullptr;
    bool coop_dirty = false;                         // a cooperative kernel timed out: reset its counters
    cudaEvent_t ev_binf = nullptr;                   // ||u_0||_inf readback of a solve
    cudaStream_t stream2 = nullptr;                  // speculative Krylov extensions (PHIPM_OPT_SPEC); ||u_0||_inf
    // ||u_0||_inf of a solve on stream2 (PHIPM_OPT_SIDE_MAXABS): its own reduction scratch, because the
    // kernels of the main stream use part / counter / raw at the same time
    double *part_mx = nullptr, *raw_mx = nullptr;
    unsigned *counter_mx = nullptr;
    bool mx_side_pending = false;                    // the side-stream reduction has not been read yet
    int *dec_d = nullptr;                            // device acceptance decision of an attempt (PHIPM_OPT_PRECOMBINE)
    cudaEvent_t ev_main = nullptr, ev_spec = nullptr;
    bool spec_pending = false;                       // an extension on stream2 not yet joined to stream
    // device-driven solves of small problems (solve_small.cuh)
    SsAttempt *ss_att_d = nullptr;                   // attempt records (device)
    SsOut *ss_out_h = nullptr, *ss_out_d = nullptr;  // stats and status (mapped pinned)
    int ss_att_pending = 0;                          // records of the last solve still on the device
    bool defer = false, deferred = false;            // batch fast path: launch the device solve, collect later
    std::vector<GraphRec> graphs;                    // captured two-kernel extensions (PHIPM_OPT_GRAPH)
    DevState *st = nullptr;
    int32_t *tlo = nullptr, *thi = nullptr;                  // CSR per-tile column ranges
    int16_t *off16 = nullptr;                                // CSR int16 column offsets (x-ring path)
    int64_t off16_cap = 0;
    int64_t ntile_cap = 0;
    AttemptResult *res_h = nullptr, *res_d = nullptr;
    struct MaxPub {
        double v[MAXZ];
        int seq;
        int aseq;                                    // ||A||_inf from the first SpMV (fused CSR path) ...
        double anorm;                                // ... published here
    } *mx_h = nullptr, *mx_d = nullptr;               // ||u_0||_inf published to mapped pinned memory
    int mx_seq = 0, mx_aseq = 0;
    bool fuse_anorm = false;                         // this solve's first SpMV computes ||A||_inf
    long long *expm_clk_h = nullptr, *expm_clk_d = nullptr;   // PHIPM_EXPM_CLOCKS=1 debug timestamps
    // PHIPM_KCLOCKS=<file>: per-CTA %globaltimer stamps of every streaming launch (measurement tool)
    unsigned long long *kclk_d = nullptr;
    struct KclkRec { int cls, grid, ncols; };
    std::vector<KclkRec> kclk_recs;
    const char *kclk_path = nullptr;
    unsigned long long *pclk_d = nullptr;            // persistent kernel phase stamps
    struct PclkRec { int grid, steps; long long off; };
    std::vector<PclkRec> pclk_recs;
    size_t pclk_used = 0;
    double *raw_h = nullptr;                 // pinned staging for small readbacks
    // host-buffer solve staging
    double *hu = nullptr, *hw = nullptr;
    int32_t *hrp = nullptr, *hcol = nullptr;
    double *hval = nullptr;
    int64_t nnz_cap = 0;
    // profiling
    bool prof = false;
    bool trace = false;
    bool pdl = true;
    std::vector<phipm_trace_rec> tracebuf;
    std::vector<phipm_attempt> attempts;     // controller trajectory of the last solve
    int64_t nattempts = 0;
    int64_t ncheb_fallback = 0;              // attempts whose Chebyshev interval was too wide
    int64_t ntrace = 0;
    std::vector<ProfRec> pending;
    std::vector<cudaEvent_t> pool;
    phipm_profile acc{};
    int seq = 0;
    int expm_method = PHIPM_EXPM_TAYLOR;     // phipm_expm / phipm_phi_pair
    // kernel-path selection (phipm_set_option; defaults: the measured-best paths)
    int opt[PHIPM_OPT_COUNT] = {1, 1, 1, 1, 1, 1, 0, 1, 1, 0, 1, 0, 384, 0, 1, 0, 1, 1, 1, 0, 1, 1, 0, 1, 0};
    // brick kernels: tensor maps of V, W and the w-recurrence's x_0 for the last grid / brick shape
    BrickMap brick_maps[5];                 // V planes, W planes, x_0 planes, V z-halo planes, V y-halo lines
    int krylov_path = PHIPM_PATH_NONE;      // kernel path of the last Krylov extension (phipm_krylov_path)
    int wrec_path = PHIPM_PATH_NONE;        // ... of the last w-recurrence (phipm_wrec_path)
    char err[512] = {0};
};

namespace {

int set_err(phipm_ctx *c, int code, const char *fmt, ...)
{
    if (c) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(c->err, sizeof(c->err), fmt, ap);
        va_end(ap);
    }
    return code;
}

#define CK(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return set_err(c, PHIPM_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                           __FILE__, __LINE__);                                                    \
    } while (0)

#define CK0(ctx_, call)                                                                            \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return set_err(ctx_, PHIPM_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                           __FILE__, __LINE__);                                                    \
    } while (0)

Work make_work(phipm_ctx *c)
{
    Work w;
    w.V = c->V;
    w.ldv = c->ldv;
    w.H = c->H;
    w.ldh = c->m_max + 1;
    w.hcols = c->m_max;
    w.sigma = c->sigma;
    w.g = c->g;
    w.part = c->part;
    w.part2 = c->part2;
    w.pstride = c->pstride;
    w.counter = c->counter;
    w.st = c->st;
    w.out_raw = c->raw;
    return w;
}

cudaEvent_t ev_get(phipm_ctx *c)
{
    if (!c->pool.empty()) {
        cudaEvent_t e = c->pool.back();
        c->pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

void prof_begin(phipm_ctx *c, ProfRec &r, int cls, double bytes, int ncols = 0)
{
    if (!c->prof) return;
    r.cls = cls;
    r.ncols = ncols;
    r.bytes = bytes;
    r.a = ev_get(c);
    r.b = ev_get(c);
    cudaEventRecord(r.a, c->stream);
}

void prof_end(phipm_ctx *c, ProfRec &r)
{
    if (!c->prof) return;
    cudaEventRecord(r.b, c->stream);
    c->pending.push_back(r);
}

// after a stream sync: fold pending event pairs into the accumulators
void prof_collect(phipm_ctx *c)
{
    for (auto &r : c->pending) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        switch (r.cls) {
        case PC_SPMV: c->acc.ms_spmv_dot += ms; c->acc.bytes_spmv_dot += r.bytes; c->acc.n_spmv_dot++; break;
        case PC_ORTH: c->acc.ms_orth += ms; c->acc.bytes_orth += r.bytes; c->acc.n_orth++; break;
        case PC_EXPM: c->acc.ms_expm += ms; c->acc.n_expm++; break;
        case PC_COMBINE: c->acc.ms_combine += ms; c->acc.bytes_combine += r.bytes; c->acc.n_combine++; break;
        default: c->acc.ms_other += ms; c->acc.bytes_other += r.bytes; break;
        }
        if (c->trace) {
            if (c->tracebuf.size() < 65536) c->tracebuf.push_back({r.cls, r.ncols, r.bytes, 1e3 * (double)ms});
            c->ntrace++;
        }
        c->pool.push_back(r.a);
        c->pool.push_back(r.b);
    }
    c->pending.clear();
}

int grid_for(phipm_ctx *c, int64_t units, int occ)
{
    int64_t g = std::min<int64_t>(units, (int64_t)occ * c->sm_count);
    if (g < 1) g = 1;
    if (g > c->pstride) g = c->pstride;
    return (int)g;
}

// kernel-path option of the context (phipm_set_option)
inline int opt(const phipm_ctx *c, int o) { return c->opt[o]; }

// ---------------------------------------------------------------------------------------------
// launches

// Launch with Programmatic Dependent Launch allowed: the kernel's launch and prologue overlap the
// previous kernel's tail; every kernel executes griddepcontrol.wait before touching data written
// by its predecessor (kernels.cuh: pdl_wait).
template <typename... KArgs, typename... Args>
cudaError_t launch_k(phipm_ctx *c, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = c->pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// Cooperative launch (all CTAs co-resident, or the launch fails), PDL allowed: the kernels set up
// (TMEM, halo plans, mbarriers) before griddepcontrol.wait.
template <typename... KArgs, typename... Args>
cudaError_t launch_coop(phipm_ctx *c, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = c->pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// occupancy-limited grid for a streaming kernel (cached per kernel/smem)
int stream_grid(phipm_ctx *c, const void *fn, size_t smem, int64_t ntiles)
{
    int occ = 0;
    for (auto &e : c->occ_cache)
        if (e.fn == fn && e.smem == smem) { occ = e.occ; break; }
    if (occ == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, SNT, smem);
        occ = std::max(occ, 1);
        c->occ_cache.push_back({fn, smem, occ});
    }
    return (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)occ * c->sm_count));
}

template <class Op>
int halo_cap_host(const Op &, int tile) { return tile; }
template <>
int halo_cap_host<StencilOp>(const StencilOp &S, int tile) { return halo_capacity(S.dim, S.nx, tile); }

template <class Op>
int csr_ring(const Op &, int) { return 0; }
template <>
int csr_ring<CsrOp>(const CsrOp &A, int tile) { return A.ring && 2 * tile + A.blo + A.bhi <= XRING; }

// the operator as one launch with `tile`-row tiles sees it (x ring only where it fits)
template <class Op>
Op launch_op(const Op &op, int) { return op; }
template <>
CsrOp launch_op<CsrOp>(const CsrOp &A, int tile)
{
    CsrOp o = A;
    o.ring = csr_ring(A, tile);
    return o;
}

template <class Op>
int csr_wcap(const Op &, int) { return 0; }
template <>
int csr_wcap<CsrOp>(const CsrOp &A, int tile) { return A.wtile == tile ? A.wcap : 0; }

// rows per thread: 8 (TILE 8 SNT) when every CTA gets at least half a tile, else 2;
// PHIPM_OPT_RPT = 2|4|8 overrides (tuning experiments)
int pick_rpt(phipm_ctx *c, int64_t n)
{
    const int env = opt(c, PHIPM_OPT_RPT);
    if (env == 2 || env == 4 || env == 8) return env;
    return n >= (int64_t)SNT * 8 * c->sm_count * SMINB / 2 ? 8 : 2;
}

// balanced partition: every resident CTA slot gets one contiguous range of rpc rows (a multiple
// of 32), processed in tiles of <= 256*RPT rows; small problems use fewer CTAs
void balance(phipm_ctx *c, int64_t n, int slots, int &grid, int64_t &rpc)
{
    int64_t g = std::min<int64_t>(slots, (n + 31) / 32);
    g = std::max<int64_t>(1, std::min<int64_t>(g, c->pstride));
    rpc = ((n + g - 1) / g + 31) / 32 * 32;
    grid = (int)((n + rpc - 1) / rpc);
}

unsigned long long *kclk_slot(phipm_ctx *c, int cls, int grid, int ncols)
{
    if (!c->kclk_d || (int)c->kclk_recs.size() >= KCLK_MAXL || grid > KCLK_GRID) return nullptr;
    unsigned long long *p = c->kclk_d + c->kclk_recs.size() * (size_t)KCLK_GRID * 8;
    c->kclk_recs.push_back({cls, grid, ncols});
    return p;
}

template <class Op, int RPT>
int launch_spmv_t(phipm_ctx *c, const Op &op, const SpmvArgs &a0)
{
    constexpr int TILE_ = SNT * RPT;
    SpmvArgs a = a0;
    const Op lop = launch_op(op, TILE_);
    const size_t smem = spmv_smem_bytes(halo_cap_host(op, TILE_), TILE_, a.nd, csr_wcap(op, TILE_), csr_ring(op, TILE_));
    const bool ringk = csr_ring(op, TILE_) != 0;           // CsrOp only: the x-ring instantiation
    const void *fn = ringk ? (const void *)spmv_stream_kernel<Op, RPT, 2> : (const void *)spmv_stream_kernel<Op, RPT>;
    const int slots = stream_grid(c, fn, smem, (int64_t)1 << 40);
    int grid;
    balance(c, op.n, slots, grid, a.rpc);
    a.dbg = kclk_slot(c, PC_SPMV, grid, a.nd);
    if (a.defer) c->defer_nb = grid;
    if (ringk) launch_k(c, spmv_stream_kernel<Op, RPT, 2>, grid, SNT, smem, lop, a, make_work(c));
    else launch_k(c, spmv_stream_kernel<Op, RPT>, grid, SNT, smem, lop, a, make_work(c));
    return PHIPM_OK;
}

template <class Op>
int launch_spmv(phipm_ctx *c, const Op &op, const SpmvArgs &a0, double bytes_op)
{
    SpmvArgs a = a0;
    if (a.ldx == 0) a.ldx = c->ldv;
    a.pfc = opt(c, PHIPM_OPT_COL_PREFETCH);
    if (std::is_same<Op, CsrOp>::value) a.xcol = -1;          // CSR gathers x: no on-chip tile
    ProfRec r;
    // algorithmic bytes: operator pass + streamed dot columns (the x column is reused on chip) + z
    const int nd_mem = a.nd - (a.xcol >= 0 && a.xcol < a.nd ? 1 : 0);
    const double bytes = bytes_op + 8.0 * (double)op.n * (nd_mem + a.nz);
    prof_begin(c, r, PC_SPMV, bytes, a.nd);
    if (op.n <= SMALL_N && a.nd <= MAXD && !a.xnorm) {
        // small vectors: one CTA, no grid reduction (small.cuh)
        launch_k(c, spmv_small_kernel<Op>, 1, SMALL_NT, 0, op, a, make_work(c));
        prof_end(c, r);
        c->acc.launches++;
        CK(cudaGetLastError());
        return PHIPM_OK;
    }
    int rpt = pick_rpt(c, op.n);
    if (csr_wcap(op, SNT * 8) > 0) rpt = 8;                  // CSR x-window mode uses 8 SNT-row tiles
    // largest tile whose halo + dot accumulators fit in shared memory (3-D stencils, many dots)
    while (rpt > 2 && spmv_smem_bytes(halo_cap_host(op, SNT * rpt), SNT * rpt, a.nd, csr_wcap(op, SNT * rpt),
                                      csr_ring(op, SNT * rpt)) > c->smem_optin)
        rpt >>= 1;
    // x-ring CSR: the largest tile with 2 TILE + band <= XRING
    if (csr_ring(op, SNT * 2))
        while (rpt > 2 && !csr_ring(op, SNT * rpt)) rpt >>= 1;
    if (rpt == 8) launch_spmv_t<Op, 8>(c, op, a);
    else if (rpt == 4) launch_spmv_t<Op, 4>(c, op, a);
    else launch_spmv_t<Op, 2>(c, op, a);
    prof_end(c, r);
    c->acc.launches++;
    CK(cudaGetLastError());
    return PHIPM_OK;
}

template <int RPT>
void launch_axpy_t(phipm_ctx *c, int64_t n, const AxpyArgs &a0)
{
    AxpyArgs a = a0;
    const int slots = stream_grid(c, (const void *)axpy_stream_kernel<RPT>, 0, (int64_t)1 << 40);
    int grid;
    balance(c, n, slots, grid, a.rpc);
    a.dbg = kclk_slot(c, PC_ORTH, grid, a.nc);
    launch_k(c, axpy_stream_kernel<RPT>, grid, SNT, 0, n, a, make_work(c));
}

int launch_axpy(phipm_ctx *c, int64_t n, const AxpyArgs &a_in, int cls)
{
    AxpyArgs a = a_in;
    a.pfc = opt(c, PHIPM_OPT_COL_PREFETCH);
    ProfRec r;
    const double bytes = 8.0 * (double)n * (a.nc + a.ne + 1 + (a.a0h != 0.0 ? 1 : 0));
    prof_begin(c, r, cls, bytes, a.nc + a.ne + (a.a0h != 0.0 ? 1 : 0));
    if (n <= SMALL_N) {
        launch_k(c, axpy_small_kernel, 1, SMALL_NT, 0, n, a, make_work(c));   // one CTA (small.cuh)
        prof_end(c, r);
        c->acc.launches++;
        CK(cudaGetLastError());
        return PHIPM_OK;
    }
    const int rpt = pick_rpt(c, n);
    if (rpt == 8) launch_axpy_t<8>(c, n, a);
    else if (rpt == 4) launch_axpy_t<4>(c, n, a);
    else launch_axpy_t<2>(c, n, a);
    prof_end(c, r);
    c->acc.launches++;
    CK(cudaGetLastError());
    return PHIPM_OK;
}

int launch_expm(phipm_ctx *c, ExpmArgs &a, int K)
{
    const int Kp = (K + 7) & ~7;
    const size_t need = (size_t)6 * expm_ld(Kp) * Kp * sizeof(double);
    a.use_smem = need <= c->expm_smem_limit;
    a.scratch = c->scratch;
    a.res = c->res_d;
    a.seq = ++c->seq;
    a.clk = c->expm_clk_d;
    ProfRec r;
    prof_begin(c, r, PC_EXPM, 0.0, K);
    if (a.method == PHIPM_EXPM_CHEBYSHEV && a.tridiag && a.mode != 1) {
        launch_k(c, phi_cheb_kernel, 1, CHEB_NT, 0, a);
    } else if (a.method == PHIPM_EXPM_PADE13) {
        if (a.use_smem) launch_k(c, expm_kernel<true, true>, 1, EXPM_NT, need, a);
        else launch_k(c, expm_kernel<false, true>, 1, EXPM_NT, 0, a);
    } else {
        if (a.use_smem) launch_k(c, expm_kernel<true, false>, 1, EXPM_NT, need, a);
        else launch_k(c, expm_kernel<false, false>, 1, EXPM_NT, 0, a);
    }
    prof_end(c, r);
    c->acc.launches++;
    CK(cudaGetLastError());
    return PHIPM_OK;
}

int sync(phipm_ctx *c)
{
    CK(cudaStreamSynchronize(c->stream));
    if (c->prof) prof_collect(c);
    return PHIPM_OK;
}

// Wait for the attempt result of the exponential just enqueued: spin on the sequence number its
// epilogue publishes last (after a system-scope fence) in mapped pinned memory, instead of a stream
// synchronisation.  The controller only needs that block; every later kernel is stream-ordered.
// Profiling (events to collect) and anything slower than 2 s (e.g. a fault: the stream reports it)
// fall back to cudaStreamSynchronize.
int wait_attempt(phipm_ctx *c)
{
    if (c->prof || !opt(c, PHIPM_OPT_SPIN)) return sync(c);
    const volatile int *seqp = &reinterpret_cast<volatile AttemptResult *>(c->res_h)->seq;
    const auto t0 = std::chrono::steady_clock::now();
    unsigned spins = 0;
    while (*seqp != c->seq) {
        ++spins;
        // after ~20 us of spinning give the core away between polls: concurrent solves (batch API,
        // one host thread each) would otherwise saturate the host's cores with spinners
        if (spins > 4096) std::this_thread::yield();
        if ((spins & 1023) == 0 && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(2)) return sync(c);
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    return PHIPM_OK;
}

AxpyArgs axpy0()
{
    AxpyArgs a;
    memset(&a, 0, sizeof(a));
    a.gsign = 1.0;
    return a;
}

SpmvArgs spmv0()
{
    SpmvArgs a;
    memset(&a, 0, sizeof(a));
    a.xcol = -1;
    return a;
}

// controller: ctl.cuh (shared with the device solve loop of small problems)

// ---------------------------------------------------------------------------------------------
// Krylov extension: steps j = k0 .. k1-1 (0-based), all on the device

// The whole extension k0 -> k1 in one cooperative kernel (persist.cuh) when the operator is a
// stencil and the CTA's y, halo tile and dot partials fit in shared memory (PHIPM_PERSIST=0
// disables).  Returns true if it launched (rc = status).
template <class Op>
bool launch_persist(phipm_ctx *, const Op &, double, bool, int, int, double, int &) { return false; }

// Cooperative launches zero their arrival counter on a normal exit (coop_exit); only after a grid
// phase timed out (coop_dirty) are the counters and the abort flags cleared by memsets first.
bool coop_reset(phipm_ctx *c)
{
    if (!c->coop_dirty) return true;
    if (cudaMemsetAsync(c->counter + 2, 0, 3 * sizeof(unsigned), c->stream) != cudaSuccess ||
        cudaMemsetAsync(&c->st->aborted, 0, sizeof(int), c->stream) != cudaSuccess)
        return false;
    c->coop_dirty = false;
    return true;
}

using PersistFn = void (*)(StencilOp, PersistArgs, Work);

template <int RPT, bool LANC>
PersistFn persist_fn_l(int dimc)
{
    switch (dimc) {
    case 1: return krylov_persist_kernel<RPT, LANC, 1>;
    case 2: return krylov_persist_kernel<RPT, LANC, 2>;
    case 3: return krylov_persist_kernel<RPT, LANC, 3>;
    default: return krylov_persist_kernel<RPT, LANC, 4>;
    }
}

// the instantiation for this operator (dimension class: 1, 2, 3, or 4 = 2-D 9-point) and method
template <int RPT>
PersistFn persist_fn(const StencilOp &op, bool symmetric)
{
    const int dimc = (op.dim == 2 && op.diag) ? 4 : op.dim;
    return symmetric ? persist_fn_l<RPT, true>(dimc) : persist_fn_l<RPT, false>(dimc);
}

template <int RPT>
void persist_set_smem(int mx)
{
    for (int d = 1; d <= 4; d++)
        for (int l = 0; l < 2; l++) {
            StencilOp op{};
            op.dim = d == 4 ? 2 : d;
            op.diag = d == 4;
            cudaFuncSetAttribute(persist_fn<RPT>(op, l != 0), cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        }
}

template <int RPT>
bool try_persist_rpt(phipm_ctx *c, const StencilOp &op, bool symmetric, int k0, int k1, double bthr, double bytes,
                     int &rc)
{
    constexpr int TILE_ = SNT * RPT;
    const PersistFn kfn = persist_fn<RPT>(op, symmetric);
    int grid;
    int64_t rpc;
    // CTAs: at most one per SM, and (PHIPM_OPT_PERSIST_MINROWS, default TILE/2) enough rows each that
    // the threads are busy: small problems then also reduce fewer partials per phase
    const int env_rows = opt(c, PHIPM_OPT_PERSIST_MINROWS) ? std::max(32, opt(c, PHIPM_OPT_PERSIST_MINROWS)) : 0;
    const int64_t minrows = env_rows ? env_rows : TILE_ / 2;
    const int slots = (int)std::max<int64_t>(1, std::min<int64_t>(c->sm_count, (op.n + minrows - 1) / minrows));
    balance(c, op.n, slots, grid, rpc);
    const int ndmax = symmetric ? 1 : k1;
    const size_t smem = persist_smem_bytes(halo_capacity(op.dim, op.nx, TILE_), rpc, ndmax);
    if (smem > c->smem_optin || ndmax + 1 > MAXD + 2) return false;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, SNT, smem) != cudaSuccess ||
        occ < 1 || grid > occ * c->sm_count) {
        cudaGetLastError();
        return false;
    }
    PersistArgs a;
    a.k0 = k0;
    a.k1 = k1;
    a.symmetric = symmetric ? 1 : 0;
    a.bthr = bthr;
    a.rpc = rpc;
    a.flag = c->counter + 2;
    a.abort = c->counter + 3;
    a.exit_ctr = c->counter + 4;
    a.timeout_ns = 2000000000ull;
    // PHIPM_KCLOCKS: 2 stamps per CTA per phase (2 phases per step), separate buffer
    a.dbg = nullptr;
    const size_t need = (size_t)2 * (k1 - k0) * grid * 2;
    if (c->pclk_d && c->pclk_used + need <= PCLK_CAP) {
        a.dbg = c->pclk_d + c->pclk_used;
        c->pclk_recs.push_back({grid, k1 - k0, (long long)c->pclk_used});
        c->pclk_used += need;
    }
    rc = PHIPM_OK;
    if (!coop_reset(c)) {
        rc = set_err(c, PHIPM_ECUDA, "persist: memset failed");
        return true;
    }
    ProfRec r;
    prof_begin(c, r, PC_SPMV, bytes, k1 - k0);
    const cudaError_t e = launch_coop(c, kfn, grid, SNT, smem, op, a, make_work(c));
    prof_end(c, r);
    c->acc.launches++;
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;                                      // fall back to the two-kernel path
    }
    c->krylov_path = PHIPM_PATH_PERSIST_SMEM;
    return true;
}

PersistFn persist_tm_fn(const StencilOp &op)
{
    switch ((op.dim == 2 && op.diag) ? 4 : op.dim) {
    case 1: return krylov_persist_tm_kernel<1>;
    case 2: return krylov_persist_tm_kernel<2>;
    case 3: return krylov_persist_tm_kernel<3>;
    default: return krylov_persist_tm_kernel<4>;
    }
}

// Lanczos with the CTA's y / v~_j in tensor memory and double-buffered halo tiles (persist_tm.cuh),
// when every CTA's rows fit the 8 pair slots per thread (PHIPM_OPT_TMEM = 0 disables)
bool try_persist_tm(phipm_ctx *c, const StencilOp &op, int k0, int k1, double bthr, double bytes, int &rc)
{
    if (!opt(c, PHIPM_OPT_TMEM)) return false;
    constexpr int TILE_ = SNT * 4;
    int grid;
    int64_t rpc;
    const int slots = (int)std::max<int64_t>(1, std::min<int64_t>(c->sm_count, (op.n + TILE_ / 2 - 1) / (TILE_ / 2)));
    balance(c, op.n, slots, grid, rpc);
    if ((rpc + TILE_ - 1) / TILE_ * 2 > TM_PAIRS) return false;
    const size_t smem = persist_tm_smem_bytes(halo_capacity(op.dim, op.nx, TILE_));
    if (smem > c->smem_optin) return false;
    const PersistFn kfn = persist_tm_fn(op);
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, SNT, smem) != cudaSuccess || occ < 1 ||
        grid > occ * c->sm_count) {
        cudaGetLastError();
        return false;
    }
    PersistArgs a;
    a.k0 = k0;
    a.k1 = k1;
    a.symmetric = 1;
    a.bthr = bthr;
    a.rpc = rpc;
    a.flag = c->counter + 2;
    a.abort = c->counter + 3;
    a.exit_ctr = c->counter + 4;
    a.timeout_ns = 2000000000ull;
    a.dbg = nullptr;
    const size_t need = (size_t)2 * (k1 - k0) * grid * 2;
    if (c->pclk_d && c->pclk_used + need <= PCLK_CAP) {
        a.dbg = c->pclk_d + c->pclk_used;
        c->pclk_recs.push_back({grid, k1 - k0, (long long)c->pclk_used});
        c->pclk_used += need;
    }
    rc = PHIPM_OK;
    if (!coop_reset(c)) {
        rc = set_err(c, PHIPM_ECUDA, "persist: memset failed");
        return true;
    }
    ProfRec r;
    prof_begin(c, r, PC_SPMV, bytes, k1 - k0);
    const cudaError_t e = launch_coop(c, kfn, grid, SNT, smem, op, a, make_work(c));
    prof_end(c, r);
    c->acc.launches++;
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    c->krylov_path = PHIPM_PATH_PERSIST_TMEM;
    return true;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (the library does not link libcuda)
using TmapEncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

TmapEncodeFn tmap_encode_fn()
{
    static TmapEncodeFn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            p = nullptr;
        }
        return (TmapEncodeFn)p;
    }();
    return fn;
}

// 4-D tensor map (x, y, z, column) over `ncols` vectors of an nx x ny x nz grid, `ld` doubles apart; box = one
// plane of a brick with its halo: (nx + 4) x (ylen + 2) x 1 x 1, zero fill outside the grid.  Cached per
// context slot (0: the basis V, 1: the w-recurrence vectors W, 2: x_0 of the w-recurrence)
bool brick_tensor_map(phipm_ctx *c, int slot, const double *base, int ncols, int64_t ld, const StencilOp &op,
                      const BrickGeom &g, int box_y = 0, int box_z = 1, int box_x = 0)
{
    if (box_y == 0) box_y = g.ylen + 2;                    // (default: a whole plane with its y halo ...
    if (box_x == 0) box_x = op.nx + 4;                     // ... and two zero-filled points left and right)
    BrickMap &m = c->brick_maps[slot];
    if (m.base == base && m.nx == op.nx && m.ny == op.ny && m.nz == op.nz && m.ylen == box_y && m.zlen == box_z &&
        m.xlen == box_x)
        return true;
    const TmapEncodeFn enc = tmap_encode_fn();
    if (!enc || ((uintptr_t)base & 15) || (ld & 1)) return false;
    const cuuint64_t gdim[4] = {(cuuint64_t)op.nx, (cuuint64_t)op.ny, (cuuint64_t)op.nz, (cuuint64_t)ncols};
    const cuuint64_t gstr[3] = {(cuuint64_t)op.nx * 8, (cuuint64_t)op.nx * op.ny * 8, (cuuint64_t)ld * 8};
    const cuuint32_t box[4] = {(cuuint32_t)box_x, (cuuint32_t)box_y, (cuuint32_t)box_z, 1};
    const cuuint32_t est[4] = {1, 1, 1, 1};
    const CUresult r = enc(&m.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double *>(base), gdim, gstr, box, est,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        m.base = nullptr;
        return false;
    }
    m.base = base;
    m.nx = op.nx;
    m.ny = op.ny;
    m.nz = op.nz;
    m.ylen = box_y;
    m.zlen = box_z;
    m.xlen = box_x;
    return true;
}

constexpr int64_t BRICK_AUTO_MIN_N = 65536;   // brick = auto: grids larger than the cluster Lanczos kernel's range

// the brick decomposition of this operator under PHIPM_OPT_BRICK (0 off, 1 auto: x-lines that fill >= 3/4 of
// their 64-point warp segments, 2 whenever one exists)
bool brick_plan(phipm_ctx *c, const StencilOp &op, BrickGeom &g)
{
    const int mode = opt(c, PHIPM_OPT_BRICK);
    if (!mode || op.dim != 3 || op.diag) return false;
    if (!brick_geometry(op.nx, op.ny, op.nz, c->sm_count, c->smem_optin - 2048, g)) return false;
    if (mode == 1 && 4 * op.nx < 3 * 64 * g.nseg) return false;
    return g.py * g.pz <= c->pstride;
}

// Lanczos on 3-D bricks staged by tensor-map TMA (persist_brick.cuh).  PHIPM_OPT_BRICK: 0 off, 1 auto
// (3-D 7-point grids whose x-lines fill >= 3/4 of their 64-point warp segments), 2 whenever a brick
// decomposition exists
bool try_persist_brick(phipm_ctx *c, const StencilOp &op, int k0, int k1, double bthr, double bytes, int &rc)
{
    BrickGeom g;
    if (!brick_plan(c, op, g)) return false;
    const bool halo = opt(c, PHIPM_OPT_BRICK_HALO) != 0;   // interior resident in shared memory, halo copies only
    const bool ragged = g.nseg * 64 != op.nx;
    if (halo) {
        if (!brick_tensor_map(c, 3, c->V, c->m_max + 1, c->ldv, op, g, g.ylen, 1, op.nx) ||
            !brick_tensor_map(c, 4, c->V, c->m_max + 1, c->ldv, op, g, 1, g.zlen, op.nx))
            return false;
    } else if (!brick_tensor_map(c, 0, c->V, c->m_max + 1, c->ldv, op, g)) {
        return false;
    }
    const size_t smem = halo ? brick_halo_smem_bytes(g) : brick_smem_bytes(g);
    const int grid = g.py * g.pz;
    const auto kfn = ragged ? krylov_brick_tm_kernel<true> : krylov_brick_tm_kernel<false>;
    const auto hfn = ragged ? krylov_brick_halo_kernel<true> : krylov_brick_halo_kernel<false>;
    int occ = 0;
    if ((halo ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, hfn, SNT, smem)
              : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, SNT, smem)) != cudaSuccess ||
        occ < 1 || grid > occ * c->sm_count || grid > c->pstride) {
        cudaGetLastError();
        return false;
    }
    PersistArgs a;
    a.k0 = k0;
    a.k1 = k1;
    a.symmetric = 1;
    a.bthr = bthr;
    a.rpc = 0;
    a.flag = c->counter + 2;
    a.abort = c->counter + 3;
    a.exit_ctr = c->counter + 4;
    a.timeout_ns = 2000000000ull;
    a.dbg = nullptr;
    const size_t need = (size_t)2 * (k1 - k0) * grid * 2;
    if (c->pclk_d && c->pclk_used + need <= PCLK_CAP) {
        a.dbg = c->pclk_d + c->pclk_used;
        c->pclk_recs.push_back({grid, k1 - k0, (long long)c->pclk_used});
        c->pclk_used += need;
    }
    rc = PHIPM_OK;
    if (!coop_reset(c)) {
        rc = set_err(c, PHIPM_ECUDA, "persist: memset failed");
        return true;
    }
    ProfRec r;
    prof_begin(c, r, PC_SPMV, bytes, k1 - k0);
    const cudaError_t e =
        halo ? launch_coop(c, hfn, grid, SNT, smem, c->brick_maps[3].map, c->brick_maps[4].map, op, g, a, make_work(c))
             : launch_coop(c, kfn, grid, SNT, smem, c->brick_maps[0].map, op, g, a, make_work(c));
    prof_end(c, r);
    c->acc.launches++;
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    c->krylov_path = PHIPM_PATH_BRICK;
    return true;
}

// The whole w-recurrence of a step in one cooperative kernel (persist_wrec.cuh) for stencil
// operators with n > SMALL_N (PHIPM_OPT_WREC = 0 disables).  Returns true if it launched (rc = status).
template <class Op>
bool launch_wrec_persist(phipm_ctx *, const Op &, const WrecArgs &, double, int &) { return false; }

using WrecFn = void (*)(StencilOp, WrecArgs, PersistArgs, Work);

WrecFn wrec_fn(const StencilOp &op)
{
    switch ((op.dim == 2 && op.diag) ? 4 : op.dim) {
    case 1: return wrec_persist_kernel<1>;
    case 2: return wrec_persist_kernel<2>;
    case 3: return wrec_persist_kernel<3>;
    default: return wrec_persist_kernel<4>;
    }
}

// the w-recurrence on TMA-staged bricks (persist_brick.cuh: wrec_brick_kernel); the u-terms are read with
// 16-byte loads, so every u pointer must be 16-byte aligned (else the contiguous-range kernel)
bool try_wrec_brick(phipm_ctx *c, const StencilOp &op, const WrecArgs &w, double bytes, int &rc)
{
    if (op.n <= BRICK_AUTO_MIN_N && opt(c, PHIPM_OPT_BRICK) != 2) return false;
    BrickGeom g;
    if (!brick_plan(c, op, g)) return false;
    for (int j = 0; j < w.p; j++)
        for (int i = 0; i < w.nz[j]; i++)
            if ((uintptr_t)w.z[j][i] & 15) return false;
    if (!brick_tensor_map(c, 1, c->W, c->p_max + 1, c->ldv, op, g)) return false;
    if (!brick_tensor_map(c, 2, w.x0, 1, op.n + (op.n & 1), op, g)) return false;
    const size_t smem = brick_smem_bytes(g);
    const int grid = g.py * g.pz;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, wrec_brick_kernel, SNT, smem) != cudaSuccess || occ < 1 ||
        grid > occ * c->sm_count) {
        cudaGetLastError();
        return false;
    }
    PersistArgs a{};
    a.flag = c->counter + 2;
    a.abort = c->counter + 3;
    a.exit_ctr = c->counter + 4;
    a.timeout_ns = 2000000000ull;
    // PHIPM_KCLOCKS: 2 stamps per CTA per pass (recorded as (p + 1) / 2 two-phase steps)
    const size_t need = (size_t)2 * ((w.p + 1) / 2) * grid * 2;
    if (c->pclk_d && c->pclk_used + need <= PCLK_CAP) {
        a.dbg = c->pclk_d + c->pclk_used;
        cudaMemsetAsync(a.dbg, 0, need * sizeof(unsigned long long), c->stream);
        c->pclk_recs.push_back({grid, (w.p + 1) / 2, (long long)c->pclk_used});
        c->pclk_used += need;
    }
    rc = PHIPM_OK;
    if (!coop_reset(c)) {
        rc = set_err(c, PHIPM_ECUDA, "wrec: memset failed");
        return true;
    }
    ProfRec r;
    prof_begin(c, r, PC_SPMV, bytes, 0);
    const cudaError_t e = launch_coop(c, wrec_brick_kernel, grid, SNT, smem, c->brick_maps[2].map, c->brick_maps[1].map,
                                      op, g, w, a, make_work(c));
    prof_end(c, r);
    c->acc.launches++;
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    c->wrec_path = PHIPM_PATH_BRICK;
    return true;
}

template <>
bool launch_wrec_persist<StencilOp>(phipm_ctx *c, const StencilOp &op, const WrecArgs &w, double bytes, int &rc)
{
    if (!opt(c, PHIPM_OPT_WREC) || op.n <= SMALL_N || w.p < 1) return false;
    if (try_wrec_brick(c, op, w, bytes, rc)) return true;
    constexpr int TILE_ = SNT * 4;
    int grid;
    int64_t rpc;
    const int slots = (int)std::max<int64_t>(1, std::min<int64_t>(c->sm_count, (op.n + TILE_ / 2 - 1) / (TILE_ / 2)));
    balance(c, op.n, slots, grid, rpc);
    const size_t smem = wrec_smem_bytes(halo_capacity(op.dim, op.nx, TILE_));
    if (smem > c->smem_optin) return false;
    const WrecFn kfn = wrec_fn(op);
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, SNT, smem) != cudaSuccess || occ < 1 ||
        grid > occ * c->sm_count) {
        cudaGetLastError();
        return false;
    }
    PersistArgs a{};
    a.rpc = rpc;
    a.flag = c->counter + 2;
    a.abort = c->counter + 3;
    a.exit_ctr = c->counter + 4;
    a.timeout_ns = 2000000000ull;
    rc = PHIPM_OK;
    if (!coop_reset(c)) {
        rc = set_err(c, PHIPM_ECUDA, "wrec: memset failed");
        return true;
    }
    ProfRec r;
    prof_begin(c, r, PC_SPMV, bytes, 0);
    const cudaError_t e = launch_coop(c, kfn, grid, SNT, smem, op, w, a, make_work(c));
    prof_end(c, r);
    c->acc.launches++;
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    c->wrec_path = PHIPM_PATH_PERSIST_SMEM;
    return true;
}

template <>
bool launch_persist<StencilOp>(phipm_ctx *c, const StencilOp &op, double bytes_op, bool symmetric, int k0, int k1,
                               double bthr, int &rc)
{
    // PHIPM_OPT_PERSIST: 0 off, 1 (default) auto, 2 always.  Auto: n <= 2^19, or a Lanczos extension of
    // any size; measured with the all-reduce phase end (profiles/round1): c2 +17 %, c4 +3.6 %, while
    // c3 (Arnoldi, n = 1M) is even with the two-kernel path, whose PDL overlap it loses
    const int env = opt(c, PHIPM_OPT_PERSIST);
    if (env == 0 || op.n <= SMALL_N) return false;
    if (env == 1 && op.n > ((int64_t)1 << 19) && !symmetric) return false;
    double bytes = 0.0;
    const double n = (double)op.n;
    for (int j = k0; j < k1; j++) bytes += bytes_op + 8.0 * n * (symmetric ? 4.0 : 2.0 * j + 3.0);
    // (small grids keep the 2048-row tiles: a 4096-row tile would leave half a CTA's threads idle)
    // (auto: above the cluster kernel's range; measured 9-11 % faster per step than the shared-memory
    // persistent kernel on 3-D grids of 110K-262K rows, tools/brick_small.py)
    if (symmetric && (op.n > BRICK_AUTO_MIN_N || opt(c, PHIPM_OPT_BRICK) == 2) &&
        try_persist_brick(c, op, k0, k1, bthr, bytes, rc))
        return true;
    if (symmetric && op.n >= (int64_t)SNT * 4 * c->sm_count / 2 && try_persist_tm(c, op, k0, k1, bthr, bytes, rc))
        return true;
    // largest tile that fits (halo + the CTA's y + dot partials); RPT = 8 would spill
    if (op.n >= (int64_t)SNT * 4 * c->sm_count / 2 && try_persist_rpt<4>(c, op, symmetric, k0, k1, bthr, bytes, rc))
        return true;
    return try_persist_rpt<2>(c, op, symmetric, k0, k1, bthr, bytes, rc);
}

using ClusterLzFn = void (*)(StencilOp, SmallArgs, ClArgs, Work);

template <int NT, int R>
ClusterLzFn cluster_lz_fn(int dc)
{
    switch (dc) {
    case 1: return krylov_cluster_lanczos_kernel<NT, R, 1>;
    case 2: return krylov_cluster_lanczos_kernel<NT, R, 2>;
    case 3: return krylov_cluster_lanczos_kernel<NT, R, 3>;
    default: return krylov_cluster_lanczos_kernel<NT, R, 4>;
    }
}

// Lanczos extension of a stencil on one thread-block cluster (persist_cl.cuh); false: not applicable
// (CSR operators, sizes whose slice or halo does not fit, a refused cluster launch)
struct ClPlan {
    int cs, nt;
    int64_t rpc, reach, blen;
    ClusterLzFn kfn;
};

// whether (and how) the cluster Lanczos kernel takes a stencil extension
inline bool cluster_lz_plan(const phipm_ctx *c, const StencilOp &op, ClPlan &pl)
{
    const int o = opt(c, PHIPM_OPT_CLUSTER_LZ);
    if (o == 0) return false;
    const int64_t n = op.n;
    pl.reach = op.dim == 3 ? (int64_t)op.nx * op.ny : op.dim == 2 ? op.nx + (op.diag ? 1 : 0) : 1;
    if (o == 1) {
        // auto: above the single-CTA sizes, about 4096 rows per CTA
        if (n <= SMALL_N || n > (int64_t)CLZ_MAXCS * 4096) return false;
        pl.cs = 2;
        while (pl.cs < CLZ_MAXCS && (n + pl.cs - 1) / pl.cs > 4096) pl.cs *= 2;
    } else {
        pl.cs = o < 0 ? 1 : o;
    }
    pl.rpc = (n + pl.cs - 1) / pl.cs;
    const int64_t last = n - (int64_t)(pl.cs - 1) * pl.rpc;
    if (pl.cs > 1 && (last < pl.reach || pl.rpc < pl.reach)) return false;
    pl.blen = cl_buf_len(op, pl.rpc, (int)pl.reach, pl.cs);
    if ((size_t)pl.blen * sizeof(double) + 4096 > c->smem_optin) return false;
    const int dc = (op.dim == 2 && op.diag) ? 4 : op.dim;
    if (pl.rpc <= 256 * 4) { pl.kfn = cluster_lz_fn<256, 4>(dc); pl.nt = 256; }
    else if (pl.rpc <= 512 * 8) { pl.kfn = cluster_lz_fn<512, 8>(dc); pl.nt = 512; }
    else return false;
    return true;
}

template <class Op>
bool try_cluster_lz(phipm_ctx *, const Op &, double, int, int, double)
{
    return false;
}

template <>
bool try_cluster_lz<StencilOp>(phipm_ctx *c, const StencilOp &op, double bytes_op, int k0, int k1, double bthr)
{
    ClPlan pl;
    if (k1 <= k0 || !cluster_lz_plan(c, op, pl)) return false;
    const int64_t n = op.n;
    const int cs = pl.cs, nt = pl.nt;
    const size_t smem = (size_t)pl.blen * sizeof(double);
    const ClusterLzFn kfn = pl.kfn;
    SmallArgs sa;
    sa.k0 = k0;
    sa.k1 = k1;
    sa.symmetric = 1;
    sa.orth = 0;
    sa.bthr = bthr;
    ClArgs ca;
    ca.rpc = pl.rpc;
    ca.reach = (int)pl.reach;
    ca.cs = cs;
    ca.blen = (int)pl.blen;
    double bytes = 0.0;
    for (int j = k0; j < k1; j++) bytes += bytes_op + 8.0 * (double)n * 4.0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = c->pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = cs;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = cs > 1 ? 2 : 1;
    ProfRec r;
    prof_begin(c, r, PC_SPMV, bytes, k1 - k0);
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kfn, op, sa, ca, make_work(c));
    prof_end(c, r);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    c->acc.launches++;
    return true;
}

// Speculative Krylov extension (PHIPM_OPT_SPEC): an extension runs on a second stream, concurrently
// with the exponential of the current attempt, when it occupies few SMs (the single-CTA kernels,
// n <= SMALL_N, or the cluster Lanczos kernel): the extension then hides behind the exponential
// instead of following the host's decision.
template <class Op>
bool spec_path(const phipm_ctx *c, const Op &op, bool symmetric)
{
    if (!opt(c, PHIPM_OPT_SPEC)) return false;
    if (op.n <= SMALL_N) return true;
    if constexpr (std::is_same<Op, StencilOp>::value) {
        ClPlan pl;
        return symmetric && cluster_lz_plan(c, op, pl);
    }
    return false;
}

// the launch helpers enqueue on c->stream: point it at the second stream for one enqueue
struct OnStream2 {
    phipm_ctx *c;
    cudaStream_t saved;
    explicit OnStream2(phipm_ctx *cc) : c(cc), saved(cc->stream) { c->stream = c->stream2; }
    ~OnStream2() { c->stream = saved; }
};

template <class Op>
int enqueue_krylov_stream(phipm_ctx *c, const Op &op, double bytes_op, bool symmetric, int orth, int k0, int k1,
                          double bthr);

// PHIPM_OPT_GRAPH: the two-kernel extension k0 -> k1 (2(k1 - k0) launches, more with CGS2) captured once as a
// CUDA graph on the context's private stream and replayed from a per-context cache keyed by the operator,
// k0, k1, the breakdown threshold and the context options (everything the captured launches depend on; the
// workspace pointers are the context's own).  The kernels read all step state from device memory, so a
// replay is the same computation as the stream launches (same kernels, arguments, order).
template <class Op>
int enqueue_krylov_graph(phipm_ctx *c, const Op &op, double bytes_op, bool symmetric, int orth, int k0, int k1,
                         double bthr)
{
    std::vector<unsigned char> key(sizeof(Op) + 5 * sizeof(int) + sizeof(double) + sizeof(c->opt) + sizeof(void *));
    unsigned char *kp = key.data();
    auto put = [&](const void *p, size_t b) {
        memcpy(kp, p, b);
        kp += b;
    };
    const int sym = symmetric ? 1 : 0;
    const int tag = std::is_same<Op, StencilOp>::value ? 1 : std::is_same<Op, CsrOp>::value ? 2 : 3;
    const void *sp = (const void *)c->stream;
    put(&op, sizeof(Op));
    put(&tag, sizeof(int));
    put(&sym, sizeof(int));
    put(&orth, sizeof(int));
    put(&k0, sizeof(int));
    put(&k1, sizeof(int));
    put(&bthr, sizeof(double));
    put(c->opt, sizeof(c->opt));
    put(&sp, sizeof(void *));
    for (auto &g : c->graphs)
        if (g.key == key) {
            CK(cudaGraphLaunch(g.exec, c->stream));
            c->acc.launches += g.nlaunch;
            return PHIPM_OK;
        }
    // capture on the private stream (the caller's stream may be the legacy stream, which cannot capture)
    const int64_t l0 = c->acc.launches;
    cudaGraph_t graph = nullptr;
    int rc;
    {
        OnStream2 on2(c);
        CK(cudaStreamBeginCapture(c->stream2, cudaStreamCaptureModeThreadLocal));
        rc = enqueue_krylov_stream(c, op, bytes_op, symmetric, orth, k0, k1, bthr);
        const cudaError_t e = cudaStreamEndCapture(c->stream2, &graph);
        if (!rc && e != cudaSuccess) rc = set_err(c, PHIPM_ECUDA, "graph capture: %s", cudaGetErrorString(e));
    }
    if (rc) {
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        return rc;
    }
    GraphRec g;
    g.key = key;
    g.nlaunch = c->acc.launches - l0;
    c->acc.launches = l0;
    const cudaError_t e = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return set_err(c, PHIPM_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
    if (c->graphs.size() >= 64) {
        cudaGraphExecDestroy(c->graphs.front().exec);
        c->graphs.erase(c->graphs.begin());
    }
    c->graphs.push_back(g);
    CK(cudaGraphLaunch(g.exec, c->stream));
    c->acc.launches += g.nlaunch;
    return PHIPM_OK;
}

template <class Op>
int enqueue_krylov(phipm_ctx *c, const Op &op, double bytes_op, bool symmetric, int orth, int k0, int k1, double bthr)
{
    if (symmetric && try_cluster_lz(c, op, bytes_op, k0, k1, bthr)) {
        c->krylov_path = PHIPM_PATH_CLUSTER;
        return PHIPM_OK;
    }
    const int64_t n = op.n;
    if (n <= SMALL_N && k1 > k0) {
        c->krylov_path = PHIPM_PATH_SINGLE_CTA;
        // small problems: the whole extension in one single-CTA kernel (small.cuh)
        SmallArgs sa;
        sa.k0 = k0;
        sa.k1 = k1;
        sa.symmetric = symmetric ? 1 : 0;
        sa.orth = orth;
        sa.bthr = bthr;
        double bytes = 0.0;
        for (int j = k0; j < k1; j++)
            bytes += bytes_op + 8.0 * (double)n * (symmetric ? 4.0 : 2.0 * j + 3.0);
        ProfRec r;
        prof_begin(c, r, PC_SPMV, bytes, k1 - k0);
        if (symmetric && n <= SLZ_NT * SLZ_R && opt(c, PHIPM_OPT_SMALL_LZ))
            launch_k(c, krylov_small_lanczos_kernel<Op>, 1, SLZ_NT, (size_t)n * sizeof(double), op, sa, make_work(c));
        else
            launch_k(c, krylov_small_kernel<Op>, 1, SMALL_NT, (size_t)n * sizeof(double), op, sa, make_work(c));
        prof_end(c, r);
        c->acc.launches++;
        CK(cudaGetLastError());
        return PHIPM_OK;
    }
    if (k1 > k0 && orth != PHIPM_ORTH_CGS2) {
        int rc = PHIPM_OK;
        if (launch_persist(c, op, bytes_op, symmetric, k0, k1, bthr, rc)) return rc;
    }
    c->krylov_path = PHIPM_PATH_TWO_KERNEL;
    if (k1 > k0 && opt(c, PHIPM_OPT_GRAPH) && !c->prof && !c->kclk_d)
        return enqueue_krylov_graph(c, op, bytes_op, symmetric, orth, k0, k1, bthr);
    return enqueue_krylov_stream(c, op, bytes_op, symmetric, orth, k0, k1, bthr);
}

// the two-kernel path of an extension: per step the fused SpMV + dots and the update + norm
template <class Op>
int enqueue_krylov_stream(phipm_ctx *c, const Op &op, double bytes_op, bool symmetric, int orth, int k0, int k1,
                          double bthr)
{
    const int64_t n = op.n;
    // Arnoldi (CGS): lagged normalisation (PHIPM_OPT_LAG = 0 disables).  Step j > k0's SpMV works on the raw
    // v~_j and also reduces ||v~_j||^2 (free: the x tile is on chip), its finalize derives sigma_j and
    // h_{j,j-1}; so the update passes need no grid reduction except the extension's last one, which
    // provides h_{k1,k1-1} and sigma_{k1} for the exponential.
    const int env_lag = opt(c, PHIPM_OPT_LAG);
    // (stencils only: a CSR SpMV would have to re-read its own x rows for the norm; c5 measured even)
    const bool lag = env_lag && !symmetric && orth == PHIPM_ORTH_CGS && std::is_same<Op, StencilOp>::value;
    for (int j = k0; j < k1; j++) {
        double *vj = c->V + (int64_t)j * c->ldv;
        double *vn = c->V + (int64_t)(j + 1) * c->ldv;
        const bool lag_j = lag && j > k0;                   // sigma_j still unknown at this SpMV
        SpmvArgs s = spmv0();
        s.x = vj;
        s.xscale = c->sigma + j;
        s.y = c->Y;
        s.V = c->V;
        s.ldv = c->ldv;
        s.ynorm = 1;
        s.j = j;
        s.check_brk = 1;
        AxpyArgs u = axpy0();
        u.out = vn;
        u.base = c->Y;
        u.a0h = 1.0;
        u.V = c->V;
        u.ldv = c->ldv;
        u.g = c->g;
        u.gsign = -1.0;
        u.onorm = 1;
        u.fin = FIN_NORM;
        u.j = j;
        u.check_brk = 1;
        u.bthr = bthr;
        u.rev = 1;
        if (symmetric) {
            // Alg. 2: w = A v_j - t_{j,j-1} v_{j-1}; t_jj = v_j^T w; w -= t_jj v_j
            if (j > 0) {
                s.nz = 1;
                s.z[0] = c->V + (int64_t)(j - 1) * c->ldv;
                s.zc[0] = -1.0;
                s.zcd[0] = &c->st->lz;
            }
            s.d0 = j;
            s.nd = 1;
            s.xcol = 0;                      // v_j is x
            s.fin = FIN_LANCZOS;
            u.c0 = j;
            u.nc = 1;
            u.lanczos = 1;
        } else {
            // Alg. 1 (classical Gram-Schmidt form): h = V_j^T w; w -= V_j h
            s.d0 = 0;
            s.nd = j + 1;
            s.xcol = j;                      // v_j is x
            s.fin = FIN_ARNOLDI;
            u.c0 = 0;
            u.nc = j + 1;
            if (lag_j) {
                s.xscale = nullptr;          // raw A v~_j; sigma_j is applied in the finalize / update
                s.xnorm = 1;
                s.bthr = bthr;
                s.fin = FIN_ARNOLDI_LAG;
                u.a0d = c->sigma + j;
            }
            if (lag && j + 1 < k1) {         // the next SpMV reduces ||v~_{j+1}||^2
                u.onorm = 0;
                u.fin = FIN_NONE;
            }
        }
        // deferred finalize (PHIPM_OPT_DEFER): the streaming SpMV leaves its partials to the update kernel
        s.defer = opt(c, PHIPM_OPT_DEFER) && n > SMALL_N && !s.anorm &&
                  (s.fin == FIN_ARNOLDI || s.fin == FIN_LANCZOS || s.fin == FIN_ARNOLDI_LAG);
        c->defer_nb = 0;
        int rc = launch_spmv(c, op, s, bytes_op);
        if (rc) return rc;
        if (s.defer && c->defer_nb > 0) {
            u.dfin = s.fin;
            u.dnb = c->defer_nb;
            u.dnd = s.nd;
            u.dnv = s.nd + s.ynorm + s.xnorm;
            u.dj = j;
            u.dbthr = s.bthr;
        }
        rc = launch_axpy(c, n, u, PC_ORTH);
        if (rc) return rc;
        if (!symmetric && orth == PHIPM_ORTH_CGS2) {
            SpmvArgs d = spmv0();
            d.x = vn;
            d.V = c->V;
            d.ldv = c->ldv;
            d.d0 = 0;
            d.nd = j + 1;
            d.fin = FIN_REORTH;
            d.j = j;
            d.check_brk = 1;
            rc = launch_spmv(c, IdentOp{n}, d, 8.0 * (double)n);
            if (rc) return rc;
            AxpyArgs r = u;
            r.base = vn;
            r.dfin = 0;                      // (the reorthogonalisation SpMV finalizes itself)
            rc = launch_axpy(c, n, r, PC_ORTH);
            if (rc) return rc;
        }
    }
    return PHIPM_OK;
}

// ||u_k||_inf of u[k0..k1).  publish = true: the result goes to mapped pinned memory with a sequence
// number the host spins on (no copy node in the stream); otherwise it is copied to raw_h
int enqueue_maxabs_u(phipm_ctx *c, int64_t n, const double *const *u, int k0, int k1, bool publish, bool side = false)
{
    MaxAbsArgs ma;
    memset(&ma, 0, sizeof(ma));
    ma.nv = k1 - k0;
    for (int k = k0; k < k1; k++) ma.x[k - k0] = u[k];
    if (publish) {
        ma.pub = c->mx_d->v;
        ma.pub_seq = &c->mx_d->seq;
        ma.seq = ++c->mx_seq;
    }
    const int grid = grid_for(c, (n + NT - 1) / NT, c->occ_axpy);
    Work wk = make_work(c);
    if (side) {
        // one vector, published: on stream2 with private scratch, concurrent with the main stream's kernels
        wk.part = c->part_mx;
        wk.counter = c->counter_mx;
        wk.out_raw = c->raw_mx;
    }
    maxabs_kernel<<<grid, NT, 0, side ? c->stream2 : c->stream>>>(n, ma, wk);
    c->acc.launches++;
    CK(cudaGetLastError());
    if (!publish)
        CK(cudaMemcpyAsync(c->raw_h + k0, c->raw, ma.nv * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    return PHIPM_OK;
}

// Eq. (wrecurrence): w_0 = u_k, w_j = A w_{j-1} + sum_l t_k^l/l! u_{j+l}; w_p -> V[:,0]
// x0 = w_0 = u_k; ldx0 > 0: x0 is the caller's u_0 (n even, 16-B aligned), halos clamp to n
template <class Op>
int enqueue_wrec_op(phipm_ctx *c, const Op &op, double bytes_op, int p, const double *const *u, double tk,
                    const double *x0, int64_t ldx0)
{
    const int64_t n = op.n;
    if (p == 0) {
        AxpyArgs a = axpy0();
        a.out = c->V;
        a.base = x0;
        a.a0h = 1.0;
        a.V = c->V;
        a.ldv = c->ldv;
        a.onorm = 1;
        a.fin = FIN_SEED;
        return launch_axpy(c, n, a, PC_OTHER);
    }
    {
        // one cooperative kernel for all p SpMVs (stencils); else p streaming launches
        WrecArgs wa;
        memset(&wa, 0, sizeof(wa));
        wa.p = p;
        wa.x0 = x0;
        wa.ldx = ldx0 ? ldx0 : c->ldv;
        wa.W = c->W;
        double bytes = 0.0;
        for (int j = 1; j <= p; j++) {
            double coef = 1.0;
            int nz = 0;
            for (int l = 0; l <= p - j; l++) {
                if (l > 0) coef = coef * tk / (double)l;
                if (l > 0 && coef == 0.0) continue;
                wa.z[j - 1][nz] = u[j + l];
                wa.zc[j - 1][nz] = coef;
                nz++;
            }
            wa.nz[j - 1] = nz;
            bytes += bytes_op + 8.0 * (double)n * nz;
        }
        int rc = PHIPM_OK;
        c->wrec_path = PHIPM_PATH_NONE;
        if (p <= WREC_MAXP && launch_wrec_persist(c, op, wa, bytes, rc)) return rc;
    }
    for (int j = 1; j <= p; j++) {
        SpmvArgs s = spmv0();
        s.x = (j == 1) ? x0 : c->W + (int64_t)(j - 1) * c->ldv;
        if (j == 1 && ldx0) s.ldx = ldx0;
        s.y = (j == p) ? c->V : c->W + (int64_t)j * c->ldv;
        // terms whose coefficient t_k^l / l! is exactly 0 (the first step, t_k = 0: only u_j)
        // are not read: adding 0 * u changes no sum
        double coef = 1.0;
        s.nz = 0;
        for (int l = 0; l <= p - j; l++) {
            if (l > 0) coef = coef * tk / (double)l;
            if (l > 0 && coef == 0.0) continue;
            s.z[s.nz] = u[j + l];
            s.zc[s.nz] = coef;
            s.nz++;
        }
        s.ynorm = (j == p);
        s.fin = (j == p) ? FIN_SEED : FIN_NONE;
        if (j == 1 && c->fuse_anorm) {
            s.anorm = 1;
            s.anorm_pub = &c->mx_d->anorm;
            s.anorm_seq = &c->mx_d->aseq;
            s.anorm_seqv = ++c->mx_aseq;
            c->fuse_anorm = false;
        }
        int rc = launch_spmv(c, op, s, bytes_op);
        if (rc) return rc;
    }
    return PHIPM_OK;
}

// ---------------------------------------------------------------------------------------------
// the solve (Algorithm 3)

// ---------------------------------------------------------------------------------------------
// device-driven solve of a small symmetric problem (solve_small.cuh, PHIPM_OPT_DEVSOLVE)

constexpr int SS_ATT_CAP = 65536;

template <class Op>
bool devsolve_path(const phipm_ctx *c, const Op &op, const Problem &P, const phipm_opts &o, double normA, int p)
{
    return opt(c, PHIPM_OPT_DEVSOLVE) && op.n <= SMALL_N && P.symmetric && o.expm_method == PHIPM_EXPM_TAYLOR &&
           normA >= 0.0 && !c->prof && p + 1 <= SS_MAXU;
}

template <class Op, int R>
void ss_set_smem(int mx)
{
    cudaFuncSetAttribute(small_solve_kernel<Op, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
}

int finish_small_dev(phipm_ctx *c, phipm_stats &S);

template <class Op>
int solve_small_dev(phipm_ctx *c, const Op &op, double t_end, double normA, double bthr, int p,
                    const double *const *u, const phipm_opts &o, const Problem &P, double *w, phipm_stats &S)
{
    const int64_t n = op.n;
    if (!c->ss_att_d) {
        if (cudaMalloc((void **)&c->ss_att_d, sizeof(SsAttempt) * SS_ATT_CAP) != cudaSuccess ||
            cudaHostAlloc((void **)&c->ss_out_h, sizeof(SsOut), cudaHostAllocMapped) != cudaSuccess ||
            cudaHostGetDevicePointer((void **)&c->ss_out_d, c->ss_out_h, 0) != cudaSuccess)
            return set_err(c, PHIPM_ENOMEM, "device solve: allocation failed");
    }
    SmallSolveArgs a;
    memset(&a, 0, sizeof(a));
    a.t_end = t_end;
    a.tol = o.tol;
    a.normA = normA;
    a.bthr = bthr;
    a.p = p;
    a.m_init = o.m_init;
    a.P = P;
    for (int k = 0; k <= p; k++) a.u[k] = u[k];
    a.w = w;
    a.ucur = c->U;
    a.W = c->W;
    a.scratch = c->scratch;
    a.comb = c->comb;
    a.combd = c->combd;
    a.res = reinterpret_cast<AttemptResult *>(c->raw);   // device-global slot (raw has MAXD+2 doubles)
    a.att = c->ss_att_d;
    a.att_cap = SS_ATT_CAP;
    a.out = c->ss_out_d;
    a.clk = c->expm_clk_d;                               // PHIPM_EXPM_CLOCKS: phase cycles of the solve
    const size_t dyn = c->smem_optin - 8192;
    const size_t vbytes = (size_t)((n + 15) & ~15) * sizeof(double);
    a.esm_cap = (int)((dyn - vbytes) / sizeof(double));
    const int R = (int)((n + SS_NT - 1) / SS_NT);
    void (*kfn)(Op, SmallSolveArgs, Work) = R <= 2 ? small_solve_kernel<Op, 2>
                                          : R <= 4 ? small_solve_kernel<Op, 4>
                                          : R <= 8 ? small_solve_kernel<Op, 8>
                                                   : small_solve_kernel<Op, 16>;
    c->ss_out_h->status = -1;
    CK(launch_k(c, kfn, 1, SS_NT, dyn, op, a, make_work(c)));
    c->acc.launches++;
    if (c->defer) {                                  // batch fast path: collected by finish_small_dev
        c->deferred = true;
        return PHIPM_OK;
    }
    return finish_small_dev(c, S);
}

// wait for a device-driven solve and read its stats / status / attempt count
int finish_small_dev(phipm_ctx *c, phipm_stats &S)
{
    c->deferred = false;
    int rc = sync(c);
    if (rc) return rc;
    SsOut R_;
    memcpy(&R_, (const void *)c->ss_out_h, sizeof(R_));
    S.nsteps = R_.nsteps;
    S.nreject = R_.nreject;
    S.nspmv = R_.nspmv;
    S.nexpm = R_.nexpm;
    S.m_last = R_.m_last;
    S.m_peak = R_.m_peak;
    S.t_reached = R_.t_reached;
    c->attempts.clear();
    c->nattempts = R_.nattempts;
    c->ss_att_pending = std::min(R_.nattempts, SS_ATT_CAP);
    switch (R_.status) {
    case SS_OK: return PHIPM_OK;
    case SS_ABORT: return set_err(c, PHIPM_ECUDA, "device solve: aborted");
    case SS_NONFINITE: return set_err(c, PHIPM_ENONFINITE, "non-finite value in the device solve");
    case SS_SINGULAR: return set_err(c, PHIPM_ESINGULAR, "singular denominator");
    case SS_STEP: return set_err(c, PHIPM_ESTEP, "step size control failed at t = %g", R_.t_reached);
    default: return set_err(c, PHIPM_ECUDA, "device solve: no result (status %d)", R_.status);
    }
}

template <class Op>
int solve_impl(phipm_ctx *c, double t_end, const Op &op, double bytes_op, int64_t NA, double normA_in, int p,
               const double *const *u, const phipm_opts &o, double *w, phipm_stats *stats)
{
    const int64_t n = op.n;
    double normA = normA_in;
    phipm_stats S{};
    S.t_reached = 0.0;
    c->attempts.clear();
    c->nattempts = 0;
    c->ss_att_pending = 0;
    // join a speculative extension still running on stream2 (stream order from here on)
    auto join_spec = [&]() {
        if (c->spec_pending) {
            cudaStreamWaitEvent(c->stream, c->ev_spec, 0);
            c->spec_pending = false;
        }
    };
    auto finish = [&](int rc) {
        join_spec();
        if (c->mx_side_pending) {                      // an error return before ||u_0||_inf was read
            cudaStreamSynchronize(c->stream2);
            c->mx_side_pending = false;
        }
        if (stats) *stats = S;
        return rc;
    };
    join_spec();                       // (an earlier solve that ended in an error may have left one)
    if (t_end == 0.0) {
        if (w != u[0]) CK(cudaMemcpyAsync(w, u[0], n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
        int rc = sync(c);
        return finish(rc);
    }
    auto enqueue_maxabs = [&](int k0, int k1, bool publish) { return enqueue_maxabs_u(c, n, u, k0, k1, publish); };
    auto enqueue_wrec = [&](double tk, const double *x0, int64_t ldx0) {
        return enqueue_wrec_op(c, op, bytes_op, p, u, tk, x0, ldx0);
    };

    Problem P;
    P.p = p;
    P.n = n;
    P.NA = NA;
    P.symmetric = o.symmetric != 0;
    P.m_max = (int)std::min<int64_t>(o.m_max, n);
    P.fixed_m = o.fixed_m != 0;
    P.eq6_variant = o.eq6_variant != 0;
    int m = std::min(o.m_init, P.m_max);
    const double mbar = 0.5 * ((double)o.m_init + (double)P.m_max);
    // normA < 0: ||A||_inf is computed by the first SpMV (fused CSR path); the Krylov kernels enqueued
    // before the host knows it take the breakdown threshold from device memory (bthr < 0)
    const bool anorm_dev = normA < 0.0;
    const double bthr = anorm_dev ? -1.0 : (double)n * EPS_MACH * normA;
    if (devsolve_path(c, op, P, o, normA, p)) return finish(solve_small_dev(c, op, t_end, normA, bthr, p, u, o, P, w, S));

    // b_inf of Eq. (tau_0) = ||u_0||_inf, or the first nonzero ||u_k||_inf (R7); all zero -> w = 0.
    // ||u_0||_inf is read back through an event, and the first step's w-recurrence and initial
    // Krylov extension -- which do not depend on it: tau enters only the exponential -- are
    // enqueued before the host waits for it.  The other u_k are only read when u_0 = 0.
    const bool spin_binf = !c->prof;                 // profiling collects events at a stream sync instead
    // PHIPM_OPT_SIDE_MAXABS: nothing on the GPU waits for ||u_0||_inf, so its reduction runs on stream2 (ordered
    // after the caller's inputs by an event) and is enqueued AFTER the w-recurrence and the first extension:
    // those start at once and the reduction fills the SMs / thread slots they leave free
    const bool side_mx = spin_binf && c->stream2 && opt(c, PHIPM_OPT_SIDE_MAXABS);
    if (side_mx) {
        CK(cudaEventRecord(c->ev_main, c->stream));
    } else {
        int rc = enqueue_maxabs(0, 1, spin_binf);
        if (rc) return finish(rc);
        if (!spin_binf) CK(cudaEventRecord(c->ev_binf, c->stream));
    }
    // the running solution u_k lives in the padded workspace vector U (TMA-readable)
    double *ucur = c->U;
    // (H is not cleared: the exponential reads only its Hessenberg part, which every extension writes)
    // The first step reads u_0 in place when its halo copies can (n even, 16-B aligned: bulk copies
    // clamp to n); otherwise u_0 goes to the padded workspace first.  Later steps read U.
    const bool direct = (n % 2 == 0) && ((reinterpret_cast<uintptr_t>(u[0]) & 15) == 0);
    const double *x0 = direct ? u[0] : ucur;
    if (!direct) CK(cudaMemcpyAsync(ucur, u[0], n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    int enq = 0;                      // Krylov columns already enqueued for the current step
    {
        int rc = enqueue_wrec(0.0, x0, direct ? n : 0);
        if (rc) return finish(rc);
        if (m > 0) {
            rc = enqueue_krylov(c, op, bytes_op, P.symmetric, o.orth, 0, m, bthr);
            if (rc) return finish(rc);
            enq = m;
        }
    }
    if (side_mx) {
        CK(cudaStreamWaitEvent(c->stream2, c->ev_main, 0));
        int rc = enqueue_maxabs_u(c, n, u, 0, 1, true, true);
        if (rc) return finish(rc);
        c->mx_side_pending = true;
    }
    double b_inf;
    if (spin_binf) {
        // spin on the published sequence number (fallback: stream sync after 2 s, e.g. on a fault)
        const volatile int *seqp = &c->mx_h->seq;
        const auto t0 = std::chrono::steady_clock::now();
        unsigned spins = 0;
        bool synced = false;
        while (*seqp != c->mx_seq) {
            if ((++spins & 1023) == 0 && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(2)) {
                int rc = sync(c);
                if (rc) return finish(rc);
                if (side_mx && cudaStreamSynchronize(c->stream2) != cudaSuccess)
                    return finish(set_err(c, PHIPM_ECUDA, "||u_0|| reduction failed"));
                synced = true;
                if (*seqp != c->mx_seq) return finish(set_err(c, PHIPM_ECUDA, "||u_0|| result not published"));
            }
        }
        (void)synced;
        std::atomic_thread_fence(std::memory_order_acquire);
        b_inf = ((const volatile double *)c->mx_h->v)[0];
        c->mx_side_pending = false;                    // (published: the side-stream kernel has read u_0)
    } else {
        CK(cudaEventSynchronize(c->ev_binf));
        b_inf = c->raw_h[0];
    }
    c->raw_h[0] = b_inf;
    if (anorm_dev) {
        const volatile int *aseq = &c->mx_h->aseq;
        const auto t0 = std::chrono::steady_clock::now();
        unsigned spins = 0;
        while (*aseq != c->mx_aseq) {
            if ((++spins & 1023) == 0 && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(2)) {
                int rc = sync(c);
                if (rc) return finish(rc);
                if (*aseq != c->mx_aseq) return finish(set_err(c, PHIPM_ECUDA, "||A|| result not published"));
            }
        }
        std::atomic_thread_fence(std::memory_order_acquire);
        normA = ((const volatile double *)&c->mx_h->anorm)[0];
    }
    if (b_inf == 0.0) {
        {
            int rc = sync(c);
            if (rc) return finish(rc);
        }
        if (p > 0) {
            int rc = enqueue_maxabs(1, p + 1, false);
            if (rc) return finish(rc);
            rc = sync(c);
            if (rc) return finish(rc);
        }
        for (int k = 1; k <= p && b_inf == 0.0; k++) b_inf = c->raw_h[k];
        if (b_inf == 0.0) {
            CK(cudaMemsetAsync(w, 0, n * sizeof(double), c->stream));
            S.t_reached = t_end;
            return finish(sync(c));
        }
    }
    if (!std::isfinite(b_inf)) {
        sync(c);
        return finish(set_err(c, PHIPM_ENONFINITE, "non-finite input vector"));
    }
    double tau = (normA == 0.0) ? t_end : std::min(t_end, tau0(normA, b_inf, o.tol, mbar));
    if (!(tau > 0.0)) tau = t_end;

    double tk = 0.0;
    S.m_peak = m;
    bool first = true;
    bool step0 = true;                // the current step is the first (its u_k is x0)
    bool combined = false;            // the accepted attempt's guarded combine has already run
    const bool pre_ok = opt(c, PHIPM_OPT_PRECOMBINE) && !c->prof && n > SMALL_N;
    // Eq. (step): u_{k+1} = sum_{i<=mu} comb_i v~_i + sum_{j<p} tau^j/j! w_j  (w_0 = u_k in place); guard:
    // device decision words (run only if guard[0] == guard_val, nc from guard[1])
    auto enqueue_combine = [&](bool last, int nc, const int *guard, int guard_val) {
        AxpyArgs a = axpy0();
        a.out = last ? w : ucur;           // the last step writes the caller's w directly
        a.base = step0 ? x0 : ucur;
        a.a0h = (p >= 1) ? 1.0 : 0.0;
        a.a0d = (p >= 1) ? c->combd : nullptr;
        a.V = c->V;
        a.ldv = c->ldv;
        a.c0 = 0;
        a.nc = nc;
        a.g = c->comb;
        a.gsign = 1.0;
        a.ne = std::max(p - 1, 0);
        for (int j = 1; j < p; j++) {
            a.e[j - 1] = c->W + (int64_t)j * c->ldv;
            a.ec[j - 1] = 1.0;
        }
        a.ecd = c->combd + 1;
        a.guard = guard;
        a.guard_val = guard_val;
        return launch_axpy(c, n, a, PC_COMBINE);
    };
    const bool spec_ok = spec_path(c, op, P.symmetric) && !P.fixed_m;
    int spec_from = 0;                 // first column of the pending speculative extension
    bool cheb_off = false;             // the Chebyshev method was found unreliable in this solve
    while (tk < t_end) {
        if (tau > t_end - tk) tau = t_end - tk;
        if (!first) {
            join_spec();                   // the seed below rewrites the state the extension uses
            enq = 0;
            int rc = enqueue_wrec(tk, ucur, 0);
            if (rc) return finish(rc);
        }
        first = false;
        S.nspmv += p;
        int k = 0;
        bool brk = false;
        CtlMem mem;
        int attempts = 0;
        double tau_used = tau;
        int m_used = m, mu = 0;
        bool corr = false;
        for (;;) {
            attempts++;
            if (std::max(k, enq) < m && !brk) {
                join_spec();
                int rc = enqueue_krylov(c, op, bytes_op, P.symmetric, o.orth, std::max(k, enq), m, bthr);
                if (rc) return finish(rc);
                enq = m;
            } else if (c->spec_pending && m > spec_from) {
                join_spec();               // this attempt uses columns of the speculative extension
            }
            // Speculation (PHIPM_OPT_SPEC): while the exponential of this attempt runs, extend the basis
            // on stream2 to the largest m Algorithm 3 can ask for next, min((4m+2)/3, m_max) (the clamp
            // in control()).  It only adds columns beyond m: the exponential reads H, sigma and the
            // state of columns < m, and takes a breakdown position beyond m as none (expm.cuh).  An
            // accepted or tau-branch attempt leaves the columns unused (the stats count the algorithm's
            // SpMVs, not the speculative ones).
            if (spec_ok && !brk && !c->spec_pending) {
                const int ms = std::min((4 * m + 2) / 3, P.m_max);
                if (ms > std::max(k, enq)) {
                    const int k0s = std::max(k, enq);
                    CK(cudaEventRecord(c->ev_main, c->stream));
                    CK(cudaStreamWaitEvent(c->stream2, c->ev_main, 0));
                    int rc;
                    {
                        OnStream2 on2(c);
                        rc = enqueue_krylov(c, op, bytes_op, P.symmetric, o.orth, k0s, ms, bthr);
                    }
                    if (rc) return finish(rc);
                    CK(cudaEventRecord(c->ev_spec, c->stream2));
                    c->spec_pending = true;
                    spec_from = k0s;
                    enq = ms;
                }
            }
            ExpmArgs ea;
            memset(&ea, 0, sizeof(ea));
            ea.mode = 0;
            ea.method = cheb_off ? PHIPM_EXPM_TAYLOR : o.expm_method;
            ea.tridiag = P.symmetric ? 1 : 0;     // (Chebyshev method: Lanczos only)
            ea.m = m;
            ea.p = p;
            ea.tau = tau;
            ea.H = c->H;
            ea.ldh = c->m_max + 1;
            ea.sigma = c->sigma;
            ea.st = c->st;
            ea.comb = c->comb;
            ea.combd = c->combd;
            // PHIPM_OPT_PRECOMBINE: the exponential's epilogue takes the acceptance decision itself and the
            // combine of this attempt is enqueued behind it right away, guarded by that decision; an accepted
            // step then needs no host round trip between the two kernels, and after a rejection the guarded
            // kernel exits at once while the host is still deciding
            const bool precomb = pre_ok && ea.method != PHIPM_EXPM_CHEBYSHEV;
            if (precomb) {
                ea.dec = c->dec_d;
                ea.t_end = t_end;
                ea.tol = o.tol;
            }
            int rc = launch_expm(c, ea, m + p + 1);
            if (rc) return finish(rc);
            if (precomb) {
                rc = enqueue_combine(tau >= t_end - tk, 0, c->dec_d, c->seq);
                if (rc) return finish(rc);
            }
            rc = wait_attempt(c);
            if (rc) return finish(rc);
            AttemptResult R;
            memcpy(&R, (const void *)c->res_h, sizeof(R));
            if (R.seq != c->seq) return finish(set_err(c, PHIPM_ECUDA, "stale attempt result"));
            combined = false;
            // Chebyshev method: if the interval is too wide (status 7), or if the rounding-noise bound of
            // the error estimate exceeds 1e-2 max(omega, delta) (the last component is then a
            // cancellation of large Chebyshev terms, interval wider than ~mu, and an accept could rest
            // on noise), this attempt and the rest of the solve take the augmented exponential
            if (ea.method == PHIPM_EXPM_CHEBYSHEV && R.status == 0) {
                const double om = t_end * R.eps / (tau * o.tol), om_noise = t_end * R.eps_noise / (tau * o.tol);
                if (om_noise > 1e-2 * std::max(om, 1.2)) R.status = CHEB_STATUS_RANGE;
            }
            if (R.status == CHEB_STATUS_RANGE) {
                cheb_off = true;
                ea.method = PHIPM_EXPM_TAYLOR;
                rc = launch_expm(c, ea, m + p + 1);
                if (rc) return finish(rc);
                rc = wait_attempt(c);
                if (rc) return finish(rc);
                memcpy(&R, (const void *)c->res_h, sizeof(R));
                if (R.seq != c->seq) return finish(set_err(c, PHIPM_ECUDA, "stale attempt result"));
                c->ncheb_fallback++;
            }
            S.nexpm++;
            // basis actually built
            int kb;
            if (R.brk >= 0) { kb = std::max(k, R.brk); brk = true; }
            else kb = std::max(k, m);
            if (R.brk >= 0 && R.brk < k) kb = k;
            S.nspmv += kb - k;
            k = kb;
            if (R.status == 3) {
                c->coop_dirty = true;
                return finish(set_err(c, PHIPM_ECUDA, "persistent Krylov kernel: grid phase timed out"));
            }
            if (R.status == 5) return finish(set_err(c, PHIPM_ENONFINITE, "non-finite value in the Krylov step"));
            if (R.status == 6) return finish(set_err(c, PHIPM_ESINGULAR, "singular Pade denominator"));
            mu = R.mu;
            corr = R.h != 0.0 && !(R.brk >= 0 && R.brk <= mu);
            const double eps = R.eps;
            const double omega = t_end * eps / (tau * o.tol);
            if (!std::isfinite(omega)) return finish(set_err(c, PHIPM_ENONFINITE, "non-finite error estimate"));
            // (with a guarded combine in flight the device's decision is the decision: it is the same IEEE
            // expression, and the combine has acted on it)
            const bool accepted = (precomb && R.accepted >= 0) ? R.accepted != 0 : omega <= 1.2;
            combined = precomb && R.accepted >= 0 && accepted;
            Decision d = control(P, mem, tau, m, eps, omega, R.normH1, t_end - tk, accepted);
            if (c->attempts.size() < 65536)
                c->attempts.push_back({tk, tau, omega, eps, R.normH1, R.beta, m, mu, accepted ? 1 : 0, d.branch});
            c->nattempts++;
            tau_used = tau;
            m_used = m;
            S.m_peak = std::max(S.m_peak, m);
            tau = d.tau_next;
            m = d.m_next;
            if (accepted) break;
            S.nreject++;
            if (attempts >= 100 || tau < 1e-15 * t_end) {
                S.t_reached = tk;
                cudaMemcpyAsync(w, step0 ? x0 : ucur, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream);
                cudaStreamSynchronize(c->stream);
                return finish(set_err(c, PHIPM_ESTEP, "step size control failed at t = %g", tk));
            }
        }
        // Eq. (step): u_{k+1} = sum_{i<=mu} comb_i v~_i + sum_{j<p} tau^j/j! w_j  (w_0 = u_k in place)
        const bool last = tau_used >= t_end - tk;
        if (!combined) {
            int rc = enqueue_combine(last, mu + (corr ? 1 : 0), nullptr, 0);
            if (rc) return finish(rc);
        }
        if (last) tk = t_end;
        else tk += tau_used;
        S.nsteps++;
        step0 = false;
        S.m_last = m_used;
        S.t_reached = tk;
    }
    join_spec();
    int rc = sync(c);
    return finish(rc);
}

// ---------------------------------------------------------------------------------------------
// operator construction / validation

int make_stencil(phipm_ctx *c, const phipm_stencil *S, StencilOp &op)
{
    if (!S) return set_err(c, PHIPM_EINVAL, "null stencil");
    if (S->dim < 1 || S->dim > 3 || S->nx < 1 || S->ny < 1 || S->nz < 1)
        return set_err(c, PHIPM_EINVAL, "bad stencil dims");
    if ((S->dim < 2 && S->ny != 1) || (S->dim < 3 && S->nz != 1))
        return set_err(c, PHIPM_EINVAL, "stencil: unused dimensions must be 1");
    op.dim = S->dim;
    op.nx = S->nx;
    op.ny = S->ny;
    op.nz = S->nz;
    op.n = (int64_t)S->nx * S->ny * S->nz;
    if (op.n >= ((int64_t)1 << 31)) return set_err(c, PHIPM_EINVAL, "stencil too large");
    const double cc[11] = {S->c_center, S->c_xm, S->c_xp, S->c_ym, S->c_yp, S->c_zm, S->c_zp,
                           S->c_xmym, S->c_xpym, S->c_xmyp, S->c_xpyp};
    for (int i = 0; i < 11; i++) op.c[i] = cc[i];
    if (S->dim < 3) op.c[5] = op.c[6] = 0.0;
    if (S->dim < 2) op.c[3] = op.c[4] = 0.0;
    if (S->points == 9 && S->dim != 2) return set_err(c, PHIPM_EINVAL, "stencil: points = 9 needs dim = 2");
    op.diag = S->points == 9 ? 1 : 0;
    op.sdj = S->dim >= 2 ? (2 * SNT) / S->nx : 0;          // 2 SNT rows = sdj lines + sdi points
    op.sdi = S->dim >= 2 ? 2 * SNT - op.sdj * S->nx : 2 * SNT;
    if (!op.diag) op.c[7] = op.c[8] = op.c[9] = op.c[10] = 0.0;
    return PHIPM_OK;
}

int64_t stencil_nnz(const StencilOp &s)
{
    const int64_t nx = s.nx, ny = s.ny, nz = s.nz, n = s.n;
    if (s.diag) return (3 * nx - 2) * (3 * ny - 2);             // 9-point: (3nx-2)(3ny-2)
    int64_t nnz = n + 2 * (n - ny * nz);                       // x neighbours: 2(nx-1) per line
    if (s.dim >= 2) nnz += 2 * (n - nx * nz);
    if (s.dim >= 3) nnz += 2 * (n - nx * ny);
    return nnz;
}

// ||A||_inf of the stencil: max over the boundary classes present, each row summed in ascending
// column order (z-, y-, x-, centre, x+, y+, z+) like a sequential CSR row sum.
double stencil_infnorm(const StencilOp &s)
{
    double best = 0.0;
    auto classes = [](int N, int *lo, int *hi, int &cnt) {
        // positions: first, interior, last (those that exist)
        cnt = 0;
        if (N == 1) { lo[cnt] = 0; hi[cnt] = 0; cnt++; return; }
        lo[cnt] = 0; hi[cnt] = 1; cnt++;
        if (N > 2) { lo[cnt] = 1; hi[cnt] = 1; cnt++; }
        lo[cnt] = 1; hi[cnt] = 0; cnt++;
    };
    int xl[3], xh[3], yl[3], yh[3], zl[3], zh[3], cx, cy, cz;
    classes(s.nx, xl, xh, cx);
    classes(s.dim >= 2 ? s.ny : 1, yl, yh, cy);
    classes(s.dim >= 3 ? s.nz : 1, zl, zh, cz);
    for (int a = 0; a < cz; a++)
        for (int b = 0; b < cy; b++)
            for (int d = 0; d < cx; d++) {
                // ascending column order of the CSR row (9-point corners around the y-neighbours)
                const bool dg = s.diag != 0;
                double t = 0.0;
                if (s.dim >= 3 && zl[a]) t = t + std::fabs(s.c[5]);
                if (dg && yl[b] && xl[d]) t = t + std::fabs(s.c[7]);
                if (s.dim >= 2 && yl[b]) t = t + std::fabs(s.c[3]);
                if (dg && yl[b] && xh[d]) t = t + std::fabs(s.c[8]);
                if (xl[d]) t = t + std::fabs(s.c[1]);
                t = t + std::fabs(s.c[0]);
                if (xh[d]) t = t + std::fabs(s.c[2]);
                if (dg && yh[b] && xl[d]) t = t + std::fabs(s.c[9]);
                if (s.dim >= 2 && yh[b]) t = t + std::fabs(s.c[4]);
                if (dg && yh[b] && xh[d]) t = t + std::fabs(s.c[10]);
                if (s.dim >= 3 && zh[a]) t = t + std::fabs(s.c[6]);
                best = std::max(best, t);
            }
    return best;
}

int make_csr(phipm_ctx *c, const phipm_csr *A, CsrOp &op)
{
    if (!A || !A->row_ptr || A->n <= 0 || A->nnz < 0 || (A->nnz > 0 && (!A->col || !A->val)))
        return set_err(c, PHIPM_EINVAL, "bad csr descriptor");
    if (A->nnz >= ((int64_t)1 << 31) || A->n >= ((int64_t)1 << 31)) return set_err(c, PHIPM_EINVAL, "csr too large");
    op.n = A->n;
    op.rp = A->row_ptr;
    op.col = A->col;
    op.val = A->val;
    const double mean = A->n > 0 ? (double)A->nnz / (double)A->n : 1.0;
    int glog = 0;
    while (glog < 5 && (double)(1 << (glog + 1)) <= mean) glog++;
    op.glog = glog;
    op.tlo = op.thi = nullptr;
    op.wtile = op.wcap = 0;
    op.ell = 0;
    op.ring = op.blo = op.bhi = 0;
    op.pf = 0;
    op.pf_end = op.n;
    op.off16 = nullptr;
    return PHIPM_OK;
}

// CSR x-window mode: per-tile column ranges for 2048-row tiles (one pass over col); tiles whose
// range fits CSR_WCAP doubles gather x from shared memory (stream.cuh)
constexpr int CSR_WCAP = 10496;                             // 82 KB: band +-4096 around 2048 rows

// One analysis pass over a CSR matrix (csr_analyze_kernel): ||A||_inf (a1 setup, bit-exact), and
// whether rows have a uniform length L (vectorised ELL path, PHIPM_OPT_CSR_ELL = 0 disables) within a
// band that fits the shared x ring (PHIPM_OPT_CSR_RING = 0 disables).
int analyze_csr(phipm_ctx *c, CsrOp &op, int64_t nnz, double *normA, int mode = 3, int16_t *off16 = nullptr)
{
    op.ell = 0;
    op.ring = op.blo = op.bhi = 0;
    const int env_ell = opt(c, PHIPM_OPT_CSR_ELL), env_ring = opt(c, PHIPM_OPT_CSR_RING);
    if (op.n == 0) {
        *normA = 0.0;
        return PHIPM_OK;
    }
    const int64_t L = (nnz % op.n == 0 && nnz / op.n <= 128) ? nnz / op.n : -1;
    CsrAnalysis *d = reinterpret_cast<CsrAnalysis *>(c->raw);
    CK(cudaMemsetAsync(d, 0, sizeof(CsrAnalysis), c->stream));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((op.n + CSRA_NT - 1) / CSRA_NT, (int64_t)c->sm_count * 16));
    ProfRec r;
    prof_begin(c, r, PC_OTHER, ((mode & 1) ? 8.0 : 0.0) * (double)nnz + ((mode & 2) ? 4.0 : 0.0) * (double)nnz +
                                   ((mode & 4) && off16 && L > 0 ? 2.0 : 0.0) * (double)nnz + 4.0 * (double)(op.n + 1));
    // band and uniformity only, rows of a power-of-two length >= 4, 16-B aligned columns: the streaming
    // kernel (csr_analyze_ell_kernel); if the rows turn out not to be uniform, the general pass follows
    int lgL = -1;
    if (mode == 2 && L >= 4 && (L & (L - 1)) == 0 && ((uintptr_t)op.col & 15) == 0)
        for (lgL = 0; ((int64_t)1 << lgL) < L; lgL++) {
        }
    if (lgL >= 2) {
        const int g2 = (int)std::max<int64_t>(1, std::min<int64_t>(((int64_t)nnz / 4 + 255) / 256, (int64_t)c->sm_count * 8));
        csr_analyze_ell_kernel<<<g2, 256, 0, c->stream>>>(op.n, op.rp, op.col, lgL, d);
    } else {
        csr_analyze_kernel<<<grid, CSRA_NT, 0, c->stream>>>(op, (int)L, d, mode, off16);
    }
    prof_end(c, r);
    c->acc.launches++;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(c->raw_h, d, sizeof(CsrAnalysis), cudaMemcpyDeviceToHost, c->stream));
    int rc = sync(c);
    if (rc) return rc;
    CsrAnalysis h;
    memcpy(&h, c->raw_h, sizeof(h));
    if (lgL >= 2 && h.nonuniform) {
        CK(cudaMemsetAsync(d, 0, sizeof(CsrAnalysis), c->stream));
        csr_analyze_kernel<<<grid, CSRA_NT, 0, c->stream>>>(op, (int)L, d, mode, off16);
        c->acc.launches++;
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(c->raw_h, d, sizeof(CsrAnalysis), cudaMemcpyDeviceToHost, c->stream));
        rc = sync(c);
        if (rc) return rc;
        memcpy(&h, c->raw_h, sizeof(h));
    }
    if (mode & 1) memcpy(normA, &h.norm_bits, sizeof(double));
    if (!(mode & 2)) return PHIPM_OK;
    if (!env_ell || L < 4 || (L % 4) || ((L / 4) & (L / 4 - 1)) || h.nonuniform) return PHIPM_OK;
    if (((uintptr_t)op.val & 15) || ((uintptr_t)op.col & 15)) return PHIPM_OK;
    op.ell = (int)L;
    op.pf = opt(c, PHIPM_OPT_CSR_PREFETCH);
    op.pf_end = op.n;
    op.blo = (h.blo + 1) & ~1;
    op.bhi = (h.bhi + 1) & ~1;
    op.ring = (env_ring && 2 * SNT * 2 + op.blo + op.bhi <= XRING) ? 1 : 0;
    // int16 column offsets (written by this pass when asked): usable when the band fits int16
    if ((mode & 4) && off16 && op.ring && h.blo <= 32767 && h.bhi <= 32767) op.off16 = off16;
    return PHIPM_OK;
}

int enable_csr_window(phipm_ctx *c, CsrOp &op)
{
    if (opt(c, PHIPM_OPT_CSR_WINDOW) != 1 || op.ring) return PHIPM_OK;                  // default off (measured slower, round 1)
    const int tile = SNT * 8;
    const int64_t ntiles = (op.n + tile - 1) / tile;
    if (ntiles > c->ntile_cap || op.n < (int64_t)tile) return PHIPM_OK;   // small problems: global gathers
    const int grid = (int)std::min<int64_t>((ntiles + 7) / 8, (int64_t)c->sm_count * 8);
    csr_tile_range_kernel<<<grid, 256, 0, c->stream>>>(op.n, op.rp, op.col, tile, c->tlo, c->thi);
    c->acc.launches++;
    CK(cudaGetLastError());
    op.tlo = c->tlo;
    op.thi = c->thi;
    op.wtile = tile;
    op.wcap = CSR_WCAP;
    return PHIPM_OK;
}

// algorithmic bytes of one SpMV: val + column indices (4 B, or 2 B as int16 offsets) + row_ptr + x + y
double csr_bytes(const CsrOp &op, int64_t nnz)
{
    return (op.off16 ? 10.0 : 12.0) * (double)nnz + 4.0 * (double)(op.n + 1) + 16.0 * (double)op.n;
}

int check_common(phipm_ctx *c, double t, int64_t n, int p, const double *const *u, const double *w,
                 phipm_opts &o)
{
    if (!c) return PHIPM_EINVAL;
    if (!(t >= 0.0) || !std::isfinite(t)) return set_err(c, PHIPM_EINVAL, "t must be finite and >= 0");
    if (n <= 0 || n > c->n_max) return set_err(c, PHIPM_EINVAL, "n=%lld out of range (n_max %lld)", (long long)n, (long long)c->n_max);
    if (p < 0 || p > c->p_max) return set_err(c, PHIPM_EINVAL, "p=%d out of range (p_max %d)", p, c->p_max);
    if (!u || !w) return set_err(c, PHIPM_EINVAL, "null u or w");
    for (int k = 0; k <= p; k++)
        if (!u[k]) return set_err(c, PHIPM_EINVAL, "null u[%d]", k);
    for (int k = 1; k <= p; k++)
        if (u[k] == w) return set_err(c, PHIPM_EINVAL, "w may alias u[0] only");
    if (!(o.tol > 0.0)) return set_err(c, PHIPM_EINVAL, "tol must be > 0");
    if (o.m_max > c->m_max) return set_err(c, PHIPM_EINVAL, "opts.m_max %d > context m_max %d", o.m_max, c->m_max);
    if (o.m_init < 1 || o.m_init > o.m_max) return set_err(c, PHIPM_EINVAL, "m_init must be in [1, m_max]");
    if (o.expm_method != PHIPM_EXPM_TAYLOR && o.expm_method != PHIPM_EXPM_PADE13 &&
        o.expm_method != PHIPM_EXPM_CHEBYSHEV)
        return set_err(c, PHIPM_EINVAL, "unknown expm_method %d", o.expm_method);
    if (o.orth != PHIPM_ORTH_CGS && o.orth != PHIPM_ORTH_CGS2) return set_err(c, PHIPM_EINVAL, "bad orth");
    return PHIPM_OK;
}

phipm_opts resolve_opts(const phipm_opts *o)
{
    phipm_opts r;
    phipm_default_opts(&r);
    if (o) r = *o;
    return r;
}

// ---------------------------------------------------------------------------------------------
// Block solve: nb problems sharing the CSR operator A, t, p, tol.  One controller
// drives all of them in lockstep (Alg. 3/4 on the block's largest error estimate: omega = max_b
// omega_b, so every problem meets its tolerance when the block step is accepted); each Krylov step
// multiplies all nb basis vectors by A in one SpMM pass over val/col (spmm.cuh), then every problem
// runs its own fused dot / update kernels (identity operator) on its own basis.  Workspaces are the
// nb contexts'; every launch goes to ctx[0]'s stream.

int launch_spmm_one(phipm_ctx *c0, const CsrOp &op, SpmmArgs &sa, double bytes, int64_t ldx, int T)
{
    if (T > 0) {
        SpmmRing g;
        g.T = T;
        g.R = (2 * T + op.blo + op.bhi + 31) & ~31;
        g.ldx = ldx;
        const size_t smem = (size_t)sa.nb * g.R * sizeof(double);
        int grid;
        balance(c0, op.n, c0->sm_count, grid, sa.rpc);
        ProfRec r;
        prof_begin(c0, r, PC_SPMV, bytes, sa.nb);
        if (sa.nb <= 2) launch_k(c0, spmm_csr_ring_kernel<2>, grid, SNT, smem, op, sa, g);
        else if (sa.nb <= 4) launch_k(c0, spmm_csr_ring_kernel<4>, grid, SNT, smem, op, sa, g);
        else launch_k(c0, spmm_csr_ring_kernel<SPMM_MAXB>, grid, SNT, smem, op, sa, g);
        prof_end(c0, r);
    } else {
        int occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, spmm_csr_kernel, SPMM_NT, 0);
        int grid;
        balance(c0, op.n, std::max(occ, 1) * c0->sm_count, grid, sa.rpc);
        ProfRec r;
        prof_begin(c0, r, PC_SPMV, bytes, sa.nb);
        launch_k(c0, spmm_csr_kernel, grid, SPMM_NT, 0, op, sa);
        prof_end(c0, r);
    }
    c0->acc.launches++;
    CK0(c0, cudaGetLastError());
    return PHIPM_OK;
}

// Y_b = A X_b for the block.  Banded uniform-row CSR: x rings in shared memory, in chunks of as many
// vectors as fit with T = 1024 (else 512) rows per tile, one pass over val/col per chunk; other
// matrices: one pass with L1 gathers.  bytes_op: the operator's algorithmic bytes of one SpMV.
int launch_spmm(phipm_ctx *c0, const CsrOp &op, const SpmmArgs &sa, double bytes_op, int64_t ldx)
{
    const double n = (double)op.n;
    if (op.ell > 0 && opt(c0, PHIPM_OPT_CSR_RING)) {
        for (int T = 1024; T >= 512; T >>= 1) {
            const size_t ring = (size_t)((2 * T + op.blo + op.bhi + 31) & ~31) * sizeof(double);
            const int fit = (int)std::min<size_t>(c0->smem_optin / ring, SPMM_MAXB);
            if (fit < 1) continue;
            const int per = std::min(fit, (sa.nb + ((sa.nb + fit - 1) / fit) - 1) / ((sa.nb + fit - 1) / fit));
            for (int b0 = 0; b0 < sa.nb; b0 += per) {
                SpmmArgs s = sa;
                s.nb = std::min(per, sa.nb - b0);
                for (int b = 0; b < s.nb; b++) {
                    s.x[b] = sa.x[b0 + b];
                    s.y[b] = sa.y[b0 + b];
                    s.brk[b] = sa.brk[b0 + b];
                }
                int rc = launch_spmm_one(c0, op, s, bytes_op - 16.0 * n + 16.0 * n * s.nb, ldx, T);
                if (rc) return rc;
            }
            return PHIPM_OK;
        }
    }
    SpmmArgs s = sa;
    return launch_spmm_one(c0, op, s, bytes_op - 16.0 * n + 16.0 * n * sa.nb, ldx, 0);
}

// Krylov steps j = k0 .. k1-1 of every problem (lockstep)
int enqueue_krylov_block(phipm_ctx *const *cs, int nb, const CsrOp &op, double bytes_op, bool symmetric, int k0,
                         int k1, double bthr)
{
    phipm_ctx *c0 = cs[0];
    const int64_t n = op.n;
    for (int j = k0; j < k1; j++) {
        SpmmArgs sa;
        memset(&sa, 0, sizeof(sa));
        sa.nb = nb;
        for (int b = 0; b < nb; b++) {
            sa.x[b] = cs[b]->V + (int64_t)j * cs[b]->ldv;
            sa.y[b] = cs[b]->W + (int64_t)cs[b]->p_max * cs[b]->ldv;    // free slot of W
            sa.brk[b] = &cs[b]->st->brk;
        }
        // operator bytes once, plus nb x (gathered x once, y written)
        int64_t ldx = cs[0]->ldv;                          // readable length of every x_b (V columns)
        for (int b = 1; b < nb; b++) ldx = std::min(ldx, cs[b]->ldv);
        int rc = launch_spmm(c0, op, sa, bytes_op, ldx);
        if (rc) return rc;
        for (int b = 0; b < nb; b++) {
            phipm_ctx *c = cs[b];
            double *vn = c->V + (int64_t)(j + 1) * c->ldv;
            SpmvArgs s = spmv0();
            s.x = sa.y[b];                   // raw A v~_j
            s.xscale = c->sigma + j;
            s.y = c->Y;
            s.V = c->V;
            s.ldv = c->ldv;
            s.ynorm = 1;
            s.j = j;
            s.check_brk = 1;
            AxpyArgs u = axpy0();
            u.out = vn;
            u.base = c->Y;
            u.a0h = 1.0;
            u.V = c->V;
            u.ldv = c->ldv;
            u.g = c->g;
            u.gsign = -1.0;
            u.onorm = 1;
            u.fin = FIN_NORM;
            u.j = j;
            u.check_brk = 1;
            u.bthr = bthr;
            u.rev = 1;
            if (symmetric) {
                if (j > 0) {
                    s.nz = 1;
                    s.z[0] = c->V + (int64_t)(j - 1) * c->ldv;
                    s.zc[0] = -1.0;
                    s.zcd[0] = &c->st->lz;
                }
                s.d0 = j;
                s.nd = 1;
                s.fin = FIN_LANCZOS;
                u.c0 = j;
                u.nc = 1;
                u.lanczos = 1;
            } else {
                s.d0 = 0;
                s.nd = j + 1;
                s.fin = FIN_ARNOLDI;
                u.c0 = 0;
                u.nc = j + 1;
            }
            rc = launch_spmv(c, IdentOp{n}, s, 16.0 * (double)n);
            if (!rc) rc = launch_axpy(c, n, u, PC_ORTH);
            if (rc) return rc;
        }
    }
    return PHIPM_OK;
}

// Eq. (wrecurrence) for the block: w_{j,b} = A w_{j-1,b} + sum_l t_k^l/l! u_{j+l,b}, the products by
// SpMM (raw A w_{j-1,b} into a scratch column), the u-terms (and w_p's norm, FIN_SEED) by each
// problem's identity-operator pass; w_0 = U_b (the running solution)
int enqueue_wrec_block(phipm_ctx *const *cs, int nb, const CsrOp &op, double bytes_op, int p,
                       const double *const *const *u, double tk)
{
    if (p == 0) {
        for (int b = 0; b < nb; b++) {
            int rc = enqueue_wrec_op(cs[b], op, bytes_op, 0, u[b], tk, cs[b]->U, 0);
            if (rc) return rc;
        }
        return PHIPM_OK;
    }
    const int64_t n = op.n;
    int64_t ldx = cs[0]->ldv;
    for (int b = 1; b < nb; b++) ldx = std::min(ldx, cs[b]->ldv);
    for (int j = 1; j <= p; j++) {
        SpmmArgs sa;
        memset(&sa, 0, sizeof(sa));
        sa.nb = nb;
        for (int b = 0; b < nb; b++) {
            phipm_ctx *c = cs[b];
            sa.x[b] = (j == 1) ? c->U : c->W + (int64_t)(j - 1) * c->ldv;
            sa.y[b] = c->W + (int64_t)c->p_max * c->ldv;
        }
        int rc = launch_spmm(cs[0], op, sa, bytes_op, ldx);
        if (rc) return rc;
        for (int b = 0; b < nb; b++) {
            phipm_ctx *c = cs[b];
            SpmvArgs s = spmv0();
            s.x = sa.y[b];
            s.y = (j == p) ? c->V : c->W + (int64_t)j * c->ldv;
            double coef = 1.0;
            s.nz = 0;
            for (int l = 0; l <= p - j; l++) {
                if (l > 0) coef = coef * tk / (double)l;
                if (l > 0 && coef == 0.0) continue;
                s.z[s.nz] = u[b][j + l];
                s.zc[s.nz] = coef;
                s.nz++;
            }
            s.ynorm = (j == p);
            s.fin = (j == p) ? FIN_SEED : FIN_NONE;
            rc = launch_spmv(c, IdentOp{n}, s, 16.0 * (double)n);
            if (rc) return rc;
        }
    }
    return PHIPM_OK;
}

int solve_block_impl(phipm_ctx *const *cs, int nb, double t_end, const CsrOp &op, double bytes_op, int64_t NA,
                     double normA, int p, const double *const *const *u, const phipm_opts &o, double *const *w,
                     phipm_stats *stats)
{
    phipm_ctx *c0 = cs[0];
    const int64_t n = op.n;
    std::vector<phipm_stats> S((size_t)nb);
    for (auto &s : S) s = phipm_stats{};
    auto finish = [&](int rc) {
        if (stats)
            for (int b = 0; b < nb; b++) stats[b] = S[b];
        return rc;
    };
    for (int b = 0; b < nb; b++) {
        cs[b]->attempts.clear();
        cs[b]->nattempts = 0;
        cs[b]->ss_att_pending = 0;
    }
    if (t_end == 0.0) {
        for (int b = 0; b < nb; b++)
            if (w[b] != u[b][0]) CK0(c0, cudaMemcpyAsync(w[b], u[b][0], n * sizeof(double), cudaMemcpyDeviceToDevice, c0->stream));
        return finish(sync(c0));
    }
    Problem P;
    P.p = p;
    P.n = n;
    P.NA = NA;
    P.symmetric = o.symmetric != 0;
    P.m_max = (int)std::min<int64_t>(o.m_max, n);
    P.fixed_m = o.fixed_m != 0;
    P.eq6_variant = o.eq6_variant != 0;
    int m = std::min(o.m_init, P.m_max);
    const double mbar = 0.5 * ((double)o.m_init + (double)P.m_max);
    const double bthr = (double)n * EPS_MACH * normA;
    // b_inf of Eq. (tau_0) per problem (R7); the block starts with the smallest tau_0 (largest b_inf)
    double binf_max = 0.0;
    std::vector<char> zero((size_t)nb, 0);
    for (int b = 0; b < nb; b++) {
        phipm_ctx *c = cs[b];
        int rc = enqueue_maxabs_u(c, n, u[b], 0, p + 1, false);
        if (rc) return finish(rc);
    }
    {
        int rc = sync(c0);
        if (rc) return finish(rc);
    }
    for (int b = 0; b < nb; b++) {
        double bi = 0.0;
        for (int k = 0; k <= p && bi == 0.0; k++) bi = cs[b]->raw_h[k];
        if (!std::isfinite(bi)) return finish(set_err(c0, PHIPM_ENONFINITE, "non-finite input vector (problem %d)", b));
        zero[b] = bi == 0.0;
        binf_max = std::max(binf_max, bi);
    }
    if (binf_max == 0.0) {
        for (int b = 0; b < nb; b++) CK0(c0, cudaMemsetAsync(w[b], 0, n * sizeof(double), c0->stream));
        for (auto &s : S) s.t_reached = t_end;
        return finish(sync(c0));
    }
    double tau = (normA == 0.0) ? t_end : std::min(t_end, tau0(normA, binf_max, o.tol, mbar));
    if (!(tau > 0.0)) tau = t_end;
    for (int b = 0; b < nb; b++) {
        CK0(c0, cudaMemcpyAsync(cs[b]->U, u[b][0], n * sizeof(double), cudaMemcpyDeviceToDevice, c0->stream));
        S[b].m_peak = m;
    }
    double tk = 0.0;
    std::vector<int> kb((size_t)nb), mub((size_t)nb);
    std::vector<char> brk((size_t)nb), corr((size_t)nb);
    while (tk < t_end) {
        if (tau > t_end - tk) tau = t_end - tk;
        {
            int rc = enqueue_wrec_block(cs, nb, op, bytes_op, p, u, tk);
            if (rc) return finish(rc);
        }
        for (int b = 0; b < nb; b++) {
            S[b].nspmv += p;
            kb[b] = 0;
            brk[b] = 0;
        }
        int enq = 0;
        CtlMem mem;
        int attempts = 0;
        double tau_used = tau;
        int m_used = m;
        for (;;) {
            attempts++;
            if (enq < m) {
                int rc = enqueue_krylov_block(cs, nb, op, bytes_op, P.symmetric, enq, m, bthr);
                if (rc) return finish(rc);
                enq = m;
            }
            for (int b = 0; b < nb; b++) {
                phipm_ctx *c = cs[b];
                ExpmArgs ea;
                memset(&ea, 0, sizeof(ea));
                ea.mode = 0;
                ea.method = o.expm_method == PHIPM_EXPM_PADE13 ? PHIPM_EXPM_PADE13 : PHIPM_EXPM_TAYLOR;
                ea.tridiag = P.symmetric ? 1 : 0;
                ea.m = m;
                ea.p = p;
                ea.tau = tau;
                ea.H = c->H;
                ea.ldh = c->m_max + 1;
                ea.sigma = c->sigma;
                ea.st = c->st;
                ea.comb = c->comb;
                ea.combd = c->combd;
                int rc = launch_expm(c, ea, m + p + 1);
                if (rc) return finish(rc);
            }
            double eps_max = 0.0, nh_max = 0.0;
            for (int b = 0; b < nb; b++) {
                phipm_ctx *c = cs[b];
                int rc = wait_attempt(c);
                if (rc) return finish(rc);
                AttemptResult R;
                memcpy(&R, (const void *)c->res_h, sizeof(R));
                if (R.seq != c->seq) return finish(set_err(c0, PHIPM_ECUDA, "stale attempt result (problem %d)", b));
                S[b].nexpm++;
                int k2;
                if (R.brk >= 0) { k2 = std::max(kb[b], R.brk); brk[b] = 1; }
                else k2 = std::max(kb[b], m);
                if (R.brk >= 0 && R.brk < kb[b]) k2 = kb[b];
                S[b].nspmv += k2 - kb[b];
                kb[b] = k2;
                if (R.status == 5) return finish(set_err(c0, PHIPM_ENONFINITE, "non-finite value (problem %d)", b));
                if (R.status == 6) return finish(set_err(c0, PHIPM_ESINGULAR, "singular Pade denominator"));
                if (R.status == 3) return finish(set_err(c0, PHIPM_ECUDA, "grid phase timed out"));
                mub[b] = R.mu;
                corr[b] = R.h != 0.0 && !(R.brk >= 0 && R.brk <= R.mu);
                eps_max = std::max(eps_max, R.eps);
                nh_max = std::max(nh_max, R.normH1);
            }
            const double omega = t_end * eps_max / (tau * o.tol);
            if (!std::isfinite(omega)) return finish(set_err(c0, PHIPM_ENONFINITE, "non-finite error estimate"));
            const bool accepted = omega <= 1.2;
            Decision d = control(P, mem, tau, m, eps_max, omega, nh_max, t_end - tk, accepted);
            for (int b = 0; b < nb; b++) {
                if (cs[b]->attempts.size() < 65536)
                    cs[b]->attempts.push_back({tk, tau, omega, eps_max, nh_max, 0.0, m, mub[b], accepted ? 1 : 0, d.branch});
                cs[b]->nattempts++;
                S[b].m_peak = std::max(S[b].m_peak, m);
            }
            tau_used = tau;
            m_used = m;
            tau = d.tau_next;
            m = d.m_next;
            if (accepted) break;
            for (auto &s : S) s.nreject++;
            if (attempts >= 100 || tau < 1e-15 * t_end) {
                for (int b = 0; b < nb; b++) {
                    S[b].t_reached = tk;
                    cudaMemcpyAsync(w[b], cs[b]->U, n * sizeof(double), cudaMemcpyDeviceToDevice, c0->stream);
                }
                cudaStreamSynchronize(c0->stream);
                return finish(set_err(c0, PHIPM_ESTEP, "step size control failed at t = %g", tk));
            }
        }
        const bool last = tau_used >= t_end - tk;
        for (int b = 0; b < nb; b++) {
            phipm_ctx *c = cs[b];
            AxpyArgs a = axpy0();
            a.out = last ? w[b] : c->U;
            a.base = c->U;
            a.a0h = (p >= 1) ? 1.0 : 0.0;
            a.a0d = (p >= 1) ? c->combd : nullptr;
            a.V = c->V;
            a.ldv = c->ldv;
            a.c0 = 0;
            a.nc = mub[b] + (corr[b] ? 1 : 0);
            a.g = c->comb;
            a.gsign = 1.0;
            a.ne = std::max(p - 1, 0);
            for (int j = 1; j < p; j++) {
                a.e[j - 1] = c->W + (int64_t)j * c->ldv;
                a.ec[j - 1] = 1.0;
            }
            a.ecd = c->combd + 1;
            int rc = launch_axpy(c, n, a, PC_COMBINE);
            if (rc) return finish(rc);
        }
        if (last) tk = t_end;
        else tk += tau_used;
        for (auto &s : S) {
            s.nsteps++;
            s.m_last = m_used;
            s.t_reached = tk;
        }
    }
    return finish(sync(c0));
}

} // namespace

// Persistent worker pool of the batch API (phipm_solve_*_batch): threads are created once and grow
// to the largest batch seen, so a batch call costs a queue push per problem, not a thread start.
// The pool is never destroyed (its idle threads wait on a condition variable until process exit).
class WorkerPool {
public:
    static WorkerPool &get()
    {
        static WorkerPool *p = new WorkerPool();
        return *p;
    }
    // run fn(0..nb-1) on pool threads and wait for all of them
    template <class F>
    void run(int nb, F &fn)
    {
        std::mutex dmu;
        std::condition_variable dcv;
        int left = nb;
        {
            std::lock_guard<std::mutex> lk(mu_);
            while ((int)th_.size() < nb) th_.emplace_back([this] { loop(); });
            for (int b = 0; b < nb; b++)
                q_.push_back([&, b] {
                    fn(b);
                    std::lock_guard<std::mutex> l2(dmu);
                    if (--left == 0) dcv.notify_one();
                });
        }
        cv_.notify_all();
        std::unique_lock<std::mutex> lk(dmu);
        dcv.wait(lk, [&] { return left == 0; });
    }

private:
    void loop()
    {
        for (;;) {
            std::function<void()> job;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [this] { return !q_.empty(); });
                job = std::move(q_.front());
                q_.pop_front();
            }
            job();
        }
    }
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> q_;
    std::vector<std::thread> th_;
};

// Run nb solves concurrently on the worker pool (phipm_solve_*_batch).  Each worker first makes the
// context's device current: pool threads start on device 0, and a context may live on another GPU.
template <class F>
static int run_batch(phipm_ctx *const *ctx, int nb, int *status, F solve_one)
{
    if (nb == 0) return PHIPM_OK;
    if (!ctx || nb < 0) return PHIPM_EINVAL;
    for (int b = 0; b < nb; b++)
        for (int b2 = 0; b2 < b; b2++)
            if (!ctx[b] || ctx[b] == ctx[b2]) return PHIPM_EINVAL;   // one context per problem
    if (!ctx[0]) return PHIPM_EINVAL;
    std::vector<int> st((size_t)nb, PHIPM_OK);
    auto job = [&](int b) {
        const cudaError_t e = cudaSetDevice(ctx[b]->dev);
        st[b] = (e == cudaSuccess) ? solve_one(b)
                                   : set_err(ctx[b], PHIPM_ECUDA, "cudaSetDevice(%d): %s", ctx[b]->dev,
                                             cudaGetErrorString(e));
    };
    WorkerPool::get().run(nb, job);
    int rc = PHIPM_OK;
    for (int b = 0; b < nb; b++) {
        if (status) status[b] = st[b];
        if (rc == PHIPM_OK && st[b] != PHIPM_OK) rc = st[b];
    }
    return rc;
}

// =============================================================================================
// C ABI

extern "C" {

int phipm_set_option(phipm_ctx *c, int option, int value)
{
    if (!c || option < 0 || option >= PHIPM_OPT_COUNT) return PHIPM_EINVAL;
    bool ok;
    switch (option) {
    case PHIPM_OPT_PERSIST: ok = value >= 0 && value <= 2; break;
    case PHIPM_OPT_BRICK: ok = value >= 0 && value <= 2; break;
    case PHIPM_OPT_RPT: ok = value == 0 || value == 2 || value == 4 || value == 8; break;
    case PHIPM_OPT_PERSIST_MINROWS: ok = value >= 0; break;
    case PHIPM_OPT_CSR_PREFETCH: ok = value >= 0 && value <= (1 << 20); break;
    case PHIPM_OPT_COL_PREFETCH: ok = value == 0 || value == 1; break;
    case PHIPM_OPT_FUSE_ANORM: ok = value == 0 || value == 1; break;
    case PHIPM_OPT_CSR_OFF16: ok = value == 0 || value == 1; break;
    case PHIPM_OPT_DEVSOLVE: ok = value == 0 || value == 1; break;
    case PHIPM_OPT_GRAPH: ok = value == 0 || value == 1; break;
    case PHIPM_OPT_CLUSTER_LZ: ok = value >= -1 && value <= 16 && (value <= 1 || (value & (value - 1)) == 0); break;
    default: ok = value == 0 || value == 1; break;
    }
    if (!ok) return set_err(c, PHIPM_EINVAL, "option %d: value %d out of range", option, value);
    c->opt[option] = value;
    if (option == PHIPM_OPT_PDL) c->pdl = value != 0;
    return PHIPM_OK;
}

int phipm_get_option(const phipm_ctx *c, int option, int *value)
{
    if (!c || !value || option < 0 || option >= PHIPM_OPT_COUNT) return PHIPM_EINVAL;
    *value = c->opt[option];
    return PHIPM_OK;
}

int phipm_set_expm_method(phipm_ctx *c, int method)
{
    if (!c || (method != PHIPM_EXPM_TAYLOR && method != PHIPM_EXPM_PADE13 && method != PHIPM_EXPM_CHEBYSHEV))
        return PHIPM_EINVAL;
    c->expm_method = method;
    return PHIPM_OK;
}

void phipm_default_opts(phipm_opts *o)
{
    if (!o) return;
    o->tol = 1e-7;
    o->m_init = 10;
    o->m_max = 100;
    o->symmetric = 0;
    o->fixed_m = 0;
    o->eq6_variant = 0;
    o->orth = PHIPM_ORTH_CGS;
    o->profile = 0;
    o->expm_method = PHIPM_EXPM_TAYLOR;
}

const char *phipm_strerror(int s)
{
    switch (s) {
    case PHIPM_OK: return "ok";
    case PHIPM_EINVAL: return "invalid argument";
    case PHIPM_ENOMEM: return "out of memory";
    case PHIPM_ECUDA: return "CUDA error";
    case PHIPM_ESTEP: return "step size control failed";
    case PHIPM_ENONFINITE: return "non-finite value";
    case PHIPM_ESINGULAR: return "singular Pade denominator";
    default: return "unknown status";
    }
}

const char *phipm_last_error(const phipm_ctx *c) { return c ? c->err : "null context"; }

int phipm_get_profile(const phipm_ctx *c, phipm_profile *out)
{
    if (!c || !out) return PHIPM_EINVAL;
    *out = c->acc;
    return PHIPM_OK;
}

void phipm_reset_profile(phipm_ctx *c)
{
    if (!c) return;
    c->acc = phipm_profile{};
    c->tracebuf.clear();
    c->ntrace = 0;
}

int phipm_get_trace(const phipm_ctx *c, phipm_trace_rec *out, int max, int *count)
{
    if (!c || !count || (max > 0 && !out)) return PHIPM_EINVAL;
    const int nrec = (int)std::min<size_t>(c->tracebuf.size(), (size_t)std::max(max, 0));
    for (int i = 0; i < nrec; i++) out[i] = c->tracebuf[i];
    *count = (int)c->ntrace;
    return PHIPM_OK;
}

int phipm_krylov_path(const phipm_ctx *c)
{
    return c ? c->krylov_path : PHIPM_PATH_NONE;
}

int phipm_brick_plan(int nx, int ny, int nz, int ctas, int64_t smem_bytes, int *out10)
{
    if (!out10 || nx < 1 || ny < 1 || nz < 1 || ctas < 1 || smem_bytes < 0) return PHIPM_EINVAL;
    BrickGeom g;
    if (!brick_geometry(nx, ny, nz, ctas, (size_t)smem_bytes, g)) return -1;
    const int v[10] = {g.py, g.pz, g.ylen, g.zlen, g.nseg, g.ncol, g.ngrp, g.ppg, g.lstride, g.pstride};
    for (int i = 0; i < 10; i++) out10[i] = v[i];
    return PHIPM_OK;
}

int phipm_wrec_path(const phipm_ctx *c)
{
    return c ? c->wrec_path : PHIPM_PATH_NONE;
}

int phipm_get_clocks(const phipm_ctx *c, long long *out16)
{
    if (!c || !out16) return PHIPM_EINVAL;
    for (int i = 0; i < 16; i++) out16[i] = c->expm_clk_h ? c->expm_clk_h[i] : 0;
    return PHIPM_OK;
}

int phipm_get_attempts(const phipm_ctx *c, phipm_attempt *out, int max, int *count)
{
    if (!c || !count || (max > 0 && !out)) return PHIPM_EINVAL;
    if (c->ss_att_pending > 0) {                     // a device-driven solve: records still on the device
        phipm_ctx *cm = const_cast<phipm_ctx *>(c);
        static_assert(sizeof(SsAttempt) == sizeof(phipm_attempt), "attempt record layouts");
        cm->attempts.resize(c->ss_att_pending);
        if (cudaMemcpy(cm->attempts.data(), c->ss_att_d, sizeof(SsAttempt) * c->ss_att_pending,
                       cudaMemcpyDeviceToHost) != cudaSuccess)
            return set_err(cm, PHIPM_ECUDA, "attempt records: copy failed");
        cm->ss_att_pending = 0;
    }
    const int nrec = (int)std::min<size_t>(c->attempts.size(), (size_t)std::max(max, 0));
    for (int i = 0; i < nrec; i++) out[i] = c->attempts[i];
    *count = (int)c->nattempts;
    return PHIPM_OK;
}

void phipm_destroy(phipm_ctx *c)
{
    if (!c) return;
    cudaStreamSynchronize(c->stream);
    for (auto &r : c->pending) { c->pool.push_back(r.a); c->pool.push_back(r.b); }
    for (auto e : c->pool) cudaEventDestroy(e);
    if (c->ev_binf) cudaEventDestroy(c->ev_binf);
    if (c->stream2) {
        cudaStreamSynchronize(c->stream2);
        cudaStreamDestroy(c->stream2);
    }
    if (c->ev_main) cudaEventDestroy(c->ev_main);
    if (c->ss_att_d) cudaFree(c->ss_att_d);
    for (auto &g : c->graphs) cudaGraphExecDestroy(g.exec);
    if (c->ss_out_h) cudaFreeHost(c->ss_out_h);
    if (c->ev_spec) cudaEventDestroy(c->ev_spec);
    cudaFree(c->V); cudaFree(c->W); cudaFree(c->Y); cudaFree(c->U); cudaFree(c->H); cudaFree(c->sigma); cudaFree(c->g);
    cudaFree(c->part_mx); cudaFree(c->raw_mx); cudaFree(c->counter_mx); cudaFree(c->dec_d);
    cudaFree(c->part); cudaFree(c->part2); cudaFree(c->comb); cudaFree(c->combd); cudaFree(c->scratch); cudaFree(c->raw);
    cudaFree(c->counter); cudaFree(c->st); cudaFree(c->tlo); cudaFree(c->thi); cudaFree(c->off16);
    cudaFree(c->hu); cudaFree(c->hw); cudaFree(c->hrp); cudaFree(c->hcol); cudaFree(c->hval);
    if (c->res_h) cudaFreeHost(c->res_h);
    if (c->mx_h) cudaFreeHost(c->mx_h);
    if (c->expm_clk_h) cudaFreeHost(c->expm_clk_h);
    if (c->kclk_d) {
        // dump: int32 count, then per launch int32 {cls, grid, ncols} and grid*8 uint64 stamps
        FILE *f = fopen(c->kclk_path, "wb");
        if (f) {
            const int cnt = (int)c->kclk_recs.size();
            fwrite(&cnt, 4, 1, f);
            std::vector<unsigned long long> h((size_t)KCLK_GRID * 8);
            for (int i = 0; i < cnt; i++) {
                const auto &r = c->kclk_recs[i];
                fwrite(&r, sizeof(r), 1, f);
                cudaMemcpy(h.data(), c->kclk_d + (size_t)i * KCLK_GRID * 8, sizeof(unsigned long long) * r.grid * 8,
                           cudaMemcpyDeviceToHost);
                fwrite(h.data(), sizeof(unsigned long long), (size_t)r.grid * 8, f);
            }
            fclose(f);
        }
        cudaFree(c->kclk_d);
        if (c->pclk_d) {
            std::string pp = std::string(c->kclk_path) + ".p";
            FILE *g = fopen(pp.c_str(), "wb");
            if (g) {
                const int cnt = (int)c->pclk_recs.size();
                fwrite(&cnt, 4, 1, g);
                for (const auto &r : c->pclk_recs) {
                    const size_t nst = (size_t)2 * r.steps * r.grid * 2;
                    std::vector<unsigned long long> h(nst);
                    cudaMemcpy(h.data(), c->pclk_d + r.off, nst * 8, cudaMemcpyDeviceToHost);
                    int hd[2] = {r.grid, r.steps};
                    fwrite(hd, 4, 2, g);
                    fwrite(h.data(), 8, nst, g);
                }
                fclose(g);
            }
            cudaFree(c->pclk_d);
        }
    }
    if (c->raw_h) cudaFreeHost(c->raw_h);
    delete c;
}

int phipm_create(phipm_ctx **out, int64_t n_max, int m_max, int p_max, void *stream)
{
    if (!out) return PHIPM_EINVAL;
    *out = nullptr;
    if (n_max <= 0 || n_max >= ((int64_t)1 << 31) || m_max < 1 || m_max + 1 > MAXD || p_max < 0 || p_max > P_MAX_ABS - 0)
        return PHIPM_EINVAL;
    phipm_ctx *c = new phipm_ctx();
    c->stream = (cudaStream_t)stream;
    c->n_max = n_max;
    c->m_max = m_max;
    c->p_max = p_max;
    c->ldv = (n_max + 31) / 32 * 32;
    c->kmax = m_max + p_max + 1;
    cudaError_t e = cudaGetDevice(&c->dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, c->dev);
    if (e != cudaSuccess) {
        snprintf(c->err, sizeof(c->err), "no CUDA device: %s", cudaGetErrorString(e));
        delete c;
        return PHIPM_ECUDA;
    }
    // streaming kernels: grid = min(tiles, occupancy x SMs); allow large dynamic smem (halo tiles)
    {
        int optin = 0;
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->dev);
        const int mx = std::max(48 * 1024, optin - 8 * 1024);   // minus the kernels' static smem
        c->smem_optin = (size_t)mx;
        cudaFuncSetAttribute(spmv_stream_kernel<StencilOp, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(spmv_stream_kernel<StencilOp, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(spmv_stream_kernel<StencilOp, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(spmv_stream_kernel<CsrOp, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(spmv_stream_kernel<IdentOp, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(krylov_small_kernel<StencilOp>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMALL_N * 8);
        cudaFuncSetAttribute(krylov_small_kernel<CsrOp>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMALL_N * 8);
        ss_set_smem<StencilOp, 2>(mx);
        ss_set_smem<StencilOp, 4>(mx);
        ss_set_smem<StencilOp, 8>(mx);
        ss_set_smem<StencilOp, 16>(mx);
        ss_set_smem<CsrOp, 2>(mx);
        ss_set_smem<CsrOp, 4>(mx);
        ss_set_smem<CsrOp, 8>(mx);
        ss_set_smem<CsrOp, 16>(mx);
        for (int dc = 1; dc <= 4; dc++)
            for (ClusterLzFn f : {cluster_lz_fn<256, 4>(dc), cluster_lz_fn<512, 8>(dc)}) {
                cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
                cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            }
        cudaFuncSetAttribute(spmv_stream_kernel<CsrOp, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(spmv_stream_kernel<CsrOp, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(spmv_stream_kernel<CsrOp, 2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(spmv_stream_kernel<CsrOp, 4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(spmv_stream_kernel<CsrOp, 8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(spmv_stream_kernel<IdentOp, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(spmv_stream_kernel<IdentOp, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        for (int d = 1; d <= 4; d++) {
            StencilOp op{};
            op.dim = d == 4 ? 2 : d;
            op.diag = d == 4;
            cudaFuncSetAttribute(persist_tm_fn(op), cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        }
        cudaFuncSetAttribute(krylov_brick_tm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(krylov_brick_tm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(krylov_brick_halo_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(krylov_brick_halo_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(wrec_brick_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        for (int d = 1; d <= 4; d++) {
            StencilOp op{};
            op.dim = d == 4 ? 2 : d;
            op.diag = d == 4;
            cudaFuncSetAttribute(wrec_fn(op), cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        }
        persist_set_smem<4>(mx);
        persist_set_smem<2>(mx);
        cudaFuncSetAttribute(spmm_csr_ring_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(spmm_csr_ring_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(spmm_csr_ring_kernel<SPMM_MAXB>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        int occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, maxabs_kernel, NT, 0);
        c->occ_axpy = std::max(1, occ);
        c->occ_spmv = 4;
        c->pstride = std::max(c->sm_count * 8, 1024);
    }
    int smem_optin = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->dev);
    {
        cudaFuncAttributes fa;
        cudaFuncGetAttributes(&fa, expm_kernel<true, true>);     // the larger static smem of the two
        c->expm_smem_limit = (size_t)std::max(0, smem_optin - (int)fa.sharedSizeBytes - 1024);
        cudaFuncSetAttribute(expm_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->expm_smem_limit);
        cudaFuncSetAttribute(expm_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->expm_smem_limit);
    }
    cudaGetLastError();

    const size_t vbytes = (size_t)c->ldv * sizeof(double);
    bool ok = true;
    auto A = [&](void **p, size_t b) {
        if (!ok) return;
        if (cudaMalloc(p, b) != cudaSuccess) ok = false;
        else cudaMemset(*p, 0, b);
    };
    A((void **)&c->V, vbytes * (m_max + 1));
    A((void **)&c->W, vbytes * (p_max + 1));
    A((void **)&c->Y, vbytes);
    A((void **)&c->U, vbytes);
    A((void **)&c->H, sizeof(double) * (m_max + 1) * m_max);
    A((void **)&c->sigma, sizeof(double) * (MAXD + 1));
    A((void **)&c->g, sizeof(double) * (MAXD + 1));
    A((void **)&c->part, sizeof(double) * (size_t)c->pstride * (MAXD + 2));
    A((void **)&c->part2, sizeof(double) * (size_t)c->pstride * (MAXD + 2));
    A((void **)&c->dec_d, sizeof(int) * 4);
    A((void **)&c->part_mx, sizeof(double) * (size_t)c->pstride * 2);
    A((void **)&c->raw_mx, sizeof(double) * 2);
    A((void **)&c->counter_mx, sizeof(unsigned) * 8);
    A((void **)&c->comb, sizeof(double) * (MAXD + 1));
    A((void **)&c->combd, sizeof(double) * (P_MAX_ABS + 1));
    {
        const int kp = (c->kmax + 7) & ~7;
        A((void **)&c->scratch, sizeof(double) * 6 * (size_t)expm_ld(kp) * kp);
    }
    A((void **)&c->raw, sizeof(double) * (MAXD + 2));
    A((void **)&c->counter, sizeof(unsigned) * 8);
    if (ok && cudaEventCreateWithFlags(&c->ev_binf, cudaEventDisableTiming) != cudaSuccess) ok = false;
    if (ok && cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking) != cudaSuccess) ok = false;
    if (ok && cudaEventCreateWithFlags(&c->ev_main, cudaEventDisableTiming) != cudaSuccess) ok = false;
    if (ok && cudaEventCreateWithFlags(&c->ev_spec, cudaEventDisableTiming) != cudaSuccess) ok = false;
    A((void **)&c->st, sizeof(DevState));
    c->ntile_cap = n_max / 512 + 2;
    A((void **)&c->tlo, sizeof(int32_t) * c->ntile_cap);
    A((void **)&c->thi, sizeof(int32_t) * c->ntile_cap);
    if (ok && cudaHostAlloc((void **)&c->res_h, sizeof(AttemptResult), cudaHostAllocMapped) != cudaSuccess) ok = false;
    if (ok && cudaHostAlloc((void **)&c->mx_h, sizeof(*c->mx_h), cudaHostAllocMapped) != cudaSuccess) ok = false;
    if (ok && cudaHostGetDevicePointer((void **)&c->mx_d, c->mx_h, 0) != cudaSuccess) ok = false;
    if (ok) memset(c->mx_h, 0, sizeof(*c->mx_h));
    if (ok && cudaHostGetDevicePointer((void **)&c->res_d, c->res_h, 0) != cudaSuccess) ok = false;
    if (ok && cudaHostAlloc((void **)&c->raw_h, sizeof(double) * (MAXD + 2), cudaHostAllocDefault) != cudaSuccess) ok = false;
    if (ok && getenv("PHIPM_EXPM_CLOCKS")) {
        if (cudaHostAlloc((void **)&c->expm_clk_h, sizeof(long long) * 16, cudaHostAllocMapped) != cudaSuccess ||
            cudaHostGetDevicePointer((void **)&c->expm_clk_d, c->expm_clk_h, 0) != cudaSuccess)
            ok = false;
    }
    if (ok && getenv("PHIPM_KCLOCKS")) {
        c->kclk_path = getenv("PHIPM_KCLOCKS");
        if (cudaMalloc((void **)&c->pclk_d, sizeof(unsigned long long) * PCLK_CAP) != cudaSuccess ||
            cudaMemset(c->pclk_d, 0, sizeof(unsigned long long) * PCLK_CAP) != cudaSuccess ||
            cudaMalloc((void **)&c->kclk_d, sizeof(unsigned long long) * KCLK_MAXL * KCLK_GRID * 8) != cudaSuccess ||
            cudaMemset(c->kclk_d, 0, sizeof(unsigned long long) * KCLK_MAXL * KCLK_GRID * 8) != cudaSuccess)
            ok = false;
    }
    if (ok && cudaDeviceSynchronize() != cudaSuccess) ok = false;
    if (!ok) {
        cudaGetLastError();
        phipm_destroy(c);
        return PHIPM_ENOMEM;
    }
    memset(c->res_h, 0, sizeof(AttemptResult));
    *out = c;
    return PHIPM_OK;
}

int phipm_solve_stencil(phipm_ctx *c, double t, const phipm_stencil *S, int p, const double *const *u,
                        const phipm_opts *opts, double *w, phipm_stats *stats)
{
    if (!c) return PHIPM_EINVAL;
    StencilOp op;
    int rc = make_stencil(c, S, op);
    if (rc) return rc;
    phipm_opts o = resolve_opts(opts);
    rc = check_common(c, t, op.n, p, u, w, o);
    if (rc) return rc;
    c->prof = o.profile != 0;
    c->trace = o.profile >= 2;
    return solve_impl(c, t, op, 16.0 * (double)op.n, stencil_nnz(op), stencil_infnorm(op), p, u, o, w, stats);
}

int phipm_solve_csr(phipm_ctx *c, double t, const phipm_csr *A, int p, const double *const *u,
                    const phipm_opts *opts, double *w, phipm_stats *stats)
{
    if (!c) return PHIPM_EINVAL;
    CsrOp op;
    int rc = make_csr(c, A, op);
    if (rc) return rc;
    phipm_opts o = resolve_opts(opts);
    rc = check_common(c, t, op.n, p, u, w, o);
    if (rc) return rc;
    c->prof = o.profile != 0;
    c->trace = o.profile >= 2;
    // a1 setup, once per call: the operator's layout (row_ptr, col), and ||A||_inf.  On the banded
    // uniform-row path (x ring) the first w-recurrence SpMV reads val anyway and computes ||A||_inf
    // (PHIPM_OPT_FUSE_ANORM), so the analysis pass does not read val; otherwise a second pass does.
    double normA = 0.0;
    // int16 column offsets for the x-ring path (PHIPM_OPT_CSR_OFF16): candidates are uniform-row
    // matrices (nnz = L n, L % 4 == 0); the analysis pass writes them while it reads col
    int16_t *o16 = nullptr;
    if (opt(c, PHIPM_OPT_CSR_OFF16) && A->nnz > 0 && A->nnz % op.n == 0 && (A->nnz / op.n) % 4 == 0 &&
        A->nnz / op.n <= 128 && op.n > SMALL_N && t > 0.0) {
        if (A->nnz > c->off16_cap) {
            cudaFree(c->off16);
            c->off16 = nullptr;
            c->off16_cap = 0;
            if (cudaMalloc(&c->off16, sizeof(int16_t) * A->nnz) == cudaSuccess) c->off16_cap = A->nnz;
            else cudaGetLastError();
        }
        o16 = c->off16;
    }
    rc = analyze_csr(c, op, A->nnz, &normA, o16 ? 6 : 2, o16);
    if (rc) return rc;
    const bool fuse = op.ring && opt(c, PHIPM_OPT_FUSE_ANORM) && p >= 1 && op.n > SMALL_N && t > 0.0;
    if (fuse) {
        CK(cudaMemsetAsync(&c->st->anorm_bits, 0, sizeof(unsigned long long), c->stream));
        c->fuse_anorm = true;
        normA = -1.0;
    } else {
        CsrOp tmp = op;
        rc = analyze_csr(c, tmp, A->nnz, &normA, 1);
        if (rc) return rc;
    }
    rc = enable_csr_window(c, op);
    if (rc) return rc;
    rc = solve_impl(c, t, op, csr_bytes(op, A->nnz), A->nnz, normA, p, u, o, w, stats);
    c->fuse_anorm = false;
    return rc;
}

int phipm_solve_csr_batch(phipm_ctx *const *ctx, int nb, const double *t, const phipm_csr *A, const int *p,
                          const double *const *const *u, const phipm_opts *opts, double *const *w,
                          phipm_stats *stats, int *status)
{
    if (nb > 0 && (!t || !A || !p || !u || !w)) return PHIPM_EINVAL;
    return run_batch(ctx, nb, status, [&](int b) {
        return phipm_solve_csr(ctx[b], t[b], &A[b], p[b], u[b], opts, w[b], stats ? &stats[b] : nullptr);
    });
}

int phipm_solve_stencil_batch(phipm_ctx *const *ctx, int nb, const double *t, const phipm_stencil *S,
                              const int *p, const double *const *const *u, const phipm_opts *opts,
                              double *const *w, phipm_stats *stats, int *status)
{
    if (nb > 0 && (!t || !S || !p || !u || !w)) return PHIPM_EINVAL;
    // Every problem a device-driven solve (one kernel each, no host decisions): this thread launches them all,
    // then collects them (solves on distinct SMs; host threads would only add wake-ups and contention)
    {
        const phipm_opts o = resolve_opts(opts);
        bool all = nb > 0 && ctx && o.symmetric && o.expm_method == PHIPM_EXPM_TAYLOR && !o.profile;
        for (int b = 0; all && b < nb; b++) {
            StencilOp op;
            all = ctx[b] && opt(ctx[b], PHIPM_OPT_DEVSOLVE) && make_stencil(nullptr, &S[b], op) == PHIPM_OK &&
                  op.n <= SMALL_N && p[b] + 1 <= SS_MAXU && t[b] > 0.0;
            for (int b2 = 0; all && b2 < b; b2++) all = ctx[b] != ctx[b2];
        }
        if (all) {
            std::vector<int> st((size_t)nb, PHIPM_OK);
            for (int b = 0; b < nb; b++) {
                const cudaError_t e = cudaSetDevice(ctx[b]->dev);
                if (e != cudaSuccess) {
                    st[b] = set_err(ctx[b], PHIPM_ECUDA, "cudaSetDevice(%d): %s", ctx[b]->dev, cudaGetErrorString(e));
                    continue;
                }
                ctx[b]->defer = true;
                st[b] = phipm_solve_stencil(ctx[b], t[b], &S[b], p[b], u[b], opts, w[b], stats ? &stats[b] : nullptr);
                ctx[b]->defer = false;
            }
            int rc = PHIPM_OK;
            for (int b = 0; b < nb; b++) {
                if (st[b] == PHIPM_OK && ctx[b]->deferred) {
                    cudaSetDevice(ctx[b]->dev);
                    phipm_stats sb{};
                    st[b] = finish_small_dev(ctx[b], sb);
                    if (stats) stats[b] = sb;
                }
                if (status) status[b] = st[b];
                if (rc == PHIPM_OK && st[b] != PHIPM_OK) rc = st[b];
            }
            return rc;
        }
    }
    return run_batch(ctx, nb, status, [&](int b) {
        return phipm_solve_stencil(ctx[b], t[b], &S[b], p[b], u[b], opts, w[b], stats ? &stats[b] : nullptr);
    });
}

int phipm_solve_csr_block(phipm_ctx *const *ctx, int nb, double t, const phipm_csr *A, int p,
                          const double *const *const *u, const phipm_opts *opts, double *const *w,
                          phipm_stats *stats)
{
    if (!ctx || nb < 1 || nb > SPMM_MAXB || !u || !w) return PHIPM_EINVAL;
    for (int b = 0; b < nb; b++) {
        if (!ctx[b]) return PHIPM_EINVAL;
        for (int b2 = 0; b2 < b; b2++)
            if (ctx[b] == ctx[b2]) return set_err(ctx[0], PHIPM_EINVAL, "block solve: contexts must be distinct");
        if (ctx[b]->dev != ctx[0]->dev) return set_err(ctx[0], PHIPM_EINVAL, "block solve: contexts on different devices");
    }
    phipm_ctx *c0 = ctx[0];
    CsrOp op;
    int rc = make_csr(c0, A, op);
    if (rc) return rc;
    phipm_opts o = resolve_opts(opts);
    for (int b = 0; b < nb; b++) {
        rc = check_common(ctx[b], t, op.n, p, u[b], w[b], o);
        if (rc) return rc == PHIPM_EINVAL && b ? set_err(c0, PHIPM_EINVAL, "problem %d: %s", b, ctx[b]->err) : rc;
        for (int b2 = 0; b2 < nb; b2++)
            if (b2 != b && w[b] == w[b2]) return set_err(c0, PHIPM_EINVAL, "block solve: outputs must be distinct");
    }
    if (o.fixed_m < 0) return PHIPM_EINVAL;
    std::vector<cudaStream_t> saved((size_t)nb);
    for (int b = 0; b < nb; b++) {
        saved[b] = ctx[b]->stream;
        ctx[b]->prof = b == 0 && o.profile != 0;
        ctx[b]->trace = b == 0 && o.profile >= 2;
    }
    if (cudaSetDevice(c0->dev) != cudaSuccess) return set_err(c0, PHIPM_ECUDA, "cudaSetDevice failed");
    // the other contexts' work is ordered on ctx[0]'s stream for the duration of the call
    for (int b = 1; b < nb; b++) {
        cudaEvent_t e = ev_get(ctx[b]);
        cudaEventRecord(e, saved[b]);
        cudaStreamWaitEvent(c0->stream, e, 0);
        ctx[b]->pool.push_back(e);
        ctx[b]->stream = c0->stream;
    }
    double normA = 0.0;
    rc = analyze_csr(c0, op, A->nnz, &normA);
    if (!rc) rc = solve_block_impl(ctx, nb, t, op, csr_bytes(op, A->nnz), A->nnz, normA, p, u, o, w, stats);
    for (int b = 1; b < nb; b++) ctx[b]->stream = saved[b];
    return rc;
}

int phipm_reserve_host_csr(phipm_ctx *c, int64_t nnz_max)
{
    if (!c || nnz_max < 0) return PHIPM_EINVAL;
    if (nnz_max <= c->nnz_cap && c->hrp) return PHIPM_OK;
    cudaFree(c->hrp); cudaFree(c->hcol); cudaFree(c->hval);
    c->hrp = nullptr; c->hcol = nullptr; c->hval = nullptr; c->nnz_cap = 0;
    if (cudaMalloc(&c->hrp, sizeof(int32_t) * (c->n_max + 1)) != cudaSuccess ||
        cudaMalloc(&c->hcol, sizeof(int32_t) * std::max<int64_t>(nnz_max, 1)) != cudaSuccess ||
        cudaMalloc(&c->hval, sizeof(double) * std::max<int64_t>(nnz_max, 1)) != cudaSuccess) {
        cudaGetLastError();
        return set_err(c, PHIPM_ENOMEM, "reserve_host_csr: allocation failed");
    }
    c->nnz_cap = nnz_max;
    return PHIPM_OK;
}

static int host_stage_u(phipm_ctx *c, int64_t n, int p, const double *const *host_u, const double **du)
{
    if (!host_u) return set_err(c, PHIPM_EINVAL, "null u");
    if (!c->hu) {
        if (cudaMalloc(&c->hu, sizeof(double) * c->ldv * (c->p_max + 1)) != cudaSuccess ||
            cudaMalloc(&c->hw, sizeof(double) * c->ldv) != cudaSuccess) {
            cudaGetLastError();
            return set_err(c, PHIPM_ENOMEM, "host staging allocation failed");
        }
    }
    for (int k = 0; k <= p; k++) {
        if (!host_u[k]) return set_err(c, PHIPM_EINVAL, "null u[%d]", k);
        double *d = c->hu + (int64_t)k * c->ldv;
        CK(cudaMemcpyAsync(d, host_u[k], n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        du[k] = d;
    }
    return PHIPM_OK;
}

int phipm_solve_csr_host(phipm_ctx *c, double t, const phipm_csr *A, int p, const double *const *host_u,
                         const phipm_opts *opts, double *host_w, phipm_stats *stats)
{
    if (!c || !A || !host_w || !A->row_ptr || (A->nnz > 0 && (!A->col || !A->val))) return PHIPM_EINVAL;
    if (A->n <= 0 || A->n > c->n_max || p < 0 || p > c->p_max) return set_err(c, PHIPM_EINVAL, "bad size");
    int rc = phipm_reserve_host_csr(c, std::max(A->nnz, c->nnz_cap));
    if (rc) return rc;
    CK(cudaMemcpyAsync(c->hrp, A->row_ptr, sizeof(int32_t) * (A->n + 1), cudaMemcpyHostToDevice, c->stream));
    if (A->nnz > 0) {
        CK(cudaMemcpyAsync(c->hcol, A->col, sizeof(int32_t) * A->nnz, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(c->hval, A->val, sizeof(double) * A->nnz, cudaMemcpyHostToDevice, c->stream));
    }
    const double *du[P_MAX_ABS + 1];
    rc = host_stage_u(c, A->n, p, host_u, du);
    if (rc) return rc;
    phipm_csr dA = *A;
    dA.row_ptr = c->hrp;
    dA.col = c->hcol;
    dA.val = c->hval;
    rc = phipm_solve_csr(c, t, &dA, p, du, opts, c->hw, stats);
    if (rc && rc != PHIPM_ESTEP) return rc;
    CK(cudaMemcpyAsync(host_w, c->hw, sizeof(double) * A->n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return rc;
}

int phipm_solve_stencil_host(phipm_ctx *c, double t, const phipm_stencil *S, int p, const double *const *host_u,
                             const phipm_opts *opts, double *host_w, phipm_stats *stats)
{
    if (!c || !host_w) return PHIPM_EINVAL;
    StencilOp op;
    int rc = make_stencil(c, S, op);
    if (rc) return rc;
    if (op.n > c->n_max || p < 0 || p > c->p_max) return set_err(c, PHIPM_EINVAL, "bad size");
    const double *du[P_MAX_ABS + 1];
    rc = host_stage_u(c, op.n, p, host_u, du);
    if (rc) return rc;
    rc = phipm_solve_stencil(c, t, S, p, du, opts, c->hw, stats);
    if (rc && rc != PHIPM_ESTEP) return rc;
    CK(cudaMemcpyAsync(host_w, c->hw, sizeof(double) * op.n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return rc;
}

// ---- kernel-level entry points ----

double phipm_inf_norm_stencil(const phipm_stencil *S)
{
    StencilOp op;
    if (make_stencil(nullptr, S, op) != PHIPM_OK) return -1.0;
    return stencil_infnorm(op);
}

int64_t phipm_stencil_nnz(const phipm_stencil *S)
{
    StencilOp op;
    if (make_stencil(nullptr, S, op) != PHIPM_OK) return -1;
    return stencil_nnz(op);
}

int phipm_csr_from_stencil(phipm_ctx *c, const phipm_stencil *S, int32_t *row_ptr, int32_t *col, double *val)
{
    if (!c || !row_ptr || !col || !val) return PHIPM_EINVAL;
    StencilOp op;
    int rc = make_stencil(c, S, op);
    if (rc) return rc;
    const int grid = (int)std::min<int64_t>((op.n + 1 + NT - 1) / NT, (int64_t)c->sm_count * 8);
    csr_from_stencil_kernel<<<grid, NT, 0, c->stream>>>(op, row_ptr, col, val);
    c->acc.launches++;
    CK(cudaGetLastError());
    return sync(c);
}

int phipm_spmv_csr(phipm_ctx *c, const phipm_csr *A, const double *x, double *y)
{
    if (!c || !x || !y) return PHIPM_EINVAL;
    CsrOp op;
    int rc = make_csr(c, A, op);
    if (rc) return rc;
    if (op.n > c->n_max) return set_err(c, PHIPM_EINVAL, "n > n_max");
    CK(cudaMemcpyAsync(c->Y, x, op.n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    double normA = 0.0;
    rc = analyze_csr(c, op, A->nnz, &normA);
    if (rc) return rc;
    rc = enable_csr_window(c, op);
    if (rc) return rc;
    SpmvArgs s = spmv0();
    s.x = c->Y;
    s.y = y;
    rc = launch_spmv(c, op, s, csr_bytes(op, A->nnz));
    if (rc) return rc;
    return sync(c);
}

int phipm_spmv_stencil(phipm_ctx *c, const phipm_stencil *S, const double *x, double *y)
{
    if (!c || !x || !y) return PHIPM_EINVAL;
    StencilOp op;
    int rc = make_stencil(c, S, op);
    if (rc) return rc;
    if (op.n > c->n_max) return set_err(c, PHIPM_EINVAL, "n > n_max");
    CK(cudaMemcpyAsync(c->Y, x, op.n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    SpmvArgs s = spmv0();
    s.x = c->Y;
    s.y = y;
    rc = launch_spmv(c, op, s, 16.0 * (double)op.n);
    if (rc) return rc;
    return sync(c);
}

int phipm_dot(phipm_ctx *c, int64_t n, const double *x, const double *y, double *result)
{
    if (!c || !x || !y || !result || n <= 0) return PHIPM_EINVAL;
    if (n > c->n_max) return set_err(c, PHIPM_EINVAL, "n > n_max");
    // stage both operands in padded workspace vectors (TMA segment reads)
    CK(cudaMemcpyAsync(c->Y, x, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(c->U, y, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    SpmvArgs s = spmv0();
    s.x = c->Y;
    s.V = c->U;
    s.ldv = c->ldv;
    s.d0 = 0;
    s.nd = 1;
    s.fin = FIN_RAW;
    int rc = launch_spmv(c, IdentOp{n}, s, 8.0 * (double)n);
    if (rc) return rc;
    CK(cudaMemcpyAsync(c->raw_h, c->raw, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    rc = sync(c);
    if (rc) return rc;
    *result = c->raw_h[0];
    return PHIPM_OK;
}

int phipm_inf_norm_csr(phipm_ctx *c, const phipm_csr *A, double *result)
{
    if (!c || !result) return PHIPM_EINVAL;
    CsrOp op;
    int rc = make_csr(c, A, op);
    if (rc) return rc;
    return analyze_csr(c, op, A->nnz, result);
}

int phipm_expm(phipm_ctx *c, int K, const double *A, double *E)
{
    if (!c || !A || !E || K < 1 || K > c->kmax) return PHIPM_EINVAL;
    ExpmArgs a;
    memset(&a, 0, sizeof(a));
    a.mode = 1;
    a.method = c->expm_method;
    a.K = K;
    a.Ain = A;
    a.Eout = E;
    int rc = launch_expm(c, a, K);
    if (rc) return rc;
    rc = sync(c);
    if (rc) return rc;
    AttemptResult R;
    memcpy(&R, (const void *)c->res_h, sizeof(R));
    if (R.status == 5) return set_err(c, PHIPM_ENONFINITE, "expm: non-finite");
    if (R.status == 6) return set_err(c, PHIPM_ESINGULAR, "expm: singular");
    return PHIPM_OK;
}

int phipm_phi_pair(phipm_ctx *c, int mu, const double *H, int ldh, double tau, int p, double *phip, double *phip1,
                   double *normH1)
{
    if (!c || !H || !phip || !phip1 || mu < 1 || ldh < mu || p < 0 || p > c->p_max || mu > c->m_max)
        return PHIPM_EINVAL;
    ExpmArgs a;
    memset(&a, 0, sizeof(a));
    a.mode = 2;
    a.method = c->expm_method;
    a.tridiag = c->expm_method == PHIPM_EXPM_CHEBYSHEV ? 1 : 0;   // the Chebyshev method reads the band
    a.m = mu;
    a.p = p;
    a.tau = tau;
    a.H = H;
    a.ldh = ldh;
    a.phip_out = phip;
    a.phip1_out = phip1;
    int rc = launch_expm(c, a, mu + p + 1);
    if (rc) return rc;
    rc = sync(c);
    if (rc) return rc;
    if (((const volatile AttemptResult *)c->res_h)->status == CHEB_STATUS_RANGE) {
        a.method = PHIPM_EXPM_TAYLOR;
        a.tridiag = 0;
        rc = launch_expm(c, a, mu + p + 1);
        if (rc) return rc;
        rc = sync(c);
        if (rc) return rc;
    }
    if (c->expm_clk_h && c->expm_clk_h[8] == -1) {
        const long long *k = c->expm_clk_h;
        fprintf(stderr, "cheb K=%d cycles: gershgorin %lld | sturm %lld | nodes %lld | dct %lld | trunc %lld | "
                        "recurrence %lld | N=%lld nd=%lld mu=%lld\n",
                mu + p + 1, k[1] - k[0], k[2] - k[1], k[3] - k[2], k[4] - k[3], k[5] - k[4], k[6] - k[5],
                k[7] >> 32, (k[7] >> 16) & 0xffff, k[7] & 0xffff);
        double lo, hi;
        memcpy(&lo, &k[9], 8);
        memcpy(&hi, &k[10], 8);
        fprintf(stderr, "  interval of tau T: [%.6g, %.6g]\n", lo, hi);
    } else if (c->expm_clk_h) {
        const long long *k = c->expm_clk_h;
        fprintf(stderr, "expm K=%d cycles: build %lld | A2,A3,A4 %lld | norms,alpha,scale %lld | Horner %lld | "
                        "squarings %lld | m=%lld s=%lld\n",
                mu + p + 1, k[1] - k[0], k[2] - k[1], k[4] - k[2], k[3] - k[4], k[5] - k[3], k[7] >> 16,
                k[7] & 0xffff);
        fprintf(stderr, "  prep: norm loop %lld | sred+sync %lld | warp max %lld | degree %lld | scale %lld\n",
                k[8] - k[2], k[9] - k[8], k[10] - k[9], k[11] - k[10], k[4] - k[11]);
    }
    AttemptResult R;
    memcpy(&R, (const void *)c->res_h, sizeof(R));
    if (normH1) *normH1 = R.normH1;
    if (R.status == 5) return set_err(c, PHIPM_ENONFINITE, "phi_pair: non-finite");
    if (R.status == 6) return set_err(c, PHIPM_ESINGULAR, "phi_pair: singular");
    return PHIPM_OK;
}

} // extern "C"

template <class Op>
static int krylov_export(phipm_ctx *c, const Op &op, double bytes_op, double normA, const double *v, int m,
                         const phipm_opts *opts, double *V, double *H, int *k, int *brk, double *beta)
{
    phipm_opts o = resolve_opts(opts);
    if (!v || (!V) != (!H) || m < 1 || m > c->m_max) return set_err(c, PHIPM_EINVAL, "krylov: bad args");
    const int64_t n = op.n;
    if (n > c->n_max) return set_err(c, PHIPM_EINVAL, "krylov: n > n_max");
    CK(cudaMemsetAsync(c->H, 0, sizeof(double) * (c->m_max + 1) * c->m_max, c->stream));
    CK(cudaMemcpyAsync(c->Y, v, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    AxpyArgs a = axpy0();
    a.out = c->V;
    a.base = c->Y;
    a.a0h = 1.0;
    a.V = c->V;
    a.ldv = c->ldv;
    a.onorm = 1;
    a.fin = FIN_SEED;
    int rc = launch_axpy(c, n, a, PC_OTHER);
    if (rc) return rc;
    rc = enqueue_krylov(c, op, bytes_op, o.symmetric != 0, o.orth, 0, m, (double)n * EPS_MACH * normA);
    if (rc) return rc;
    DevState ds;
    CK(cudaMemcpyAsync(&ds, c->st, sizeof(ds), cudaMemcpyDeviceToHost, c->stream));
    rc = sync(c);
    if (rc) return rc;
    if (ds.aborted) {
        c->coop_dirty = true;
        return set_err(c, PHIPM_ECUDA, "persistent Krylov kernel: grid phase timed out");
    }
    const int kk = (ds.brk >= 0) ? std::min(ds.brk, m) : m;
    if (!V) {                                             // build only (no export): timing
        *k = kk;
        *brk = ds.brk >= 0 ? 1 : 0;
        *beta = ds.beta;
        return PHIPM_OK;
    }
    const int ncols = (ds.brk >= 0) ? kk : m + 1;
    dim3 grid((unsigned)std::min<int64_t>((n + 255) / 256, 1024), (unsigned)std::max(ncols, 1));
    if (ncols > 0) scale_columns_kernel<<<grid, 256, 0, c->stream>>>(n, ncols, c->V, c->ldv, c->sigma, V, n);
    CK(cudaGetLastError());
    CK(cudaMemcpy2DAsync(H, sizeof(double) * (m + 1), c->H, sizeof(double) * (c->m_max + 1),
                         sizeof(double) * (m + 1), m, cudaMemcpyDeviceToDevice, c->stream));
    rc = sync(c);
    if (rc) return rc;
    *k = kk;
    *brk = ds.brk >= 0 ? 1 : 0;
    *beta = ds.beta;
    return PHIPM_OK;
}

extern "C" {

int phipm_krylov_csr(phipm_ctx *c, const phipm_csr *A, const double *v, int m, const phipm_opts *opts, double *V,
                     double *H, int *k, int *brk, double *beta)
{
    if (!c || !k || !brk || !beta) return PHIPM_EINVAL;
    CsrOp op;
    int rc = make_csr(c, A, op);
    if (rc) return rc;
    double normA = 0.0;
    rc = analyze_csr(c, op, A->nnz, &normA);
    if (rc) return rc;
    rc = enable_csr_window(c, op);
    if (rc) return rc;
    return krylov_export(c, op, csr_bytes(op, A->nnz), normA, v, m, opts, V, H, k, brk, beta);
}

int phipm_krylov_stencil(phipm_ctx *c, const phipm_stencil *S, const double *v, int m, const phipm_opts *opts,
                         double *V, double *H, int *k, int *brk, double *beta)
{
    if (!c || !k || !brk || !beta) return PHIPM_EINVAL;
    StencilOp op;
    int rc = make_stencil(c, S, op);
    if (rc) return rc;
    return krylov_export(c, op, 16.0 * (double)op.n, stencil_infnorm(op), v, m, opts, V, H, k, brk, beta);
}

} // extern "C"
