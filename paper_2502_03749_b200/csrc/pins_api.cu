// pins_api.cu -- C ABI of libpins_b200.so (include/pins.h): workspace, kernel
// launchers, the Newton step and the host-driven PINS loop (Algorithm 2).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "pins.h"
#include "pins_kernels.cuh"
#include "pins_pass.cuh"
#include "pins_cg.cuh"
#include "pins_order.cuh"
#include "pins_tree.cuh"
#include "pins_treecl.cuh"
#include "pins_cert.cuh"

using namespace pins;

static thread_local char g_err[512] = "ok";
extern "C" const char *pins_last_error(void) { return g_err; }

#define PINS_CUDA(x)                                                                        \
    do {                                                                                    \
        cudaError_t e_ = (x);                                                               \
        if (e_ != cudaSuccess) {                                                            \
            snprintf(g_err, sizeof g_err, "%s:%d %s -> %s", __FILE__, __LINE__, #x,        \
                     cudaGetErrorString(e_));                                               \
            return PINS_ERR_CUDA;                                                           \
        }                                                                                   \
    } while (0)
#define PINS_TRY(x)                    \
    do {                               \
        int rc_ = (x);                 \
        if (rc_ != PINS_OK) return rc_; \
    } while (0)
#define PINS_ARG(cond, msg)                                              \
    do {                                                                 \
        if (!(cond)) {                                                   \
            snprintf(g_err, sizeof g_err, "invalid argument: %s", msg); \
            return PINS_ERR_ARG;                                         \
        }                                                                \
    } while (0)


// ---------------------------------------------------------------- profiling
// Device-time profile of this library's own launches (pins_prof_*, include/pins.h).
// Every launch is counted; when enabled, a pair of CUDA events brackets it on
// its own stream and pins_prof_read() folds the elapsed times per class.
namespace {
struct Prof {
    bool on = false;
    long long launches[PINS_PROF_NCLASS] = {};
    double ms[PINS_PROF_NCLASS] = {};
    double work[PINS_PROF_NCLASS] = {};   // algorithmic bytes / entries, where the host knows them
    std::vector<cudaEvent_t> pool;
    struct Pend { int cls; cudaEvent_t a, b; };
    std::vector<Pend> pend;
    cudaEvent_t get() {
        if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
        cudaEvent_t e = nullptr;
        cudaEventCreate(&e);
        return e;
    }
    void fold() {
        for (auto &p : pend) {
            float t = 0.f;
            if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&t, p.a, p.b) == cudaSuccess)
                ms[p.cls] += t;
            pool.push_back(p.a);
            pool.push_back(p.b);
        }
        pend.clear();
    }
};
Prof g_prof;
struct ProfScope {
    int cls;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    ProfScope(int c, cudaStream_t s) : cls(c), st(s) {
        ++g_prof.launches[c];
        if (g_prof.on) { a = g_prof.get(); cudaEventRecord(a, st); }
    }
    ~ProfScope() {
        if (!a) return;
        cudaEvent_t b = g_prof.get();
        cudaEventRecord(b, st);
        g_prof.pend.push_back({cls, a, b});
        if (g_prof.pend.size() > 4096) g_prof.fold();
    }
};
}  // namespace
#define LAUNCH(cls, st, ...)            \
    do {                                \
        ProfScope ps_((cls), (st));     \
        __VA_ARGS__;                    \
    } while (0)

extern "C" void pins_prof_enable(int32_t on) { g_prof.on = on != 0; }
extern "C" void pins_prof_reset(void) {
    g_prof.fold();
    const unsigned long long z[3] = {0, 0, 0};
    cudaMemcpyToSymbol(pins::g_surv, z, sizeof z);
    for (int c = 0; c < PINS_PROF_NCLASS; ++c) { g_prof.launches[c] = 0; g_prof.ms[c] = 0.0; g_prof.work[c] = 0.0; }
}
extern "C" int pins_prof_read_work(int32_t cls, double *work) {
    PINS_ARG(cls >= 0 && cls < PINS_PROF_NCLASS && work, "class / pointer");
    *work = g_prof.work[cls];
    if (cls == PINS_PROF_SWEEP_ROW || cls == PINS_PROF_EVAL || cls == PINS_PROF_KSWEEP) {
        // counted on the device: survivors (dense passes), listed entries walked (ELL walk)
        unsigned long long sv[3] = {0, 0, 0};
        PINS_CUDA(cudaMemcpyFromSymbol(sv, pins::g_surv, sizeof sv));
        *work = (double)sv[cls == PINS_PROF_SWEEP_ROW ? 0 : cls == PINS_PROF_EVAL ? 1 : 2];
    }
    return PINS_OK;
}
extern "C" int pins_prof_read(int32_t cls, int64_t *launches, double *ms) {
    PINS_ARG(cls >= 0 && cls < PINS_PROF_NCLASS && launches && ms, "class / pointers");
    g_prof.fold();
    *launches = g_prof.launches[cls];
    *ms = g_prof.ms[cls];
    return PINS_OK;
}

namespace {

// Device buffer owned by its holder (freed by the destructor; not copyable).
struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
    unsigned gen = 0;      // bumped on every (re)allocation: the new memory holds no prior content
                           // (cudaMalloc may hand back the same address, so pointers cannot tell)
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

int ensure(DevBuf &b, size_t bytes) {
    if (bytes == 0) bytes = 8;
    if (b.bytes >= bytes) return PINS_OK;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    cudaError_t e = cudaMalloc(&b.p, bytes);
    if (e != cudaSuccess) {
        snprintf(g_err, sizeof g_err, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
        return PINS_ERR_NOMEM;
    }
    b.bytes = bytes;
    ++b.gen;
    static long long n_alloc = 0;
    const long long idx = n_alloc++;
    static const long long plo = getenv("PINS_POISON_LO") ? atoll(getenv("PINS_POISON_LO")) : 0;
    static const long long phi_ = getenv("PINS_POISON_HI") ? atoll(getenv("PINS_POISON_HI")) : (1LL << 60);
    if (getenv("PINS_POISON_LIST") && idx >= plo && idx < phi_)
        fprintf(stderr, "alloc %lld: %zu bytes\n", idx, bytes);
    const char *pz = getenv("PINS_POISON");         // dev check: new buffers start as garbage
    if (pz && idx >= plo && idx < phi_)
    {
        cudaDeviceSynchronize();
        cudaMemset(b.p, atoi(pz) & 0xff, bytes);
        cudaDeviceSynchronize();
    }
    return PINS_OK;
}

template <class T>
T *ptr(DevBuf &b) { return reinterpret_cast<T *>(b.p); }

}  // namespace

struct SideBufs {
    DevBuf pa, pb, pj, psc, blk, blkoff, ticket, cnt, bcol, bval, jstar;
    // certified candidate lists of the Sinkhorn phase (pins_pass.cuh lse_sparse_kernel)
    DevBuf lcnt, lj, lD, lB, lqref, lqv, lqsv, ldqc, ldqs, lperm, lq;
    // absorbed kernel-matrix sweeps (lse_ksweep_kernel): sliced-ELL copy of the lists
    DevBuf lqd, ellj, ellK, ellL, ellrel, ellabs, elltot, lunit;
};

struct pins_workspace {
    DevBuf rowsum, gradf, colsum, gradg, rowcnt;
    DevBuf rowptr, colidx, val, colcnt, colptr, cursor, rowidx, valT;
    DevBuf cgvec, cgpart, cgst, st, ft, gt, eu, ev, bu, bv, dir, rhs, tab, fsave, gsave, uv;
    DevBuf tr_i, tr_d, tr_u8, tr_u64;   // tree-CG workspace (int / double / byte / u64 pools)
    DevBuf xprev, xsave;                // warm_start 2: previous solution, saved start
    // v2 dense passes
    SideBufs sb[2];
    DevBuf x32, y32, x64, y64, nx32, ny32, xh, yh, pinfo, ctl, gticket, pst, tol;
    DevBuf sk_gam[4], sk_gamD[4], sk_tref[4], sk_qref[4], skst;   // chunk-skip certificates: (LSE, SUM) x orientation
    const void *key_C = nullptr, *key_x = nullptr, *key_y = nullptr;
    long long key_m = -1, key_n = -1, key_ldc = -1;
    int key_kind = -1, key_d = -1;
    int cost_row = 0, cost_col = 0, dp = 4, skipk = 0;
    CUtensorMap tm_row, tm_col;        // dense C staged by TMA (PC_DENSE_*_T)
    int S[2] = {1, 1};
    long long pcap = 16;       // per (row, split) sparsify capacity
    long long lcap = 0;        // per (row, split) candidate-list capacity (0: not sized yet)
    DevBuf lctl;               // candidate-list control ints
    long long lstat[4] = {0, 0, 0, 0};   // dev statistics: record passes, sparse passes, overflows, fallbacks
    long long m = 0, n = 0, nnz = 0;
    int nsm = 0, dev = -1;
    bool tree_valid = false;
    long long tree_N = -1;
    int tree_last_its = 0, tree_backoff = 0;
    bool tree_newton = false;          // the stored factor is a Newton system's (not a certificate's)
    int tree_stale = 0;                // Newton systems solved since the factor was computed
    const int *tree_rstart = nullptr, *tree_ctr = nullptr;
    const double *tree_frec = nullptr;
    TreeArgs tree_last;                // arguments of the last tree build (certificate replay)
    // LP certificate (pins_cert.cuh): tree-dual scratch, c-transform partials, candidates
    DevBuf cz, cdd, cdf, ctc, cpart, cu0, cv0, cu1, cv1, cbu, cbv, crow;
    DevBuf ccomp, ccid, cinfo, cR, cdsh, cw;
    bool csr_ready = false, csc_ready = false;
    bool x0_enable = false;    // solve_core: warm-start the cluster tree-PCG from the previous direction
    bool dir_valid = false;    // ws->dir holds the previous Newton system's solution
    double *h = nullptr;   // pinned host scalars (64)
};

extern "C" void pins_default_params(pins_params *p) {
    p->K = 500;
    p->outer_rule = 0;
    p->outer_tol = 1e-4;
    p->T1 = 50000;
    p->sink_tol = 6.3e-4;
    p->T2 = 20;
    p->newton_tol = 1e-8;
    p->theta = 1e-4;
    p->cg_tol = 1e-6;
    p->cg_forcing = 0.5;
    p->cg_maxit = 1000;
    p->mu_rel = 1e-10;
    p->armijo_c = 1e-4;
    p->beta = 0.5;
    p->max_backtracks = 30;
    p->warm_start = 1;
}

extern "C" int pins_workspace_create(pins_workspace **out) {
    PINS_ARG(out != nullptr, "ws");
    pins_workspace *ws = new pins_workspace();
    memset(&ws->tm_row, 0, sizeof ws->tm_row);
    memset(&ws->tm_col, 0, sizeof ws->tm_col);
    PINS_CUDA(cudaGetDevice(&ws->dev));
    PINS_CUDA(cudaDeviceGetAttribute(&ws->nsm, cudaDevAttrMultiProcessorCount, ws->dev));
    PINS_CUDA(cudaMallocHost(&ws->h, 64 * sizeof(double)));
    // exp table 2^(j/64), hi + lo, from 80-bit long double
    ExpTable t;
    for (int j = 0; j < 64; ++j) {
        long double v = exp2l((long double)j / 64.0L);
        t.hi[j] = (double)v;
        t.lo[j] = (double)(v - (long double)t.hi[j]);
    }
    PINS_TRY(ensure(ws->tab, sizeof(ExpTable)));
    PINS_CUDA(cudaMemcpy(ws->tab.p, &t, sizeof t, cudaMemcpyHostToDevice));
    *out = ws;
    return PINS_OK;
}

extern "C" void pins_workspace_destroy(pins_workspace *ws) {
    if (!ws) return;
    if (ws->h) cudaFreeHost(ws->h);
    delete ws;   // every DevBuf member frees its device memory
}

namespace {

int check_problem(const pins_problem *pb) {
    PINS_ARG(pb != nullptr, "problem");
    PINS_ARG(pb->m >= 1 && pb->n >= 1, "m, n >= 1");
    PINS_ARG(pb->n < (1LL << 31) && pb->m < (1LL << 31), "m, n < 2^31");
    PINS_ARG(pb->a && pb->b, "a, b");
    PINS_ARG(pb->eta > 0.0 && std::isfinite(pb->eta), "eta > 0");
    PINS_ARG(pb->cost_scale > 0.0 && std::isfinite(pb->cost_scale), "cost_scale > 0");
    if (pb->cost_kind == PINS_COST_DENSE) {
        PINS_ARG(pb->C != nullptr && pb->ldc >= pb->n, "dense C / ldc");
    } else {
        PINS_ARG(pb->cost_kind == PINS_COST_SQEUCLID || pb->cost_kind == PINS_COST_L1, "cost_kind");
        PINS_ARG(pb->x && pb->y && pb->d >= 1 && pb->d <= 16, "points x, y, 1 <= d <= 16");
    }
    return PINS_OK;
}

CostDesc make_cd(const pins_problem *pb) {
    CostDesc cd;
    cd.kind = pb->cost_kind;
    cd.d = pb->d;
    cd.C = pb->C;
    cd.ldc = pb->ldc;
    cd.x = pb->x;
    cd.y = pb->y;
    return cd;
}

int dmax_for(int d) { return d <= 2 ? 2 : d <= 3 ? 3 : d <= 10 ? 10 : 16; }

int grid_1d(long long work, int nsm, int per_sm = 8) {
    long long g = (work + 255) / 256;
    if (g < 1) g = 1;
    return (int)std::min<long long>(g, (long long)nsm * per_sm);
}

int prepare(pins_workspace *ws, const pins_problem *pb) {
    const long long m = pb->m, n = pb->n;
    if (ws->m != m || ws->n != n) {
        ws->m = m;
        ws->n = n;
        ws->csr_ready = ws->csc_ready = false;
    }
    const long long N = m + n;
    PINS_TRY(ensure(ws->rowsum, sizeof(double) * m));
    PINS_TRY(ensure(ws->gradf, sizeof(double) * m));
    PINS_TRY(ensure(ws->colsum, sizeof(double) * n));
    PINS_TRY(ensure(ws->gradg, sizeof(double) * n));
    PINS_TRY(ensure(ws->st, sizeof(double) * 32));
    PINS_TRY(ensure(ws->ft, sizeof(double) * m));
    PINS_TRY(ensure(ws->gt, sizeof(double) * n));
    PINS_TRY(ensure(ws->eu, sizeof(double) * m));
    PINS_TRY(ensure(ws->ev, sizeof(double) * n));
    PINS_TRY(ensure(ws->dir, sizeof(double) * N));
    PINS_TRY(ensure(ws->rhs, sizeof(double) * N));
    PINS_TRY(ensure(ws->fsave, sizeof(double) * m));
    PINS_TRY(ensure(ws->gsave, sizeof(double) * n));
    PINS_TRY(ensure(ws->uv, sizeof(double) * N));
    return PINS_OK;
}

// extra reductions: st[8] = <a,f> + <b,g>, st[9] = max rowsum, st[10] = max colsum
__global__ void __launch_bounds__(1024) dots_kernel(long long m, long long n, const double *a,
                                                    const double *f, const double *b,
                                                    const double *g, const double *rowsum,
                                                    const double *colsum, double *st) {
    __shared__ double sh[32][3];
    double s = 0.0, mr = 0.0, mc = 0.0;
    for (long long i = threadIdx.x; i < m; i += 1024) {
        s = fma(a[i], f[i], s);
        mr = fmax(mr, rowsum[i]);
    }
    for (long long j = threadIdx.x; j < n; j += 1024) {
        s = fma(b[j], g[j], s);
        mc = fmax(mc, colsum[j]);
    }
    s = warp_sum(s);
    mr = warp_max(mr);
    mc = warp_max(mc);
    if ((threadIdx.x & 31) == 0) {
        sh[threadIdx.x >> 5][0] = s;
        sh[threadIdx.x >> 5][1] = mr;
        sh[threadIdx.x >> 5][2] = mc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0, a1 = 0.0, a2 = 0.0;
        for (int w = 0; w < 32; ++w) {
            t += sh[w][0];
            a1 = fmax(a1, sh[w][1]);
            a2 = fmax(a2, sh[w][2]);
        }
        st[8] = t;
        st[9] = a1;
        st[10] = a2;
    }
}

struct EvalOut {
    double gnorm, sumX, cost, dualP, nnz, maxz, maxcnt, em1, maxr, maxc, af;
};

// ===================================================================== v2
// Thread-per-row dense passes (pins_pass.cuh).
int dp_for(int d) { return d <= 4 ? 4 : d <= 12 ? 12 : 16; }

// Tensor maps of a dense C for the TMA-staged passes (pins_pass.cuh): the row
// orientation loads {16 columns x 128 rows} boxes with the 128-byte swizzle, the
// column orientation {128 columns x 32 rows} boxes.  Out-of-range elements of a
// box are zero-filled by the TMA unit (the passes mask them).
int make_dense_maps(pins_workspace *ws, const pins_problem *pb) {
    static PFN_cuTensorMapEncodeTiled encode = nullptr;
    if (!encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        PINS_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        PINS_ARG(fn != nullptr && q == cudaDriverEntryPointSuccess, "cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
    }
    const cuuint64_t dims[2] = {(cuuint64_t)pb->n, (cuuint64_t)pb->m};
    const cuuint64_t strides[1] = {(cuuint64_t)pb->ldc * sizeof(double)};
    const cuuint32_t es[2] = {1, 1};
    const cuuint32_t box_row[2] = {16, (cuuint32_t)kPT};
    const cuuint32_t box_col[2] = {(cuuint32_t)kPT, (cuuint32_t)kCC};
    CUresult r1 = encode(&ws->tm_row, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(pb->C), dims, strides,
                         box_row, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = encode(&ws->tm_col, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(pb->C), dims, strides,
                         box_col, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS) {
        snprintf(g_err, sizeof g_err, "cuTensorMapEncodeTiled failed (%d, %d)", (int)r1, (int)r2);
        return PINS_ERR_CUDA;
    }
    return PINS_OK;
}

// Forget the derived cost data of the previous problem.  Every public entry
// point that takes a pins_problem calls this first, so a workspace reused with
// a new problem -- even one whose arrays sit at the old addresses, or whose
// points were updated in place -- never sees stale coordinates, exactness
// decisions or chunk-skip certificates.  (pins_solve keeps its state across
// its own internal calls.)
void invalidate_problem(pins_workspace *ws) {
    ws->key_C = ws->key_x = ws->key_y = nullptr;
    ws->key_m = ws->key_n = ws->key_ldc = -1;
    ws->key_kind = ws->key_d = -1;
    ws->tree_valid = false;
    ws->tree_newton = false;
    ws->dir_valid = false;
    ws->tree_backoff = 0;
}

// (Re)build the derived cost data when the problem identity changes: padded
// fp32 / fp64 point copies, norms, the exact-fp32 decision, argmax seeds.
int prepare_pass(pins_workspace *ws, const pins_problem *pb, cudaStream_t st) {
    const long long m = pb->m, n = pb->n;
    const bool same = ws->key_C == pb->C && ws->key_x == pb->x && ws->key_y == pb->y && ws->key_m == m &&
                      ws->key_n == n && ws->key_kind == pb->cost_kind && ws->key_d == pb->d &&
                      ws->key_ldc == pb->ldc;
    for (int q = 0; q < 2; ++q) {
        const long long M = q == 0 ? m : n, N = q == 0 ? n : m;
        const int RB = (int)((M + kPT - 1) / kPT);
        // column splits: ~14 CTAs of 128 threads per SM per side (about 3 waves at the
        // half-sweep's 5 CTAs per SM: measured on c3, 4.19 s vs 4.44 s at 8), splits >= kCC columns
        static const double split_f = getenv("PINS_SPLIT_F") ? atof(getenv("PINS_SPLIT_F")) : 14.4;
        long long S = ((long long)(split_f * ws->nsm) + RB - 1) / RB;
        S = std::max(1LL, std::min(S, std::max(1LL, N / kCC)));
        ws->S[q] = (int)S;
        SideBufs &B = ws->sb[q];
        PINS_TRY(ensure(B.pa, sizeof(double) * S * M));
        PINS_TRY(ensure(B.pb, sizeof(double) * S * M));
        PINS_TRY(ensure(B.pj, sizeof(int) * S * M));
        PINS_TRY(ensure(B.psc, sizeof(double) * S * RB * 4));
        PINS_TRY(ensure(B.blk, sizeof(double) * RB * 8));
        PINS_TRY(ensure(B.blkoff, sizeof(long long) * (RB + 1)));
        PINS_TRY(ensure(B.cnt, sizeof(int) * S * M));
        if (B.ticket.bytes < sizeof(unsigned) * RB) {
            PINS_TRY(ensure(B.ticket, sizeof(unsigned) * RB));
            PINS_CUDA(cudaMemsetAsync(B.ticket.p, 0, B.ticket.bytes, st));
        }
        if (B.jstar.bytes < sizeof(int) * M || !same) {
            PINS_TRY(ensure(B.jstar, sizeof(int) * M));
            PINS_CUDA(cudaMemsetAsync(B.jstar.p, 0xff, sizeof(int) * M, st));
        }
    }
    if (ws->gticket.bytes == 0) {
        PINS_TRY(ensure(ws->gticket, 64));
        PINS_CUDA(cudaMemsetAsync(ws->gticket.p, 0, 64, st));
    }
    PINS_TRY(ensure(ws->pst, sizeof(double) * 32));
    PINS_TRY(ensure(ws->ctl, sizeof(int) * 8));
    PINS_TRY(ensure(ws->tol, sizeof(double) * 4));
    PINS_TRY(ensure(ws->bu, sizeof(double) * m));
    PINS_TRY(ensure(ws->bv, sizeof(double) * n));
    if (same) return PINS_OK;
    if (pb->cost_kind == PINS_COST_DENSE) {
        ws->cost_row = PC_DENSE_ROW;
        ws->cost_col = PC_DENSE_COL;
        ws->skipk = 0;
        ws->dp = 4;
        // TMA staging needs a 16-byte aligned base and row pitch (else the thread-staged path)
        const bool aligned = (reinterpret_cast<uintptr_t>(pb->C) & 15) == 0 && (pb->ldc % 2) == 0;
        if (aligned && getenv("PINS_NO_TMA") == nullptr) {
            PINS_TRY(make_dense_maps(ws, pb));
            ws->cost_row = PC_DENSE_ROW_T;
            ws->cost_col = PC_DENSE_COL_T;
        }
    } else {
        const int dp = dp_for(pb->d);
        ws->dp = dp;
        PINS_TRY(ensure(ws->x32, sizeof(float) * m * dp));
        PINS_TRY(ensure(ws->y32, sizeof(float) * n * dp));
        PINS_TRY(ensure(ws->x64, sizeof(double) * m * dp));
        PINS_TRY(ensure(ws->y64, sizeof(double) * n * dp));
        PINS_TRY(ensure(ws->nx32, sizeof(float) * m));
        PINS_TRY(ensure(ws->ny32, sizeof(float) * n));
        PINS_TRY(ensure(ws->pinfo, sizeof(unsigned long long) * 8));
        PINS_CUDA(cudaMemsetAsync(ws->pinfo.p, 0, sizeof(unsigned long long) * 8, st));
        unsigned long long *info = ptr<unsigned long long>(ws->pinfo);
        LAUNCH(PINS_PROF_VEC, st, prep_points_kernel<<<grid_1d(m, ws->nsm), 256, 0, st>>>(
            m, pb->d, dp, pb->x, ptr<float>(ws->x32), ptr<double>(ws->x64), ptr<float>(ws->nx32), info));
        LAUNCH(PINS_PROF_VEC, st, prep_points_kernel<<<grid_1d(n, ws->nsm), 256, 0, st>>>(
            n, pb->d, dp, pb->y, ptr<float>(ws->y32), ptr<double>(ws->y64), ptr<float>(ws->ny32), info + 4));
        PINS_CUDA(cudaGetLastError());
        unsigned long long hi[8];
        PINS_CUDA(cudaMemcpyAsync(hi, info, sizeof hi, cudaMemcpyDeviceToHost, st));
        PINS_CUDA(cudaStreamSynchronize(st));
        double ax, nxm, ay, nym;
        memcpy(&ax, &hi[0], 8); memcpy(&nxm, &hi[1], 8); memcpy(&ay, &hi[4], 8); memcpy(&nym, &hi[5], 8);
        const bool integral = hi[2] == 0 && hi[6] == 0;
        const double two24 = 16777216.0;
        bool exact32;
        if (pb->cost_kind == PINS_COST_SQEUCLID) {
            const double bound = (std::sqrt(nxm) + std::sqrt(nym)) * (std::sqrt(nxm) + std::sqrt(nym));
            exact32 = integral && bound < two24 && ax < two24 && ay < two24;
            ws->cost_row = ws->cost_col = exact32 ? PC_SQ32 : PC_SQ64;
            // tensor cores: fp16 operands exact for integers |x| <= 2048, d <= 16
            if (exact32 && std::max(ax, ay) <= 2048.0 && pb->d <= 16 && getenv("PINS_NO_TC") == nullptr) {
                PINS_TRY(ensure(ws->xh, sizeof(__half) * m * 16));
                PINS_TRY(ensure(ws->yh, sizeof(__half) * n * 16));
                LAUNCH(PINS_PROF_VEC, st, to_half16_kernel<<<grid_1d(m * 16, ws->nsm), 256, 0, st>>>(
                    m, dp, ptr<float>(ws->x32), ptr<__half>(ws->xh)));
                LAUNCH(PINS_PROF_VEC, st, to_half16_kernel<<<grid_1d(n * 16, ws->nsm), 256, 0, st>>>(
                    n, dp, ptr<float>(ws->y32), ptr<__half>(ws->yh)));
                PINS_CUDA(cudaGetLastError());
                ws->cost_row = ws->cost_col = PC_SQTC;
            }
        } else {
            exact32 = integral && 2.0 * pb->d * std::max(ax, ay) < two24;
            ws->cost_row = ws->cost_col = exact32 ? PC_L132 : PC_L164;
        }
        // chunk skipping needs exact fp32 distances (integer points, R10)
        ws->skipk = exact32 && getenv("PINS_NO_TILESKIP") == nullptr ? 1 : 0;
    }
    if (ws->skipk) {
        for (int q = 0; q < 4; ++q) {
            const int o = q & 1;
            const long long M = o == 0 ? m : n, N = o == 0 ? n : m;
            const long long RB = (M + kPT - 1) / kPT, S = ws->S[o];
            const long long cps = ((N + S - 1) / S + kCC - 1) / kCC + 1;
            PINS_TRY(ensure(ws->sk_gam[q], sizeof(float) * RB * S * cps * 4));
            PINS_TRY(ensure(ws->sk_gamD[q], sizeof(float) * RB * S * cps * 4));
            PINS_TRY(ensure(ws->sk_tref[q], sizeof(float) * M));
            PINS_TRY(ensure(ws->sk_qref[q], sizeof(float) * N));
        }
        PINS_TRY(ensure(ws->skst, sizeof(int) * 64));
        PINS_CUDA(cudaMemsetAsync(ws->skst.p, 0xff, sizeof(int) * 64, st));   // age -1: record first
        for (int q = 0; q < 4; ++q)
            PINS_CUDA(cudaMemsetAsync(ptr<int>(ws->skst) + 16 * q + 6, 0, sizeof(int) * 4, st));
    }
    ws->key_C = pb->C; ws->key_x = pb->x; ws->key_y = pb->y; ws->key_m = m; ws->key_n = n;
    ws->key_kind = pb->cost_kind; ws->key_d = pb->d; ws->key_ldc = pb->ldc;
    return PINS_OK;
}

// chunk-skip state q = 2 * (0 LSE, 1 SUM) + orientation
void set_skip(pins_workspace *ws, PassSide &P, int q) {
    if (!P.skipk) return;
    P.cps = (int)(((P.N + P.S - 1) / P.S + kCC - 1) / kCC + 1);
    P.gam = ptr<float>(ws->sk_gam[q]);
    P.gamD = ptr<float>(ws->sk_gamD[q]);
    P.tref = ptr<float>(ws->sk_tref[q]);
    P.qref = ptr<float>(ws->sk_qref[q]);
    P.skst = ptr<int>(ws->skst) + 16 * q;
}

// Fill the pass description of one orientation (0: rows of X, 1: columns).
void fill_side(pins_workspace *ws, const pins_problem *pb, int o, const double *f, const double *phi,
               const double *g, const double *psi, PassSide &P) {
    memset(&P, 0, sizeof P);
    const bool row = o == 0;
    P.M = row ? pb->m : pb->n;
    P.N = row ? pb->n : pb->m;
    P.S = ws->S[o];
    P.RB = (int)((P.M + kPT - 1) / kPT);
    P.dp = ws->dp;
    P.C = pb->C;
    P.ldc = pb->ldc;
    P.xr32 = ptr<float>(row ? ws->x32 : ws->y32);
    P.yc32 = ptr<float>(row ? ws->y32 : ws->x32);
    P.nxr = ptr<float>(row ? ws->nx32 : ws->ny32);
    P.nyc = ptr<float>(row ? ws->ny32 : ws->nx32);
    P.xr64 = ptr<double>(row ? ws->x64 : ws->y64);
    P.yc64 = ptr<double>(row ? ws->y64 : ws->x64);
    P.xrh = ptr<__half>(row ? ws->xh : ws->yh);
    P.ych = ptr<__half>(row ? ws->yh : ws->xh);
    P.skipk = pb->cost_kind == PINS_COST_DENSE ? 0 : ws->skipk;
    set_skip(ws, P, 2 + o);      // sum passes; half_sweep switches to the LSE state o
    P.fr = row ? f : g;
    P.phir = row ? phi : psi;
    P.gc = row ? g : f;
    P.psic = row ? psi : phi;
    P.m1_row = row ? 1 : 0;
    P.ar = row ? pb->a : pb->b;
    SideBufs &B = ws->sb[o];
    P.jstar = ptr<int>(B.jstar);
    P.pa = ptr<double>(B.pa);
    P.pb = ptr<double>(B.pb);
    P.pj = ptr<int>(B.pj);
    P.psc = ptr<double>(B.psc);
    P.blk = ptr<double>(B.blk);
    P.blkoff = ptr<long long>(B.blkoff);
    P.ticket = ptr<unsigned>(B.ticket);
    P.cnt = ptr<int>(B.cnt);
    P.bcol = ptr<int>(B.bcol);
    P.bval = ptr<double>(B.bval);
    P.cap = ws->pcap;
    P.sum = ptr<double>(row ? ws->rowsum : ws->colsum);
    P.grad = ptr<double>(row ? ws->gradf : ws->gradg);
}

#define PINS_DP_DISPATCH(DPV, ...)          \
    do {                                    \
        if ((DPV) == 4) {                   \
            constexpr int DP = 4;           \
            __VA_ARGS__;                    \
        } else if ((DPV) == 12) {           \
            constexpr int DP = 12;          \
            __VA_ARGS__;                    \
        } else {                            \
            constexpr int DP = 16;          \
            __VA_ARGS__;                    \
        }                                   \
    } while (0)

// dynamic shared memory of a pass kernel instantiation: the TMA ring for dense
// costs staged by TMA (attribute set once per instantiation), else none
template <class K>
size_t pass_smem(K kern, size_t bytes) {
    if (!bytes) return 0;
    static std::vector<const void *> done;          // per kernel (instantiations share a type)
    const void *key = reinterpret_cast<const void *>(kern);
    if (std::find(done.begin(), done.end(), key) == done.end()) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        done.push_back(key);
    }
    return bytes;
}
#define LSE_LAUNCH(CLS, C_, DP_)                                                                            \
    LAUNCH(CLS, st, lse_pass_kernel<C_, DP_><<<grid, kPT,                                                     \
           pass_smem(lse_pass_kernel<C_, DP_>, kTma<C_> ? kTmaSmem : 0), st>>>(A, tm))
#define SUM_LAUNCH(C0_, C1_, DP_)                                                                            \
    LAUNCH(PINS_PROF_EVAL, st, sum_pass_kernel<C0_, C1_, DP_><<<grid, kPT,                                    \
           pass_smem(sum_pass_kernel<C0_, C1_, DP_>, kTma<C0_> ? kTmaSmem : 0), st>>>(A, tm0, tm1))

// pcls >= 0: the profiler class of this launch (list modes book their record passes, most
// of which exit at once, under PINS_PROF_SWEEP_AUX)
cudaError_t launch_lse(int cost, int dp, int grid, cudaStream_t st, const PassArgs &A, const CUtensorMap &tm,
                       int pcls = -1) {
    const int crow = pcls >= 0 ? pcls : PINS_PROF_SWEEP_ROW, ccol = pcls >= 0 ? pcls : PINS_PROF_SWEEP_COL;
    switch (cost) {
        case PC_DENSE_ROW: LSE_LAUNCH(crow, PC_DENSE_ROW, 4); break;
        case PC_DENSE_COL: LSE_LAUNCH(ccol, PC_DENSE_COL, 4); break;
        case PC_DENSE_ROW_T: LSE_LAUNCH(crow, PC_DENSE_ROW_T, 4); break;
        case PC_DENSE_COL_T: LSE_LAUNCH(ccol, PC_DENSE_COL_T, 4); break;
        case PC_SQ32: PINS_DP_DISPATCH(dp, LSE_LAUNCH(crow, PC_SQ32, DP)); break;
        case PC_L132: PINS_DP_DISPATCH(dp, LSE_LAUNCH(crow, PC_L132, DP)); break;
        case PC_SQ64: PINS_DP_DISPATCH(dp, LSE_LAUNCH(crow, PC_SQ64, DP)); break;
        case PC_SQTC: PINS_DP_DISPATCH(dp, LSE_LAUNCH(crow, PC_SQTC, DP)); break;
        default: PINS_DP_DISPATCH(dp, LSE_LAUNCH(crow, PC_L164, DP)); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_sum(int cost, int dp, int grid, cudaStream_t st, const PassArgs &A, const CUtensorMap &tm0,
                       const CUtensorMap &tm1) {
    switch (cost) {
        case PC_DENSE_ROW: SUM_LAUNCH(PC_DENSE_ROW, PC_DENSE_COL, 4); break;
        case PC_DENSE_ROW_T: SUM_LAUNCH(PC_DENSE_ROW_T, PC_DENSE_COL_T, 4); break;
        case PC_SQ32: PINS_DP_DISPATCH(dp, SUM_LAUNCH(PC_SQ32, PC_SQ32, DP)); break;
        case PC_L132: PINS_DP_DISPATCH(dp, SUM_LAUNCH(PC_L132, PC_L132, DP)); break;
        case PC_SQ64: PINS_DP_DISPATCH(dp, SUM_LAUNCH(PC_SQ64, PC_SQ64, DP)); break;
        case PC_SQTC: PINS_DP_DISPATCH(dp, SUM_LAUNCH(PC_SQTC, PC_SQTC, DP)); break;
        default: PINS_DP_DISPATCH(dp, SUM_LAUNCH(PC_L164, PC_L164, DP)); break;
    }
    return cudaGetLastError();
}

void base_args(pins_workspace *ws, const pins_problem *pb, double s, PassArgs &A) {
    memset(&A, 0, sizeof A);
    A.eta = pb->eta;
    A.inv_eta = 1.0 / pb->eta;
    A.w = s * pb->cost_scale / pb->eta;
    A.tab = ptr<ExpTable>(ws->tab);
    A.gticket = ptr<unsigned>(ws->gticket);
    A.st = ptr<double>(ws->pst);
    A.ctl = ptr<int>(ws->ctl);
    A.count_surv = g_prof.on ? 1 : 0;
}

// One Sinkhorn half-sweep: o = 0 updates f (Alg. 2 line 5), o = 1 updates g (line 6).
// the sparse path of a half-sweep: list walk, dense fallback of failed units, merge
cudaError_t launch_lse_sparse(int cost, int dp, int grid, int gfb, int gmerge, size_t smem, cudaStream_t st,
                              const PassArgs &A) {
#define LSP_LAUNCH(C_, DP_)                                                                     \
    do {                                                                                        \
        if (smem)                                                                               \
            LAUNCH(PINS_PROF_SWEEP_ROW, st, lse_sparse_kernel<C_, DP_, true><<<grid, kPT,       \
                   pass_smem(lse_sparse_kernel<C_, DP_, true>, 64 * 1024 + 16) ? smem : 0, st>>>(A)); \
        else                                                                                    \
            LAUNCH(PINS_PROF_SWEEP_ROW, st, lse_sparse_kernel<C_, DP_, false><<<grid, kPT, 0, st>>>(A)); \
        LAUNCH(PINS_PROF_SWEEP_ROW, st, lse_fallback_kernel<C_, DP_><<<gfb, kPT, 0, st>>>(A));  \
        LAUNCH(PINS_PROF_SWEEP_ROW, st, lse_merge_kernel<<<gmerge, kPT, 0, st>>>(A));           \
    } while (0)
    switch (cost) {
        case PC_DENSE_ROW: case PC_DENSE_ROW_T: LSP_LAUNCH(PC_DENSE_ROW_T, 4); break;
        case PC_DENSE_COL: case PC_DENSE_COL_T: LSP_LAUNCH(PC_DENSE_COL_T, 4); break;
        case PC_SQ32: PINS_DP_DISPATCH(dp, LSP_LAUNCH(PC_SQ32, DP)); break;
        case PC_L132: PINS_DP_DISPATCH(dp, LSP_LAUNCH(PC_L132, DP)); break;
        case PC_SQ64: PINS_DP_DISPATCH(dp, LSP_LAUNCH(PC_SQ64, DP)); break;
        case PC_SQTC: PINS_DP_DISPATCH(dp, LSP_LAUNCH(PC_SQTC, DP)); break;
        default: PINS_DP_DISPATCH(dp, LSP_LAUNCH(PC_L164, DP)); break;
    }
#undef LSP_LAUNCH
    return cudaGetLastError();
}

constexpr size_t kKSmemMax = 220 * 1024;     // lse_ksweep_kernel: the ring + the widest split's u_j (8 B per column)

// the absorbed kernel-matrix path of a half-sweep: ELL build (only right after a record),
// ELL walk, dense fallback of failed units, merge
cudaError_t launch_lse_k(int cost, int dp, int grid, int gfb, int gmerge, size_t smem, cudaStream_t st,
                         const PassArgs &A, bool build) {
#define LSK_LAUNCH(C_, DP_)                                                                     \
    do {                                                                                        \
        if (build)                                                                              \
            LAUNCH(PINS_PROF_SWEEP_AUX, st, lse_kbuild_kernel<C_, DP_><<<grid, kPT, 0, st>>>(A)); \
        LAUNCH(PINS_PROF_KSWEEP, st, lse_ksweep_kernel<<<grid, kPT,                             \
               (pass_smem(lse_ksweep_kernel, kKSmemMax), smem), st>>>(A));                      \
        LAUNCH(PINS_PROF_SWEEP_AUX, st, lse_fallback_k_kernel<C_, DP_><<<gfb, kPT, 0, st>>>(A)); \
        LAUNCH(PINS_PROF_SWEEP_AUX, st, lse_merge_kernel<<<gmerge, kPT, 0, st>>>(A));           \
    } while (0)
    switch (cost) {
        case PC_DENSE_ROW: case PC_DENSE_ROW_T: LSK_LAUNCH(PC_DENSE_ROW_T, 4); break;
        case PC_DENSE_COL: case PC_DENSE_COL_T: LSK_LAUNCH(PC_DENSE_COL_T, 4); break;
        case PC_SQ32: PINS_DP_DISPATCH(dp, LSK_LAUNCH(PC_SQ32, DP)); break;
        case PC_L132: PINS_DP_DISPATCH(dp, LSK_LAUNCH(PC_L132, DP)); break;
        case PC_SQ64: PINS_DP_DISPATCH(dp, LSK_LAUNCH(PC_SQ64, DP)); break;
        case PC_SQTC: PINS_DP_DISPATCH(dp, LSK_LAUNCH(PC_SQTC, DP)); break;
        default: PINS_DP_DISPATCH(dp, LSK_LAUNCH(PC_L164, DP)); break;
    }
#undef LSK_LAUNCH
    return cudaGetLastError();
}

// candidate-list margin below the LSE cut (units of the exponent): wider lists, fewer
// record passes
double list_margin() {
    const char *e = getenv("PINS_LIST_MARGIN");
    return e ? atof(e) : 4.0;
}

// candidate-list buffers of both sides at capacity ws->lcap per (row, split)
int ensure_lists(pins_workspace *ws, const pins_problem *pb, cudaStream_t st, bool kmode = false) {
    for (int o = 0; o < 2; ++o) {
        const long long M = o == 0 ? pb->m : pb->n, N = o == 0 ? pb->n : pb->m, S = ws->S[o];
        const int cost = o == 0 ? ws->cost_row : ws->cost_col;
        const size_t dsz = (cost == PC_SQTC || cost == PC_SQ32 || cost == PC_L132) ? 4 : 8;
        SideBufs &B = ws->sb[o];
        PINS_TRY(ensure(B.lcnt, sizeof(int) * S * M));
        PINS_TRY(ensure(B.lj, sizeof(int) * S * ws->lcap * M));
        PINS_TRY(ensure(B.lD, dsz * S * ws->lcap * M));
        PINS_TRY(ensure(B.lB, sizeof(float) * M));
        PINS_TRY(ensure(B.lqref, sizeof(float) * N));
        PINS_TRY(ensure(B.lqv, sizeof(double) * N));
        PINS_TRY(ensure(B.lqsv, sizeof(float) * N));
        PINS_TRY(ensure(B.ldqc, sizeof(float) * (N / kCC + 2)));
        PINS_TRY(ensure(B.ldqs, sizeof(float) * S));
        PINS_TRY(ensure(B.lperm, sizeof(int) * S * M));
        PINS_TRY(ensure(B.lq, sizeof(int) * S * M));
        if (kmode) {
            const long long Mpad = (M + 31) / 32 * 32;
            PINS_TRY(ensure(B.lqd, sizeof(double) * N));
            PINS_TRY(ensure(B.ellj, sizeof(int) * S * ws->lcap * Mpad));
            PINS_TRY(ensure(B.ellK, sizeof(double) * S * ws->lcap * Mpad));
            PINS_TRY(ensure(B.ellL, sizeof(int) * S * (Mpad / 32)));
            PINS_TRY(ensure(B.ellrel, sizeof(int) * S * (Mpad / 32)));
            PINS_TRY(ensure(B.ellabs, sizeof(int) * S * (Mpad / 32)));
            PINS_TRY(ensure(B.elltot, sizeof(int) * S));
            PINS_TRY(ensure(B.lunit, 32 * S * Mpad));
        }
    }
    PINS_TRY(ensure(ws->lctl, sizeof(int) * 16));
    (void)st;
    return PINS_OK;
}

// One Sinkhorn half-sweep: o = 0 updates f (Alg. 2 line 5), o = 1 updates g (line 6).
// lmode 0: the dense pass alone; 1: the dense pass if the side's candidate lists must
// be recorded (it records them), then the sparse pass over the lists otherwise (lt:
// this half-sweep's launch index).
int half_sweep(pins_workspace *ws, const pins_problem *pb, int o, const double *phi, const double *psi,
               double s, double *f, double *g, bool check_done, bool test_tol, cudaStream_t st,
               int lmode = 0, int lt = 0, bool rec_now = true) {
    // rec_now (mode 2): queue the record pass, sort and ELL build of this half-sweep (the host
    // saw the side's re-record request at its last synchronisation); otherwise only the ELL
    // walk, the fallback scan and the merge are launched
    PassArgs A;
    base_args(ws, pb, s, A);
    fill_side(ws, pb, o, f, phi, g, psi, A.side[0]);
    set_skip(ws, A.side[0], o);
    A.side[0].fout = o == 0 ? f : g;
    A.side[0].fsave = o == 0 ? ptr<double>(ws->fsave) : nullptr;
    A.nsides = 1;
    A.G0 = A.side[0].S * A.side[0].RB;
    A.check_done = check_done ? 1 : 0;
    A.count_sweep = o == 1 ? 1 : 0;
    A.test_tol = test_tol ? 1 : 0;
    A.sink_tol = ptr<double>(ws->tol);
    const int cost = o == 0 ? ws->cost_row : ws->cost_col;
    if (lmode) {
        PassSide &P = A.side[0];
        SideBufs &B = ws->sb[o], &Bo = ws->sb[1 - o];
        P.lori = o;
        P.lcap = (int)ws->lcap;
        P.lcnt = ptr<int>(B.lcnt);
        P.lj = ptr<int>(B.lj);
        P.lD = B.lD.p;
        P.lB = ptr<float>(B.lB);
        P.lqref = ptr<float>(B.lqref);
        P.lqv = ptr<double>(B.lqv);
        P.lqsv = ptr<float>(B.lqsv);
        P.ldqs = ptr<float>(B.ldqs);
        P.lperm = ptr<int>(B.lperm);
        P.lq = ptr<int>(B.lq);
        P.oqv = ptr<double>(Bo.lqv);
        P.oqsv = ptr<float>(Bo.lqsv);
        P.oqref = ptr<float>(Bo.lqref);
        P.odqc = ptr<float>(Bo.ldqc);
        P.odqs = ptr<float>(Bo.ldqs);
        P.oS = ws->S[1 - o];
        P.lctl = ptr<int>(ws->lctl);
        A.lt = lt;
        A.lnosort = getenv("PINS_KNOSORT") != nullptr ? 1 : 0;
        A.lmargin = list_margin();
        if (lmode == 2) {
            P.lqd = ptr<double>(B.lqd);
            P.ellj = ptr<int>(B.ellj);
            P.ellK = ptr<double>(B.ellK);
            P.ellL = ptr<int>(B.ellL);
            P.ellrel = ptr<int>(B.ellrel);
            P.ellabs = ptr<int>(B.ellabs);
            P.elltot = ptr<int>(B.elltot);
            P.lunit = B.lunit.p;
            P.Mpad = (P.M + 31) / 32 * 32;
        }
        if (lmode != 2 || rec_now) {
            P.lrec = 1;
            PINS_CUDA(launch_lse(cost, ws->dp, A.G0, st, A, o == 0 ? ws->tm_row : ws->tm_col,
                                 lmode == 2 ? PINS_PROF_SWEEP_AUX : -1));
            P.lrec = 0;
            LAUNCH(lmode == 2 ? PINS_PROF_SWEEP_AUX : PINS_PROF_SWEEP_ROW, st,
                   lse_sort_kernel<<<P.S, 1024, 0, st>>>(A));
        }
        // the widest split's column values (q fp64 + qs fp32) staged per CTA when they fit
        const long long nch = (P.N + kCC - 1) / kCC, wmax = kCC * ((nch + P.S - 1) / P.S);
        const size_t stage = (size_t)wmax * 12 + 16;
        if (lmode == 2) {
            PINS_CUDA(launch_lse_k(cost, ws->dp, (int)(P.S * ((P.M + kPT - 1) / kPT)), 4 * ws->nsm, P.RB,
                                   (size_t)wmax * 8 + 16 + kKRing, st, A, rec_now));
            return PINS_OK;
        }
        P.lstage = stage <= 64 * 1024 ? 1 : 0;
        PINS_CUDA(launch_lse_sparse(cost, ws->dp, (int)(P.S * ((P.M + kPT - 1) / kPT)), 4 * ws->nsm, P.RB,
                                    P.lstage ? stage : 0, st, A));
        return PINS_OK;
    }
    PINS_CUDA(launch_lse(cost, ws->dp, A.G0, st, A, o == 0 ? ws->tm_row : ws->tm_col));
    return PINS_OK;
}

int do_sweep(pins_workspace *ws, const pins_problem *pb, const double *phi, const double *psi,
             double s, double *f, double *g, cudaStream_t st) {
    PINS_TRY(prepare_pass(ws, pb, st));
    PINS_TRY(ensure(ws->fsave, sizeof(double) * std::max(pb->m, pb->n)));
    PINS_TRY(half_sweep(ws, pb, 0, phi, psi, s, f, g, false, false, st));
    PINS_TRY(half_sweep(ws, pb, 1, phi, psi, s, f, g, false, false, st));
    return PINS_OK;
}

// Sinkhorn phase of Alg. 2 (lines 4-8) on the device: sweeps are queued in
// batches without host round trips; every row half-sweep after the first
// also computes the residual of the iterate it starts from and, when that is
// <= sink_tol, flags the phase done and rolls its own update back (so the
// phase stops at exactly the first iterate with residual <= sink_tol, as the
// oracle does); queued kernels see the flag and exit.  res0 is the full
// residual of the starting point (the caller's evaluation).  Returns sweeps.
int sinkhorn_phase(pins_workspace *ws, const pins_problem *pb, const pins_params *prm, const double *phi,
                   const double *psi, double s, double *f, double *g, double res0, int *sweeps_out,
                   cudaStream_t st) {
    *sweeps_out = 0;
    if (res0 <= prm->sink_tol || prm->T1 <= 0) return PINS_OK;
    PINS_TRY(prepare_pass(ws, pb, st));
    PINS_TRY(ensure(ws->fsave, sizeof(double) * std::max(pb->m, pb->n)));
    double tolv = prm->sink_tol;
    PINS_CUDA(cudaMemcpyAsync(ws->tol.p, &tolv, sizeof(double), cudaMemcpyHostToDevice, st));
    PINS_CUDA(cudaMemsetAsync(ws->ctl.p, 0, sizeof(int) * 8, st));
    // Candidate lists of the phase.  Mode 1 (PINS_SPARSE_SWEEP, opt-in): the certified list
    // walk, bit-identical to the dense sweeps.  Mode 2 (default; PINS_KSWEEP=0 switches it
    // off): absorbed kernel-matrix sweeps (lse_ksweep_kernel), engaged once the phase has
    // run kstart dense sweeps, so the short phases of the later EPPA iterations never pay
    // for a record.  Lists are recorded by the first sweep in a list mode and again
    // whenever too many certificates fail or a list overflows.
    const bool walk = getenv("PINS_SPARSE_SWEEP") != nullptr && prm->T1 > 1;
    const int kstart = getenv("PINS_KSWEEP_START") ? atoi(getenv("PINS_KSWEEP_START")) : 7;
    bool kavail = !walk && prm->T1 > 1 && !(getenv("PINS_KSWEEP") && getenv("PINS_KSWEEP")[0] == '0');
    for (int o = 0; o < 2 && kavail; ++o) {          // the widest split's u_j must fit in shared memory
        const long long N = o == 0 ? pb->n : pb->m, nch = (N + kCC - 1) / kCC;
        const long long wmax = kCC * ((nch + ws->S[o] - 1) / ws->S[o]);
        if ((size_t)wmax * 8 + 16 + kKRing > kKSmemMax) kavail = false;
    }
    int lmode = 0;
    // device bytes of both sides' lists (and ELL copies) at capacity cap per (row, split); the
    // capacity is a worst case -- the ELL tiles are packed, most of it is never touched -- but
    // it is allocated, so list modes are declined when it would not fit comfortably
    auto list_bytes = [&](long long cap, bool kmode) -> double {
        double tot = 0.0;
        for (int o = 0; o < 2; ++o) {
            const double M = (double)(o == 0 ? pb->m : pb->n), S = (double)ws->S[o];
            tot += S * M * (double)cap * (kmode ? 12.0 + 12.0 : 12.0);
        }
        return tot;
    };
    auto list_budget = [&]() -> double {
        size_t fr = 0, tt = 0;
        if (cudaMemGetInfo(&fr, &tt) != cudaSuccess) return 0.0;
        double have = 0.0;      // what the workspace already holds of these buffers is reusable
        for (int o = 0; o < 2; ++o)
            have += (double)(ws->sb[o].lj.bytes + ws->sb[o].lD.bytes + ws->sb[o].ellj.bytes + ws->sb[o].ellK.bytes);
        const double cap = getenv("PINS_LIST_BUDGET") ? atof(getenv("PINS_LIST_BUDGET")) : 32e9;   // bytes
        return std::min(cap, 0.5 * ((double)fr + have));
    };
    auto lists_begin = [&](int mode) -> int {
        if (ws->lcap == 0) {
            // a unit cannot list more than its split's columns: start there (capped), so the
            // usual instance never regrows
            long long wmx = 0;
            for (int o = 0; o < 2; ++o) {
                const long long N = o == 0 ? pb->n : pb->m, nch = (N + kCC - 1) / kCC;
                wmx = std::max(wmx, kCC * ((nch + ws->S[o] - 1) / ws->S[o]));
            }
            ws->lcap = getenv("PINS_LIST_CAP") ? std::max(1LL, atoll(getenv("PINS_LIST_CAP")))
                                               : std::max(64LL, std::min(wmx, 512LL));
        }
        ws->lcap = (ws->lcap + 15) / 16 * 16;     // lists padded to whole batches (8 walk, 16 ELL)
        if (mode == 2 && list_bytes(ws->lcap, true) > list_budget()) {
            kavail = false;                        // too large for this device: dense sweeps
            return PINS_OK;
        }
        PINS_TRY(ensure_lists(ws, pb, st, mode == 2));
        const int init[16] = {1, 1, -1, -1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        PINS_CUDA(cudaMemcpyAsync(ws->lctl.p, init, sizeof init, cudaMemcpyHostToDevice, st));
        lmode = mode;
        return PINS_OK;
    };
    if (walk) PINS_TRY(lists_begin(1));
    int done = 0, batch = 1, queued = 0, lt = 0;
    int *hc = reinterpret_cast<int *>(ws->h + 40);
    // Mode 2 is driven in short batches (8 sweeps).  The device raises a side's re-record
    // request when more than 2 % of its units fail their certificate; the host reads the
    // requests at every synchronisation and queues the record pass, the sort and the ELL build
    // only in the first sweep of the next batch (failed units are scanned densely meanwhile),
    // so an ordinary half-sweep is three launches: ELL walk, fallback scan, merge.
    // Churn control: while the potentials still move fast (the first sweeps of a cold start)
    // certificates fail within a sweep or two of a record.  A batch in which more than 1/8 of
    // the unit passes fell back sends the phase to dense sweeps for `cool` sweeps (doubling).
    int cool = 0, cool_len = 32;
    long long fb_prev = 0;
    bool need[2] = {true, true};
    const long long units = (long long)ws->S[0] * pb->m + (long long)ws->S[1] * pb->n;
    while (!done && queued < prm->T1) {
        if (kavail && lmode == 0 && queued >= kstart && cool <= 0) {
            PINS_TRY(lists_begin(2));                // (declines when the lists would not fit)
            fb_prev = 0;
            need[0] = need[1] = true;
        }
        const int nb = std::min(lmode == 2 ? std::min(batch, 8) : batch, prm->T1 - queued);
        for (int q = 0; q < nb; ++q) {
            const bool first = (queued + q) == 0;
            PINS_TRY(half_sweep(ws, pb, 0, phi, psi, s, f, g, true, !first, st, lmode, lt++, q == 0 && need[0]));
            PINS_TRY(half_sweep(ws, pb, 1, phi, psi, s, f, g, true, false, st, lmode, lt++, q == 0 && need[1]));
        }
        queued += nb;
        PINS_CUDA(cudaMemcpyAsync(hc, ws->ctl.p, sizeof(int) * 4, cudaMemcpyDeviceToHost, st));
        if (lmode) PINS_CUDA(cudaMemcpyAsync(hc + 4, ws->lctl.p, sizeof(int) * 16, cudaMemcpyDeviceToHost, st));
        PINS_CUDA(cudaStreamSynchronize(st));
        done = hc[0];
        *sweeps_out = hc[1];
        if (done && hc[2]) {   // roll back the f update of the half-sweep that found convergence
            PINS_CUDA(cudaMemcpyAsync(f, ws->fsave.p, sizeof(double) * pb->m, cudaMemcpyDeviceToDevice, st));
        }
        batch = std::min(batch * 2, 64);
        if (lmode == 0 && cool > 0) cool -= nb;
        if (lmode == 2) {
            need[0] = hc[4 + 0] != 0;
            need[1] = hc[4 + 1] != 0;
        }
        if (lmode == 2 && !done && hc[4 + 4] == 0) {
            const long long fb = (long long)hc[4 + 6] + hc[4 + 7];
            const long long dfb = fb - fb_prev;
            fb_prev = fb;
            if (dfb * 8 > units * nb && !getenv("PINS_KSWEEP_NOCOOL")) {
                lmode = 0;
                cool = cool_len;
                cool_len = std::min(2 * cool_len, 512);
                ++ws->lstat[1];
            }
        }
        if (lmode && !done && hc[4 + 4] > 0) {
            // a list past capacity (its (split, row) scans densely): grow the lists (the
            // stream is idle here) and record them again
            const long long ncap =
                (std::max<long long>(2 * ws->lcap, (long long)(1.25 * hc[4 + 5]) + 8) + 15) / 16 * 16;
            if (lmode == 2 && list_bytes(ncap, true) > list_budget()) {
                lmode = 0;                         // the grown lists would not fit: dense sweeps from here on
                kavail = false;
                continue;
            }
            ws->lcap = ncap;
            PINS_TRY(ensure_lists(ws, pb, st, lmode == 2));
            const int init[14] = {1, 1, -1, -1, 0, 0, hc[4 + 6], hc[4 + 7], 0, 0, 0, 0, hc[4 + 12], hc[4 + 13]};
            PINS_CUDA(cudaMemcpyAsync(ws->lctl.p, init, sizeof init, cudaMemcpyHostToDevice, st));
            ++ws->lstat[2];
            need[0] = need[1] = true;
        }
    }
    const bool lists = lmode != 0;
    if (lists) {
        ws->lstat[3] += hc[4 + 6] + hc[4 + 7];
        if (getenv("PINS_LIST_STATS"))     // dev instrumentation
            fprintf(stderr, "lists: sweeps %d cap %lld max %d overflow %d fallback units %d / %d records %d / %d "
                    "entries recorded %d / %d ELL stages (512 entries) %d / %d\n", hc[1], ws->lcap, hc[4 + 5],
                    hc[4 + 4], hc[4 + 6], hc[4 + 7], hc[4 + 12], hc[4 + 13], hc[4 + 14], hc[4 + 15], hc[4 + 10],
                    hc[4 + 11]);
    }
    return PINS_OK;
}

// Evaluation of X~(f, g) (Eq. (7)) in both orientations: sums, gradient,
// objectives; with tau > 0 also the sparsified CSR (rows) and CSC (columns).
// Grows the per-(row, split) capacity and re-runs on overflow.  Synchronises.
int run_eval(pins_workspace *ws, const pins_problem *pb, const double *phi, const double *psi, double s,
             const double *f, const double *g, double tau, bool trial, cudaStream_t st, EvalOut *out) {
    PINS_TRY(prepare(ws, pb));
    PINS_TRY(prepare_pass(ws, pb, st));
    const bool sparse = tau > 0.0;
    for (int attempt = 0; attempt < 6; ++attempt) {
        for (int q = 0; q < 2; ++q) {
            const long long M = q == 0 ? pb->m : pb->n;
            if (sparse) {
                PINS_TRY(ensure(ws->sb[q].bcol, sizeof(int) * M * ws->S[q] * ws->pcap));
                PINS_TRY(ensure(ws->sb[q].bval, sizeof(double) * M * ws->S[q] * ws->pcap));
            }
        }
        PassArgs A;
        base_args(ws, pb, s, A);
        fill_side(ws, pb, 0, f, phi, g, psi, A.side[0]);
        fill_side(ws, pb, 1, f, phi, g, psi, A.side[1]);
        A.nsides = 2;
        A.G0 = A.side[0].S * A.side[0].RB;
        const int G1 = A.side[1].S * A.side[1].RB;
        A.side[0].want_cx = 1;
        A.side[0].tau = A.side[1].tau = tau;
        if (trial) {
            A.side[0].eu = ptr<double>(ws->eu);
            A.side[0].ev = ptr<double>(ws->ev);
            A.side[0].bu = ptr<double>(ws->bu);
            A.side[0].bv = ptr<double>(ws->bv);
        }
        A.a_dot = pb->a; A.f_dot = f; A.b_dot = pb->b; A.g_dot = g;
        PINS_CUDA(launch_sum(ws->cost_row, ws->dp, A.G0 + G1, st, A, ws->tm_row, ws->tm_col));
        PINS_CUDA(cudaMemcpyAsync(ws->h, ws->pst.p, 12 * sizeof(double), cudaMemcpyDeviceToHost, st));
        PINS_CUDA(cudaStreamSynchronize(st));
        const double *h = ws->h;
        out->gnorm = h[0] + h[1];
        out->sumX = h[2];
        out->cost = h[3] * pb->cost_scale;
        out->em1 = h[4];
        out->maxz = h[5];
        out->maxcnt = h[6];
        out->nnz = h[7];
        out->af = h[8];
        out->maxr = h[9];
        out->maxc = h[10];
        out->dualP = h[8] - pb->eta * h[2];
        ws->csr_ready = ws->csc_ready = false;
        if (!sparse) return PINS_OK;
        if (out->maxcnt <= (double)ws->pcap) {
            const long long nnz = (long long)h[7];
            if ((long long)h[11] != nnz) {
                snprintf(g_err, sizeof g_err, "CSR/CSC pattern mismatch (%lld vs %lld)", nnz, (long long)h[11]);
                return PINS_ERR_NUMERIC;
            }
            PINS_TRY(ensure(ws->rowptr, sizeof(long long) * (pb->m + 1)));
            PINS_TRY(ensure(ws->colptr, sizeof(long long) * (pb->n + 1)));
            PINS_TRY(ensure(ws->colidx, sizeof(int) * std::max<long long>(nnz, 1)));
            PINS_TRY(ensure(ws->val, sizeof(double) * std::max<long long>(nnz, 1)));
            PINS_TRY(ensure(ws->rowidx, sizeof(int) * std::max<long long>(nnz, 1)));
            PINS_TRY(ensure(ws->valT, sizeof(double) * std::max<long long>(nnz, 1)));
            CsrOut O0{ptr<long long>(ws->rowptr), ptr<int>(ws->colidx), ptr<double>(ws->val),
                      ptr<long long>(ws->sb[0].blkoff)};
            CsrOut O1{ptr<long long>(ws->colptr), ptr<int>(ws->rowidx), ptr<double>(ws->valT),
                      ptr<long long>(ws->sb[1].blkoff)};
            // long rows (early EPPA): warp per row, one lane per split segment
            const int warpcopy = (double)nnz > 8.0 * (double)std::min(pb->m, pb->n) ? 1 : 0;
            LAUNCH(PINS_PROF_CSR, st, csr_build_kernel<<<A.side[0].RB + A.side[1].RB, kPT, 0, st>>>(
                A.side[0], A.side[1], 2, O0, O1, warpcopy));
            PINS_CUDA(cudaGetLastError());
            ws->nnz = nnz;
            ws->csr_ready = ws->csc_ready = true;
            return PINS_OK;
        }
        long long c = ws->pcap;
        while ((double)c < out->maxcnt) c *= 2;
        ws->pcap = c;
    }
    snprintf(g_err, sizeof g_err, "sparsify capacity did not converge");
    return PINS_ERR_NUMERIC;
}

int build_csc(pins_workspace *ws, long long m, long long n, const long long *rowptr,
              const int *colidx, const double *val, long long nnz, cudaStream_t st) {
    PINS_TRY(ensure(ws->colcnt, sizeof(int) * n));
    PINS_TRY(ensure(ws->cursor, sizeof(int) * n));
    PINS_TRY(ensure(ws->colptr, sizeof(long long) * (n + 1)));
    PINS_TRY(ensure(ws->rowidx, sizeof(int) * std::max<long long>(nnz, 1)));
    PINS_TRY(ensure(ws->valT, sizeof(double) * std::max<long long>(nnz, 1)));
    PINS_CUDA(cudaMemsetAsync(ws->colcnt.p, 0, sizeof(int) * n, st));
    PINS_CUDA(cudaMemsetAsync(ws->cursor.p, 0, sizeof(int) * n, st));
    const int gw = grid_1d(m * 32, ws->nsm);
    LAUNCH(PINS_PROF_CSR, st, csc_count_kernel<<<gw, 256, 0, st>>>(m, rowptr, colidx, ptr<int>(ws->colcnt)));
    LAUNCH(PINS_PROF_CSR, st, scan_counts_kernel<<<1, 1024, 0, st>>>(n, ptr<int>(ws->colcnt), 1LL << 40,
                                           ptr<long long>(ws->colptr)));
    LAUNCH(PINS_PROF_CSR, st, csc_fill_kernel<<<gw, 256, 0, st>>>(m, rowptr, colidx, val, ptr<long long>(ws->colptr),
                                        ptr<int>(ws->cursor), ptr<int>(ws->rowidx), ptr<double>(ws->valT)));
    LAUNCH(PINS_PROF_CSR, st, csc_sort_kernel<<<grid_1d(n, ws->nsm), 256, 0, st>>>(n, ptr<long long>(ws->colptr),
                                                         ptr<int>(ws->rowidx), ptr<double>(ws->valT)));
    PINS_CUDA(cudaGetLastError());
    return PINS_OK;
}

int cg_blocks(pins_workspace *ws, long long N, bool vec = false) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cg_kernel, kThreads, 0);
    // thread per row: one CTA per 256 rows; warp per row (vec): one warp per row, up to
    // 4 CTAs per SM (the per-iteration grid reductions read one partial per CTA)
    per_sm = std::max(1, std::min(per_sm, vec ? 4 : 2));
    long long want = vec ? (N * 32 + kThreads - 1) / kThreads : (N + kThreads - 1) / kThreads;
    return (int)std::max<long long>(1, std::min<long long>(want, (long long)ws->nsm * per_sm));
}

// CG launch on the CSR (rowptr/colidx/val) + workspace CSC.  Results in ws->cgst (device).
int run_cg(pins_workspace *ws, long long m, long long n, const long long *rowptr,
           const int *colidx, const double *val, const double *dr, const double *dc, double mu,
           const double *rhs, double *x, double rtol, int maxit, const double *gradf,
           const double *gradg, const double *a, const double *b, cudaStream_t st, long long nnz_hint = -1) {
    const long long N = m + n;
    PINS_TRY(ensure(ws->cgvec, sizeof(double) * 4 * N));
    const bool vec = (double)(nnz_hint >= 0 ? nnz_hint : ws->nnz) > 8.0 * (double)N;
    const int G = cg_blocks(ws, N, vec);
    PINS_TRY(ensure(ws->cgpart, sizeof(double) * 4 * G));
    PINS_TRY(ensure(ws->cgst, sizeof(double) * 8));
    CGArgs A;
    A.m = m;
    A.n = n;
    A.rowptr = rowptr;
    A.colidx = colidx;
    A.val = val;
    A.colptr = ptr<long long>(ws->colptr);
    A.rowidx = ptr<int>(ws->rowidx);
    A.valT = ptr<double>(ws->valT);
    A.dr = dr;
    A.dc = dc;
    A.mu = mu;
    A.rhs = rhs;
    A.x = x;
    double *v = ptr<double>(ws->cgvec);
    A.r = v;
    A.z = v + N;
    A.p = v + 2 * N;
    A.q = v + 3 * N;
    A.part = ptr<double>(ws->cgpart);
    A.rtol = rtol;
    A.maxit = maxit;
    A.gradf = gradf;
    A.gradg = gradg;
    A.a = a;
    A.b = b;
    A.st = ptr<double>(ws->cgst);
    A.vec = vec ? 1 : 0;
    void *args[] = {&A};
    cudaError_t e_cg = cudaSuccess;
    LAUNCH(PINS_PROF_CG, st, e_cg = cudaLaunchCooperativeKernel((void *)cg_kernel, dim3(G), dim3(kThreads), args, 0, st));
    PINS_CUDA(e_cg);
    return PINS_OK;
}


// ---- cluster-resident Schur-complement CG (pins_cg.cuh) ----
constexpr long long kClusterNnzMax = 400000;       // above: the grid-wide kernel streams faster
constexpr int kClusterSmem = 220 * 1024;           // dynamic shared memory per CTA
// fixed part of the cluster kernel's shared memory (vectors, pointers, heavy lists)
size_t cluster_cg_smem(long long m, long long n) {
    const long long keep = std::min(m, n), elim = std::max(m, n);
    const long long R = (keep + kCGC - 1) / kCGC, Cc = (elim + kCGC - 1) / kCGC;
    return sizeof(double) * (size_t)(8 * R + 2 * Cc) + sizeof(int) * (size_t)(2 * R + 2 * Cc + 2) + 16;
}
bool use_cluster_cg(pins_workspace *ws, long long m, long long n) {
    long long lim = kClusterNnzMax;
    if (const char *e = getenv("PINS_CLUSTER_NNZ_MAX")) lim = atoll(e);   // experiments
    return ws->nnz <= lim && cluster_cg_smem(m, n) <= (size_t)kClusterSmem - 16 * 1024 && ws->csc_ready;
}

// kept side = the smaller of (rows, columns); the other is eliminated exactly
int run_cg_cluster(pins_workspace *ws, long long m, long long n, double mu, const double *rhs, double *x,
                   double rtol, int maxit, const double *gradf, const double *gradg, const double *a,
                   const double *b, cudaStream_t st) {
    PINS_TRY(ensure(ws->cgst, sizeof(double) * 8));
    const bool keep_rows = m <= n;
    CGSArgs A;
    memset(&A, 0, sizeof A);
    A.m = keep_rows ? m : n;
    A.n = keep_rows ? n : m;
    const long long *rp = ptr<long long>(ws->rowptr), *cp = ptr<long long>(ws->colptr);
    const int *ci = ptr<int>(ws->colidx), *ri = ptr<int>(ws->rowidx);
    const double *v = ptr<double>(ws->val), *vt = ptr<double>(ws->valT);
    A.rowptr = keep_rows ? rp : cp;
    A.colidx = keep_rows ? ci : ri;
    A.val = keep_rows ? v : vt;
    A.colptr = keep_rows ? cp : rp;
    A.rowidx = keep_rows ? ri : ci;
    A.valT = keep_rows ? vt : v;
    const double *rs = ptr<double>(ws->rowsum), *cs = ptr<double>(ws->colsum);
    A.dr = keep_rows ? rs : cs;
    A.dc = keep_rows ? cs : rs;
    A.mu = mu;
    A.rhs_r = keep_rows ? rhs : rhs + m;
    A.rhs_c = keep_rows ? rhs + m : rhs;
    A.x_r = keep_rows ? x : x + m;
    A.x_c = keep_rows ? x + m : x;
    A.rtol = rtol;
    A.maxit = maxit;
    if (gradf) {
        A.grad_r = keep_rows ? gradf : gradg;
        A.grad_c = keep_rows ? gradg : gradf;
        A.a_r = keep_rows ? a : b;
        A.a_c = keep_rows ? b : a;
    }
    A.st = ptr<double>(ws->cgst);
    A.R = (int)((A.m + kCGC - 1) / kCGC);
    A.Cc = (int)((A.n + kCGC - 1) / kCGC);
    const size_t smem = kClusterSmem;
    A.smem = (int)smem;
    static bool configured = false;
    if (!configured) {
        PINS_CUDA(cudaFuncSetAttribute(cg_schur_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
        configured = true;
    }
    LAUNCH(PINS_PROF_CG, st, cg_schur_cluster_kernel<<<kCGC, kCGT, smem, st>>>(A));
    PINS_CUDA(cudaGetLastError());
    return PINS_OK;
}


// ---- spanning-tree preconditioned CG, one CTA (pins_tree.cuh) ----
constexpr int kTreeMaxNodes = 26000;               // tree-solve vector in shared memory
constexpr long long kTreeNnzMax = 400000;
bool use_tree_cg(pins_workspace *ws, long long m, long long n) {
    const char *e = getenv("PINS_CG");
    if (e && strcmp(e, "tree") != 0 && strcmp(e, "treecl") != 0) return false;
    // near-tree supports only (late EPPA: nnz ~ m + n, Thm 4.3); with many
    // off-tree edges the tree preconditioner loses its edge over Jacobi
    // adaptive: after a tree solve that needed many iterations (support far from
    // a tree), use the Jacobi-Schur cluster CG for a while, then try again
    const bool forced = e && (strcmp(e, "tree") == 0 || strcmp(e, "treecl") == 0);
    if (!forced && ws->tree_backoff > 0) {
        --ws->tree_backoff;
        return false;
    }
    // tried by default; a solve that needs > 80 iterations (support far from a
    // spanning tree) sends the next 256 Newton steps to the Jacobi-Schur cluster CG
    long long lim = kTreeNnzMax;
    if (const char *e2 = getenv("PINS_TREE_NNZ_MAX")) lim = atoll(e2);   // experiments
    return m + n <= kTreeMaxNodes && ws->nnz <= lim && ws->csc_ready;
}

int run_cg_tree(pins_workspace *ws, long long m, long long n, double mu, const double *rhs, double *x,
                double rtol, int maxit, const double *gradf, const double *gradg, const double *a,
                const double *b, cudaStream_t st, int setup_only = 0, bool force_rebuild = false,
                const double *wval = nullptr) {
    const long long N = m + n, nnz = std::max<long long>(ws->nnz, 1);
    PINS_TRY(ensure(ws->cgst, sizeof(double) * 16));
    // persistent arrays first, nnz-sized scratch last (offsets stay put as nnz changes)
    // comp hook tptr tnbr(2) deg fu fv1 fv2 tei tej tsrc(2) fs1 fs2 = 15 N, + rstart, ctr
    const long long ni_fixed = 15 * N + 1 + kTreeMaxRounds + 1 + 8 + (11 * N + 1);   // + pull lists
    const long long ni = ni_fixed + nnz;
    const long long nd = 4 * N + 2 * N + N + 3 * N + 4 * N + 3 * N + 5 * N;   // pull entries, tw, dcur, fc1/fc2/finv, r z p q, tval fw1 fw2, frec
    const unsigned old_i = ws->tr_i.gen, old_d = ws->tr_d.gen;
    PINS_TRY(ensure(ws->tr_i, sizeof(int) * ni));
    PINS_TRY(ensure(ws->tr_d, sizeof(double) * nd));
    PINS_TRY(ensure(ws->tr_u8, (size_t)(nnz + 2 * N)));
    PINS_TRY(ensure(ws->tr_u64, sizeof(unsigned long long) * N));
    if (ws->tr_i.gen != old_i || ws->tr_d.gen != old_d || ws->tree_N != N) ws->tree_valid = false;
    TreeArgs A;
    memset(&A, 0, sizeof A);
    A.m = (int)m;
    A.n = (int)n;
    A.nnz = ws->nnz;
    A.rowptr = ptr<long long>(ws->rowptr);
    A.colidx = ptr<int>(ws->colidx);
    A.val = wval ? wval : ptr<double>(ws->val);     // wval: certificate repair weights (setup only)
    A.colptr = ptr<long long>(ws->colptr);
    A.rowidx = ptr<int>(ws->rowidx);
    A.valT = ptr<double>(ws->valT);
    A.dr = ptr<double>(ws->rowsum);
    A.dc = ptr<double>(ws->colsum);
    A.mu = mu;
    A.rhs = rhs;
    A.x = x;
    A.rtol = rtol;
    A.maxit = maxit;
    A.gradf = gradf;
    A.gradg = gradg;
    A.a = a;
    A.b = b;
    A.st = ptr<double>(ws->cgst);
    int *ip = ptr<int>(ws->tr_i);
    A.pk = reinterpret_cast<int4 *>(ip); ip += 4 * N;     // 16-byte aligned: first in the pool
    A.comp = ip; ip += N;
    A.hook = ip; ip += N;
    A.tptr = ip; ip += N + 1;
    A.tnbr = ip; ip += 2 * N;
    A.deg = ip; ip += N;
    A.fu = ip; ip += N;
    A.fv1 = ip; ip += N;
    A.fv2 = ip; ip += N;
    A.rstart = ip; ip += kTreeMaxRounds + 1;
    A.ctr = ip; ip += 8;
    A.tei = ip; ip += N;
    A.tej = ip; ip += N;
    A.tsrc = ip; ip += 2 * N;
    A.fs1 = ip; ip += N;
    A.fs2 = ip; ip += N;
    A.cptr = ip; ip += N + 1;
    A.cent = ip; ip += 2 * N;
    A.ppos = ip; ip += 2 * N;
    A.rpos = ip; ip += N;
    A.cur = ip; ip += N;
    A.erow = ip;
    double *dp_ = ptr<double>(ws->tr_d);
    A.pe = reinterpret_cast<PullE *>(dp_); dp_ += 4 * N;  // 16-byte aligned: first in the pool
    A.tw = dp_; dp_ += 2 * N;
    A.dcur = dp_; dp_ += N;
    A.fc1 = dp_; dp_ += N;
    A.fc2 = dp_; dp_ += N;
    A.finv = dp_; dp_ += N;
    A.r = dp_; dp_ += N;
    A.z = dp_; dp_ += N;
    A.p = dp_; dp_ += N;
    A.q = dp_; dp_ += N;
    A.tval = dp_; dp_ += N;
    A.fw1 = dp_; dp_ += N;
    A.fw2 = dp_; dp_ += N;
    A.frec = dp_;
    unsigned char *bp = ptr<unsigned char>(ws->tr_u8);
    A.alive = bp; bp += N;
    A.sel = bp; bp += N;
    A.tmark = bp;
    A.best = ptr<unsigned long long>(ws->tr_u64);
    // reuse the stored tree while it keeps CG short (the kernel also checks that
    // every tree edge is still in the support and rebuilds otherwise)
    A.reuse = ws->tree_valid && ws->tree_last_its <= 48 && !force_rebuild && !getenv("PINS_TREE_NO_REUSE") ? 1 : 0;
    A.setup_only = setup_only;
    ws->tree_rstart = A.rstart;
    ws->tree_ctr = A.ctr;
    ws->tree_frec = A.frec;
    ws->tree_last = A;
    const size_t base = sizeof(double) * (size_t)N;
    const size_t budget = 220 * 1024;
    A.tail_cap = base < budget ? (int)((budget - base) / 40) : 0;
    const size_t smem = base + (size_t)A.tail_cap * 40;
    static size_t configured = 0;
    if (smem > configured) {
        PINS_CUDA(cudaFuncSetAttribute(tree_pcg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)std::max<size_t>(smem, 48 * 1024)));
        configured = std::max<size_t>(smem, 48 * 1024);
    }
    LAUNCH(PINS_PROF_CG, st, tree_pcg_kernel<<<1, kTT, smem, st>>>(A));
    PINS_CUDA(cudaGetLastError());
    ws->tree_valid = true;
    ws->tree_newton = wval == nullptr;
    ws->tree_stale = 0;
    ws->tree_N = N;
    return PINS_OK;
}

// Tree factor by the single-CTA kernel (setup only), then the PCG on one cluster:
// CTAs 1..7 hold the vectors, CTA 0 applies the tree preconditioner (pins_treecl.cuh)
int run_cg_tree_cluster(pins_workspace *ws, long long m, long long n, double mu, const double *rhs, double *x,
                        double rtol, int maxit, const double *gradf, const double *gradg, const double *a,
                        const double *b, cudaStream_t st) {
    const long long N = m + n;
    // The preconditioner only has to be SPD: the factor of an earlier Newton system's
    // M_T (an exact LDL^T of that SPD matrix) is one.  Late in EPPA the support and its
    // weights change little between Newton systems, so while the PCG stays short the
    // stored factor is reused instead of refactorised (the CG itself always multiplies
    // by the current M, so the system solved and its residual test are unchanged).
    static const int stale_its = getenv("PINS_STALE_ITS") ? atoi(getenv("PINS_STALE_ITS")) : 8;
    static const int stale_max = getenv("PINS_STALE_MAX") ? atoi(getenv("PINS_STALE_MAX")) : 64;
    const bool stale = ws->tree_valid && ws->tree_newton && ws->tree_N == N && ws->tree_last_its <= stale_its &&
                       ws->tree_stale < stale_max;
    if (stale) ++ws->tree_stale;
    else PINS_TRY(run_cg_tree(ws, m, n, mu, rhs, x, rtol, maxit, gradf, gradg, a, b, st, 1));
    TreeCLArgs A;
    memset(&A, 0, sizeof A);
    A.m = (int)m;
    A.n = (int)n;
    A.rowptr = ptr<long long>(ws->rowptr);
    A.colidx = ptr<int>(ws->colidx);
    A.val = ptr<double>(ws->val);
    A.colptr = ptr<long long>(ws->colptr);
    A.rowidx = ptr<int>(ws->rowidx);
    A.valT = ptr<double>(ws->valT);
    A.dr = ptr<double>(ws->rowsum);
    A.dc = ptr<double>(ws->colsum);
    A.mu = mu;
    A.rhs = rhs;
    A.x = x;
    A.rtol = rtol;
    A.maxit = maxit;
    A.gradf = gradf;
    A.gradg = gradg;
    A.a = a;
    A.b = b;
    A.st = ptr<double>(ws->cgst);
    // the packed factor written by the setup kernel (pointers recorded by run_cg_tree)
    A.rstart = ws->tree_rstart;
    A.ctr = ws->tree_ctr;
    A.frec = ws->tree_frec;
    A.cptr = ws->tree_last.cptr;
    A.pk = ws->tree_last.pk;
    A.pe = ws->tree_last.pe;
    A.R = (int)((N + kTCW - 1) / kTCW);
    const size_t base = sizeof(double) * (size_t)N;
    const size_t budget = 220 * 1024;
    // per cached tail record: the 40-byte factor record, a list offset and two list entries
    constexpr size_t kTailB = 40 + 16 + 2 * 16;      // record, pull header, two pull entries
    A.tail_cap = base + 64 < budget ? (int)((budget - base - 64) / kTailB) : 0;
    A.use_x0 = ws->x0_enable && ws->dir_valid && x == ptr<double>(ws->dir) && getenv("PINS_NO_X0") == nullptr;
    const size_t smem = std::max<size_t>(base + (size_t)A.tail_cap * kTailB + 64, sizeof(double) * 5 * (size_t)A.R);
    static size_t configured = 0;
    if (smem > configured) {
        PINS_CUDA(cudaFuncSetAttribute(cg_tree_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)std::max<size_t>(smem, 48 * 1024)));
        configured = std::max<size_t>(smem, 48 * 1024);
    }
    LAUNCH(PINS_PROF_CG, st, cg_tree_cluster_kernel<<<kCGC, kCGT, smem, st>>>(A));
    PINS_CUDA(cudaGetLastError());
    return PINS_OK;
}

// ------------------------------------------------------------ LP certificate
// (reading R11; pins_cert.cuh).  c-transform of `pin` over the cost: orient 0
// (rows of C): out_i = min_j (C_ij - pin_j); orient 1 (columns): out_j =
// min_i (C_ij - pin_i).  mode 1: out_p = max_q (self_p + pin_q - C_pq).
int ctrans(pins_workspace *ws, const pins_problem *pb, int orient, int mode, const double *pin,
           const double *self, double *out, cudaStream_t st) {
    const bool dense = pb->cost_kind == PINS_COST_DENSE;
    CtArgs A;
    memset(&A, 0, sizeof A);
    A.M = orient == 0 ? pb->m : pb->n;
    A.N = orient == 0 ? pb->n : pb->m;
    A.orient = orient;
    A.mode = mode;
    A.cd = make_cd(pb);
    if (!dense && orient == 1) std::swap(A.cd.x, A.cd.y);
    A.scale = pb->cost_scale;
    A.pin = pin;
    A.self = self;
    const long long RB = dense && orient == 0 ? (A.M + 3) / 4 : (A.M + kCtT - 1) / kCtT;
    long long S = (4LL * ws->nsm + RB - 1) / RB;
    S = std::max(1LL, std::min(S, std::max(1LL, A.N / 64)));
    A.S = (int)S;
    PINS_TRY(ensure(ws->cpart, sizeof(double) * S * A.M));
    A.part = ptr<double>(ws->cpart);
    const int grid = (int)(RB * S);
    if (dense && orient == 0) LAUNCH(PINS_PROF_VEC, st, ctrans_dense_rows_kernel<<<grid, kCtT, 0, st>>>(A));
    else if (dense) LAUNCH(PINS_PROF_VEC, st, ctrans_dense_cols_kernel<<<grid, kCtT, 0, st>>>(A));
    else if (pb->cost_kind == PINS_COST_SQEUCLID) LAUNCH(PINS_PROF_VEC, st, ctrans_points_kernel<1><<<grid, kCtT, 0, st>>>(A));
    else LAUNCH(PINS_PROF_VEC, st, ctrans_points_kernel<2><<<grid, kCtT, 0, st>>>(A));
    LAUNCH(PINS_PROF_VEC, st, ctrans_finalize_kernel<<<grid_1d(A.M, ws->nsm), 256, 0, st>>>(A.M, A.S, mode,
                                                                                        A.part, out));
    PINS_CUDA(cudaGetLastError());
    return PINS_OK;
}

struct CertOut {
    double primal = 0, pobj = 0, dobj = -INFINITY, gap = INFINITY, dual_inf = -1;
    int tree_edges = 0, used_tree = 0, components = 0, repairs = 0, violations = 0;
    long long nnz = 0;
};

// <a,u> + <b,v> on the device (deterministic), read back (synchronises)
int dual_value(pins_workspace *ws, const pins_problem *pb, const double *u, const double *v, double *out,
               cudaStream_t st) {
    LAUNCH(PINS_PROF_REDUCE, st, dots_kernel<<<1, 1024, 0, st>>>(pb->m, pb->n, pb->a, u, pb->b, v,
                                                                 ptr<double>(ws->rowsum), ptr<double>(ws->colsum),
                                                                 ptr<double>(ws->st)));
    PINS_CUDA(cudaMemcpyAsync(ws->h + 24, ptr<double>(ws->st) + 8, sizeof(double), cudaMemcpyDeviceToHost, st));
    PINS_CUDA(cudaStreamSynchronize(st));
    *out = ws->h[24];
    return PINS_OK;
}

// Measured dual infeasibility of the certified duals: max(0, max_ij u_i + v_j - C_ij)
// (one more pass; the c-transforms make it 0 up to rounding).  Synchronises.
int measure_dual_inf(pins_workspace *ws, const pins_problem *pb, CertOut *co, cudaStream_t st) {
    PINS_TRY(ctrans(ws, pb, 0, 1, ptr<double>(ws->cbv), ptr<double>(ws->cbu), ptr<double>(ws->crow), st));
    LAUNCH(PINS_PROF_REDUCE, st, vec_max_kernel<<<1, 1024, 0, st>>>(pb->m, ptr<double>(ws->crow), ptr<double>(ws->st), 12));
    PINS_CUDA(cudaMemcpyAsync(ws->h + 25, ptr<double>(ws->st) + 12, sizeof(double), cudaMemcpyDeviceToHost, st));
    PINS_CUDA(cudaStreamSynchronize(st));
    co->dual_inf = ws->h[25];
    return PINS_OK;
}

// c-transforms of (u0, v0) (rows, then columns) into (u1, v1), bound D; the
// best bound so far and its duals are kept in co / ws->cbu, cbv.
int ctrans_candidate(pins_workspace *ws, const pins_problem *pb, const double *v0, double *u1, double *v1,
                     int used_tree, CertOut *co, cudaStream_t st) {
    PINS_TRY(ctrans(ws, pb, 0, 0, v0, nullptr, u1, st));      // u'_i = min_j C_ij - v_j
    PINS_TRY(ctrans(ws, pb, 1, 0, u1, nullptr, v1, st));      // v'_j = min_i C_ij - u'_i
    double D = 0.0;
    PINS_TRY(dual_value(ws, pb, u1, v1, &D, st));
    if (std::isfinite(D) && D > co->dobj) {
        co->dobj = D;
        co->used_tree = used_tree;
        PINS_CUDA(cudaMemcpyAsync(ws->cbu.p, u1, sizeof(double) * pb->m, cudaMemcpyDeviceToDevice, st));
        PINS_CUDA(cudaMemcpyAsync(ws->cbv.p, v1, sizeof(double) * pb->n, cudaMemcpyDeviceToDevice, st));
    }
    return PINS_OK;
}

// Tree candidate (reading R11): maximum-weight spanning forest of the support,
// tree duals, component gauges by shortest paths, c-transforms; then up to
// kRepairRounds repairs: support edges the tree duals violate are forced into
// the next forest (pins_cert.cuh support_rc_kernel).
constexpr int kRepairRounds = 3;
int certify_tree(pins_workspace *ws, const pins_problem *pb, const EvalOut &cur, CertOut *co, cudaStream_t st,
                 double target_gap) {
    const long long m = pb->m, n = pb->n, N = m + n, nnz = ws->nnz;
    for (DevBuf *b : {&ws->cz, &ws->cdd, &ws->cdf, &ws->ctc}) PINS_TRY(ensure(*b, sizeof(double) * N));
    PINS_TRY(ensure(ws->ccomp, sizeof(int) * N));
    PINS_TRY(ensure(ws->ccid, sizeof(int) * N));
    PINS_TRY(ensure(ws->cinfo, sizeof(int) * 8));
    PINS_TRY(ensure(ws->cR, sizeof(unsigned long long) * kMaxComp * kMaxComp));
    PINS_TRY(ensure(ws->cdsh, sizeof(double) * kMaxComp));
    PINS_TRY(ensure(ws->cw, sizeof(double) * std::max<long long>(nnz, 1)));
    double *u0 = ptr<double>(ws->cu0), *v0 = ptr<double>(ws->cv0);
    double *u1 = ptr<double>(ws->cu1), *v1 = ptr<double>(ws->cv1);
    int *info = ptr<int>(ws->cinfo);
    const CostDesc cd = make_cd(pb);
    const double *wts = nullptr;                    // round 0: the plan's own weights
    for (int round = 0; round < kRepairRounds; ++round) {
        PINS_TRY(run_cg_tree(ws, m, n, 0.0, ptr<double>(ws->rhs), ptr<double>(ws->uv), 0.5, 1, nullptr, nullptr,
                             nullptr, nullptr, st, 1, true, wts));
        const TreeArgs &T = ws->tree_last;
        TreeDualArgs D;
        D.m = (int)m; D.n = (int)n;
        D.ctr = T.ctr; D.rstart = T.rstart;
        D.fu = T.fu; D.fv1 = T.fv1; D.fv2 = T.fv2; D.fs1 = T.fs1; D.fs2 = T.fs2;
        D.tei = T.tei; D.tej = T.tej;
        D.cd = cd;
        D.scale = pb->cost_scale;
        D.dd = ptr<double>(ws->cdd); D.df = ptr<double>(ws->cdf); D.tc = ptr<double>(ws->ctc);
        D.z = ptr<double>(ws->cz);
        D.comp = ptr<int>(ws->ccomp);
        LAUNCH(PINS_PROF_VEC, st, tree_duals_kernel<<<1, 1024, 0, st>>>(D));
        LAUNCH(PINS_PROF_VEC, st, split_duals_kernel<<<grid_1d(N, ws->nsm), 256, 0, st>>>(m, n, D.z, u0, v0));
        // component gauges (no-ops on the device when the forest is connected)
        unsigned long long *R = ptr<unsigned long long>(ws->cR);
        LAUNCH(PINS_PROF_VEC, st, comp_ids_kernel<<<1, 1024, 0, st>>>((int)N, D.comp, ptr<int>(ws->ccid), info, R));
        LAUNCH(PINS_PROF_VEC, st, comp_rmin_kernel<<<(int)((m + kCtT - 1) / kCtT), kCtT, 0, st>>>(
            m, n, cd, pb->cost_scale, u0, v0, D.comp, ptr<int>(ws->ccid), info, R));
        LAUNCH(PINS_PROF_VEC, st, comp_shift_solve_kernel<<<1, 1, 0, st>>>(info, R, ptr<double>(ws->cdsh), info + 1));
        LAUNCH(PINS_PROF_VEC, st, comp_shift_apply_kernel<<<grid_1d(N, ws->nsm), 256, 0, st>>>(
            m, n, D.comp, ptr<int>(ws->ccid), info + 1, ptr<double>(ws->cdsh), u0, v0));
        PINS_CUDA(cudaGetLastError());
        PINS_TRY(ctrans_candidate(ws, pb, v0, u1, v1, 1, co, st));
        int hi[4];
        PINS_CUDA(cudaMemcpyAsync(hi, info, sizeof(int) * 2, cudaMemcpyDeviceToHost, st));
        PINS_CUDA(cudaMemcpyAsync(hi + 2, T.ctr + 2, sizeof(int), cudaMemcpyDeviceToHost, st));
        PINS_CUDA(cudaStreamSynchronize(st));
        co->tree_edges = hi[2];
        co->components = hi[0];
        co->repairs = round;
        if (co->pobj - co->dobj <= target_gap || round + 1 == kRepairRounds) break;
        // repair: force the support edges these duals violate into the next forest
        PINS_CUDA(cudaMemsetAsync(info + 2, 0, sizeof(int), st));
        LAUNCH(PINS_PROF_VEC, st, support_rc_kernel<<<grid_1d(nnz, ws->nsm), 256, 0, st>>>(
            nnz, T.erow, ptr<int>(ws->colidx), ptr<double>(ws->val), cd, pb->cost_scale, u0, v0,
            1e-13 * (1.0 + std::fabs(cur.cost)), ptr<double>(ws->cw), round == 0 ? 1 : 0, info + 2));
        int nviol = 0;
        PINS_CUDA(cudaMemcpyAsync(&nviol, info + 2, sizeof(int), cudaMemcpyDeviceToHost, st));
        PINS_CUDA(cudaStreamSynchronize(st));
        co->violations = nviol;
        if (nviol == 0) break;
        wts = ptr<double>(ws->cw);
    }
    return PINS_OK;
}

// Certificate of the plan X~(f, g) at centre (phi, psi, s), whose evaluation
// (sums, CSR / CSC at tau) is the workspace state `cur` (reading R11): basis
// forest -> tree duals -> row / column c-transforms; the entropic duals
// ((f + phi)/s, (g + psi - eta)/s) are the second candidate; the larger
// certified bound wins.  Certified duals -> ws->cbu / cbv.
// Support of the certificate: entries X~_ij >= kThetaCert/(m n) -- far below the
// Newton sparsification threshold, so that basic edges carrying tiny flows (which
// connect otherwise separate components) are part of the graph (reading R11).
constexpr double kThetaCert = 1e-12;

int certify(pins_workspace *ws, const pins_problem *pb, const double *phi, const double *psi, double s,
            const double *f, const double *g, bool want_dual_inf, CertOut *co, cudaStream_t st,
            double target_gap = -INFINITY) {
    *co = CertOut();
    const long long m = pb->m, n = pb->n, N = m + n;
    EvalOut cur;
    PINS_TRY(run_eval(ws, pb, phi, psi, s, f, g, kThetaCert / ((double)m * (double)n), false, st, &cur));
    PINS_TRY(prepare(ws, pb));
    for (DevBuf *b : {&ws->cu0, &ws->cu1, &ws->cbu, &ws->crow}) PINS_TRY(ensure(*b, sizeof(double) * std::max(m, n)));
    for (DevBuf *b : {&ws->cv0, &ws->cv1, &ws->cbv}) PINS_TRY(ensure(*b, sizeof(double) * n));
    co->primal = cur.gnorm;
    co->pobj = cur.cost;
    co->nnz = ws->nnz;
    double *u0 = ptr<double>(ws->cu0), *v0 = ptr<double>(ws->cv0);
    double *u1 = ptr<double>(ws->cu1), *v1 = ptr<double>(ws->cv1);
    for (int cand = 0; cand < 2; ++cand) {
        if (cand == 0) {                            // tree duals of the basis forest, repaired
            if (!(N <= kTreeMaxNodes && ws->csr_ready && ws->csc_ready && ws->nnz >= 1)) continue;
            PINS_TRY(certify_tree(ws, pb, cur, co, st, target_gap));
            if (co->pobj - co->dobj <= target_gap) break;
            continue;
        } else {            // entropic duals (reading R8)
            LAUNCH(PINS_PROF_VEC, st, lp_duals_kernel<<<grid_1d(N, ws->nsm), 256, 0, st>>>(
                m, n, pb->eta, 1.0 / s, f, g, phi, psi, u0, v0));
            PINS_CUDA(cudaGetLastError());
        }
        PINS_TRY(ctrans_candidate(ws, pb, v0, u1, v1, 0, co, st));
    }
    co->gap = co->pobj - co->dobj;
    if (want_dual_inf) PINS_TRY(measure_dual_inf(ws, pb, co, st));
    return PINS_OK;
}

double cg_rtol(const pins_params *p, double gnorm) {
    if (p->cg_forcing <= 0.0 || gnorm <= 0.0) return p->cg_tol;
    return std::min(0.5, std::max(p->cg_tol, p->cg_forcing * p->newton_tol / gnorm));
}

// One Newton iteration from the current sparse evaluation state (ws buffers
// hold X~(f,g) sums, gradient and CSR).  On return the state is that of the
// new point.  info: [0] gnorm before [1] after [2] alpha [3] cg its [4] relres
// [5] nnz [6] trials.
int newton_iter(pins_workspace *ws, const pins_problem *pb, const pins_params *prm,
                const double *phi, const double *psi, double s, double *f, double *g,
                EvalOut *cur, double *info, cudaStream_t st) {
    const long long m = pb->m, n = pb->n, N = m + n;
    const double tau = prm->theta / ((double)m * (double)n);
    info[0] = cur->gnorm;
    info[5] = (double)ws->nnz;
    if (!ws->csr_ready) {
        EvalOut e;
        PINS_TRY(run_eval(ws, pb, phi, psi, s, f, g, tau, false, st, &e));
        *cur = e;
    }
    double *rhs = ptr<double>(ws->rhs);
    LAUNCH(PINS_PROF_VEC, st, scale_concat_kernel<<<grid_1d(N, ws->nsm), 256, 0, st>>>(m, n, pb->eta, ptr<double>(ws->gradf),
                                                              ptr<double>(ws->gradg), rhs));
    PINS_CUDA(cudaGetLastError());
    const double mu = prm->mu_rel * std::max(cur->maxr, cur->maxc);
    const double rtol = cg_rtol(prm, cur->gnorm);
    double *d = ptr<double>(ws->dir);
    const bool used_tree = use_tree_cg(ws, m, n);
    const char *cgsel = getenv("PINS_CG");
    // default tree path: factor on one CTA, PCG on a cluster; PINS_CG=tree keeps the
    // whole PCG on the single CTA
    const bool treecl = used_tree && !(cgsel && strcmp(cgsel, "tree") == 0);
    if (treecl) {
        PINS_TRY(run_cg_tree_cluster(ws, m, n, mu, rhs, d, rtol, prm->cg_maxit, ptr<double>(ws->gradf),
                                     ptr<double>(ws->gradg), pb->a, pb->b, st));
    } else if (used_tree) {
        PINS_TRY(run_cg_tree(ws, m, n, mu, rhs, d, rtol, prm->cg_maxit, ptr<double>(ws->gradf),
                             ptr<double>(ws->gradg), pb->a, pb->b, st));
    } else if (use_cluster_cg(ws, m, n) && !(getenv("PINS_CG") && strcmp(getenv("PINS_CG"), "cluster") != 0)) {
        PINS_TRY(run_cg_cluster(ws, m, n, mu, rhs, d, rtol, prm->cg_maxit, ptr<double>(ws->gradf),
                                ptr<double>(ws->gradg), pb->a, pb->b, st));
    } else {
        PINS_TRY(run_cg(ws, m, n, ptr<long long>(ws->rowptr), ptr<int>(ws->colidx), ptr<double>(ws->val),
                        ptr<double>(ws->rowsum), ptr<double>(ws->colsum), mu, rhs, d, rtol,
                        prm->cg_maxit, ptr<double>(ws->gradf), ptr<double>(ws->gradg), pb->a, pb->b, st));
    }
    PINS_CUDA(cudaMemcpyAsync(ws->h + 16, ws->cgst.p, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
    PINS_CUDA(cudaStreamSynchronize(st));
    const double cg_its = ws->h[16], relres = ws->h[17], slope = ws->h[18], ad = ws->h[19];
    ws->dir_valid = d == ptr<double>(ws->dir) && relres == relres;
    // algorithmic bytes of this CG launch: per iteration the CSR + CSC (12 B per
    // entry each) and ~10 vector streams of m + n doubles
    g_prof.work[PINS_PROF_CG] += cg_its * (24.0 * (double)ws->nnz + 80.0 * (double)N);
    if (used_tree) {
        ws->tree_last_its = (int)cg_its;
        if (cg_its > 80) ws->tree_backoff = 256;
    }
    if (getenv("PINS_TREE_STATS") && used_tree) {    // dev instrumentation
        double hs[16];
        cudaMemcpy(hs, ws->cgst.p, sizeof hs, cudaMemcpyDeviceToHost);
        static double acc[8] = {0};
        static long calls = 0;
        for (int q = 0; q < 7; ++q) acc[q] += hs[4 + q];
        acc[7] += hs[11];
        ++calls;
        if (calls % 200 == 1 || getenv("PINS_TREE_STATS")[0] == '2')
            fprintf(stderr, "  last call: its %.0f rebuilt %.0f stale %d rounds %.0f | kcycles mst %.1f fac %.1f pc %.1f (fwd %.1f warp %.1f bwd %.1f, R0/RW %.0f) mv %.1f total %.1f\n",
                    cg_its, hs[11], ws->tree_stale, hs[4], hs[6] / 1e3, hs[7] / 1e3, hs[8] / 1e3, hs[12] / 1e3,
                    hs[13] / 1e3, hs[14] / 1e3, hs[15], hs[9] / 1e3, hs[10] / 1e3);
        if (calls % 200 == 1)
            fprintf(stderr, "tree-cg calls %ld nnz %lld its %.0f rebuilds %.0f | Mcycles mst %.1f fac %.1f pc %.1f mv %.1f total %.1f\n",
                    calls, ws->nnz, cg_its, acc[7], acc[2] / 1e6, acc[3] / 1e6, acc[4] / 1e6, acc[5] / 1e6, acc[6] / 1e6);
    }
    info[3] = cg_its;
    info[4] = relres;
    double alpha = 1.0;
    bool ok = false;
    int trials = 0;
    EvalOut e;
    if (slope > 0.0 && std::isfinite(slope)) {
        for (int t = 0; t < prm->max_backtracks; ++t) {
            ++trials;
            LAUNCH(PINS_PROF_VEC, st, trial_prep_kernel<<<grid_1d(N, ws->nsm), 256, 0, st>>>(
                m, n, alpha, 1.0 / pb->eta, f, g, d, ptr<double>(ws->ft), ptr<double>(ws->gt),
                ptr<double>(ws->eu), ptr<double>(ws->ev), ptr<double>(ws->bu), ptr<double>(ws->bv)));
            PINS_CUDA(cudaGetLastError());
            PINS_TRY(run_eval(ws, pb, phi, psi, s, ptr<double>(ws->ft), ptr<double>(ws->gt), tau, true,
                              st, &e));
            // P(x + alpha d) - P(x) = alpha <(a,b), d> + eta sum X_new expm1(-alpha(d_i+d_j)/eta)
            const double inc = alpha * ad + pb->eta * e.em1;
            if (std::isfinite(inc) && std::isfinite(e.gnorm) && inc >= prm->armijo_c * alpha * slope) {
                ok = true;
                break;
            }
            alpha *= prm->beta;
        }
    }
    info[6] = trials;
    if (ok) {
        PINS_CUDA(cudaMemcpyAsync(f, ws->ft.p, sizeof(double) * m, cudaMemcpyDeviceToDevice, st));
        PINS_CUDA(cudaMemcpyAsync(g, ws->gt.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        *cur = e;
        info[2] = alpha;
    } else {
        PINS_TRY(run_eval(ws, pb, phi, psi, s, f, g, tau, false, st, cur));
        info[2] = 0.0;
    }
    info[1] = cur->gnorm;
    return PINS_OK;
}

bool outer_converged(const std::vector<double> &objs, const pins_params *p) {
    const size_t k = objs.size();
    if (k < 2) return false;
    const double cur = objs.back();
    const double scale = std::max(std::fabs(cur), 1e-300);
    if (p->outer_rule == 0) return std::fabs(cur - objs[k - 2]) <= p->outer_tol * scale;
    if (p->outer_rule == 1) {
        const double half = objs[(k - 1) / 2];
        return (half - cur) <= p->outer_tol * scale && k >= 4;
    }
    const size_t W = std::max<size_t>(5, k / 4);
    if (k < 2 * W + 1) return false;
    const double D1 = objs[k - 1 - 2 * W] - objs[k - 1 - W];
    const double D2 = objs[k - 1 - W] - cur;
    if (D2 <= 0.0) return D1 >= 0.0 && std::fabs(D2) <= p->outer_tol * scale;
    if (D1 <= 0.0) return false;
    const double r = D2 / D1;
    if (r >= 1.0) return false;
    return D2 * r / (1.0 - r) <= p->outer_tol * scale;
}

}  // namespace

// ------------------------------------------------------------------ C ABI
extern "C" int pins_center_init(const pins_problem *pb, double *phi, double *psi, double *s_host,
                                void *stream) {
    PINS_TRY(check_problem(pb));
    PINS_ARG(phi && psi && s_host, "phi, psi, s");
    cudaStream_t st = (cudaStream_t)stream;
    LAUNCH(PINS_PROF_VEC, st, center_init_kernel<<<grid_1d(pb->m + pb->n, 148), 256, 0, st>>>(pb->m, pb->n, pb->eta, pb->a, pb->b,
                                                                    phi, psi));
    PINS_CUDA(cudaGetLastError());
    *s_host = 1.0;
    return PINS_OK;
}

extern "C" int pins_center_update(const pins_problem *pb, double *phi, double *psi, double *s_host,
                                  const double *f, const double *g, void *stream) {
    PINS_TRY(check_problem(pb));
    PINS_ARG(phi && psi && s_host && f && g, "phi, psi, s, f, g");
    cudaStream_t st = (cudaStream_t)stream;
    LAUNCH(PINS_PROF_VEC, st, center_update_kernel<<<grid_1d(pb->m + pb->n, 148), 256, 0, st>>>(pb->m, pb->n, pb->eta, f, g, phi,
                                                                      psi));
    PINS_CUDA(cudaGetLastError());
    *s_host += 1.0;
    return PINS_OK;
}

extern "C" int pins_sinkhorn_sweep(pins_workspace *ws, const pins_problem *pb, const double *phi,
                                   const double *psi, double s, double *f, double *g, void *stream) {
    PINS_ARG(ws != nullptr, "ws");
    PINS_TRY(check_problem(pb));
    invalidate_problem(ws);
    PINS_ARG(phi && psi && f && g && s > 0.0, "phi, psi, f, g, s > 0");
    return do_sweep(ws, pb, phi, psi, s, f, g, (cudaStream_t)stream);
}

extern "C" int pins_sinkhorn(pins_workspace *ws, const pins_problem *pb, const double *phi, const double *psi,
                             double s, double *f, double *g, double tol, int32_t max_sweeps, int32_t *sweeps_host,
                             double *res_host, void *stream) {
    PINS_ARG(ws != nullptr && sweeps_host && res_host, "ws, sweeps, res");
    PINS_TRY(check_problem(pb));
    invalidate_problem(ws);
    PINS_ARG(phi && psi && f && g && s > 0.0 && max_sweeps >= 0 && tol >= 0.0, "phi, psi, f, g, s > 0, budget, tol");
    cudaStream_t st = (cudaStream_t)stream;
    pins_params prm;
    pins_default_params(&prm);
    prm.T1 = max_sweeps;
    prm.sink_tol = tol;
    EvalOut e;
    PINS_TRY(run_eval(ws, pb, phi, psi, s, f, g, 0.0, false, st, &e));
    int t = 0;
    PINS_TRY(sinkhorn_phase(ws, pb, &prm, phi, psi, s, f, g, e.gnorm, &t, st));
    if (t > 0) PINS_TRY(run_eval(ws, pb, phi, psi, s, f, g, 0.0, false, st, &e));
    *sweeps_host = t;
    *res_host = e.gnorm;
    return PINS_OK;
}

extern "C" int pins_evaluate(pins_workspace *ws, const pins_problem *pb, const double *phi,
                             const double *psi, double s, const double *f, const double *g, double tau,
                             double *r, double *c, double *out_host, void *stream) {
    PINS_ARG(ws != nullptr && out_host != nullptr, "ws, out_host");
    PINS_TRY(check_problem(pb));
    invalidate_problem(ws);
    PINS_ARG(phi && psi && f && g && s > 0.0, "phi, psi, f, g, s > 0");
    cudaStream_t st = (cudaStream_t)stream;
    EvalOut e;
    PINS_TRY(run_eval(ws, pb, phi, psi, s, f, g, tau, false, st, &e));
    if (r) PINS_CUDA(cudaMemcpyAsync(r, ws->rowsum.p, sizeof(double) * pb->m, cudaMemcpyDeviceToDevice, st));
    if (c) PINS_CUDA(cudaMemcpyAsync(c, ws->colsum.p, sizeof(double) * pb->n, cudaMemcpyDeviceToDevice, st));
    PINS_CUDA(cudaStreamSynchronize(st));
    out_host[0] = e.gnorm;
    out_host[1] = e.sumX;
    out_host[2] = e.cost;
    out_host[3] = e.dualP;
    out_host[4] = tau > 0.0 ? (double)ws->nnz : 0.0;
    out_host[5] = e.maxz;
    return PINS_OK;
}

extern "C" int pins_get_csr(pins_workspace *ws, int64_t *rowptr, int32_t *colidx, double *val,
                            int64_t cap, int64_t *nnz_host, int64_t *m_host) {
    PINS_ARG(ws != nullptr && nnz_host && m_host, "pointers");
    PINS_ARG(ws->csr_ready, "no CSR: call pins_evaluate with tau > 0 first");
    PINS_CUDA(cudaDeviceSynchronize());
    *nnz_host = ws->nnz;
    *m_host = ws->m;
    if (rowptr && colidx && val) {
        PINS_ARG(cap >= ws->nnz, "cap < nnz");
        PINS_CUDA(cudaMemcpy(rowptr, ws->rowptr.p, sizeof(int64_t) * (ws->m + 1), cudaMemcpyDeviceToDevice));
        if (ws->nnz) {
            PINS_CUDA(cudaMemcpy(colidx, ws->colidx.p, sizeof(int32_t) * ws->nnz, cudaMemcpyDeviceToDevice));
            PINS_CUDA(cudaMemcpy(val, ws->val.p, sizeof(double) * ws->nnz, cudaMemcpyDeviceToDevice));
        }
    }
    return PINS_OK;
}

extern "C" int pins_sparsify_dense(pins_workspace *ws, int64_t m, int64_t n, const double *P,
                                   int64_t ldp, double tau, int64_t *rowptr, int32_t *colidx,
                                   double *val, int64_t cap, int64_t *nnz_host, void *stream) {
    PINS_ARG(ws && P && nnz_host && m >= 1 && n >= 1 && ldp >= n && tau > 0.0, "arguments");
    PINS_ARG(m < (1LL << 31) && n < (1LL << 31), "m, n < 2^31");
    cudaStream_t st = (cudaStream_t)stream;
    PINS_TRY(ensure(ws->rowcnt, sizeof(int) * m));
    PINS_TRY(ensure(ws->rowptr, sizeof(long long) * (m + 1)));
    const int gw = grid_1d(m * 32, ws->nsm);
    LAUNCH(PINS_PROF_CSR, st, sparsify_count_kernel<<<gw, 256, 0, st>>>(m, n, P, ldp, tau, ptr<int>(ws->rowcnt)));
    LAUNCH(PINS_PROF_CSR, st, scan_counts_kernel<<<1, 1024, 0, st>>>(m, ptr<int>(ws->rowcnt), 1LL << 40,
                                                                    ptr<long long>(ws->rowptr)));
    PINS_CUDA(cudaGetLastError());
    long long *hn = reinterpret_cast<long long *>(ws->h + 48);
    PINS_CUDA(cudaMemcpyAsync(hn, ptr<long long>(ws->rowptr) + m, sizeof(long long), cudaMemcpyDeviceToHost, st));
    PINS_CUDA(cudaStreamSynchronize(st));
    const long long nnz = *hn;
    *nnz_host = nnz;
    // the workspace's rowptr buffer was reused: its evaluation CSR / CSC are stale
    ws->m = m;
    ws->nnz = nnz;
    ws->csc_ready = false;
    ws->csr_ready = false;
    if (!(rowptr && colidx && val)) return PINS_OK;
    PINS_ARG(cap >= nnz, "cap < nnz");
    LAUNCH(PINS_PROF_CSR, st, sparsify_fill_kernel<<<gw, 256, 0, st>>>(m, n, P, ldp, tau, ptr<long long>(ws->rowptr),
                                                                      colidx, val));
    PINS_CUDA(cudaGetLastError());
    PINS_CUDA(cudaMemcpyAsync(rowptr, ws->rowptr.p, sizeof(long long) * (m + 1), cudaMemcpyDeviceToDevice, st));
    PINS_CUDA(cudaStreamSynchronize(st));
    return PINS_OK;
}

extern "C" int pins_cg(pins_workspace *ws, int64_t m, int64_t n, const int64_t *rowptr,
                       const int32_t *colidx, const double *val, int64_t nnz, const double *dr,
                       const double *dc, double mu, const double *rhs, double *x, double rtol,
                       int32_t maxit, int32_t *iters_host, double *relres_host, void *stream) {
    PINS_ARG(ws && rowptr && dr && dc && rhs && x && iters_host && relres_host, "pointers");
    PINS_ARG(m >= 1 && n >= 1 && nnz >= 0 && maxit >= 0, "sizes");
    PINS_ARG(nnz == 0 || (colidx && val), "colidx/val");
    cudaStream_t st = (cudaStream_t)stream;
    const long long *rp = reinterpret_cast<const long long *>(rowptr);
    PINS_TRY(build_csc(ws, m, n, rp, colidx, val, nnz, st));
    PINS_TRY(run_cg(ws, m, n, rp, colidx, val, dr, dc, mu, rhs, x, rtol, maxit, nullptr, nullptr,
                    nullptr, nullptr, st, nnz));
    PINS_CUDA(cudaMemcpyAsync(ws->h + 16, ws->cgst.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    PINS_CUDA(cudaStreamSynchronize(st));
    *iters_host = (int32_t)ws->h[16];
    *relres_host = ws->h[17];
    return PINS_OK;
}

extern "C" int pins_newton_step(pins_workspace *ws, const pins_problem *pb, const pins_params *prm,
                                const double *phi, const double *psi, double s, double *f, double *g,
                                double *info_host, void *stream) {
    PINS_ARG(ws && prm && info_host, "ws, prm, info");
    PINS_TRY(check_problem(pb));
    invalidate_problem(ws);
    PINS_ARG(phi && psi && f && g && s > 0.0, "phi, psi, f, g, s > 0");
    cudaStream_t st = (cudaStream_t)stream;
    const double tau = prm->theta / ((double)pb->m * (double)pb->n);
    EvalOut cur;
    PINS_TRY(run_eval(ws, pb, phi, psi, s, f, g, tau, false, st, &cur));
    return newton_iter(ws, pb, prm, phi, psi, s, f, g, &cur, info_host, st);
}

extern "C" int pins_residuals(pins_workspace *ws, const pins_problem *pb, const double *phi,
                              const double *psi, double s, const double *f, const double *g, double *u,
                              double *v, double *res_host, void *stream) {
    PINS_ARG(ws && res_host, "ws, res");
    PINS_TRY(check_problem(pb));
    invalidate_problem(ws);
    PINS_ARG(phi && psi && f && g && s > 0.0, "phi, psi, f, g, s > 0");
    cudaStream_t st = (cudaStream_t)stream;
    EvalOut e;
    PINS_TRY(run_eval(ws, pb, phi, psi, s, f, g, 0.0, false, st, &e));
    const long long m = pb->m, n = pb->n;
    PINS_TRY(prepare(ws, pb));
    double *uu = u ? u : ptr<double>(ws->uv);
    double *vv = v ? v : ptr<double>(ws->uv) + m;
    LAUNCH(PINS_PROF_VEC, st, lp_duals_kernel<<<grid_1d(m + n, ws->nsm), 256, 0, st>>>(m, n, pb->eta, 1.0 / s, f, g, phi, psi, uu, vv));
    PINS_CUDA(cudaGetLastError());
    LAUNCH(PINS_PROF_REDUCE, st, dots_kernel<<<1, 1024, 0, st>>>(m, n, pb->a, uu, pb->b, vv, ptr<double>(ws->rowsum),
                                    ptr<double>(ws->colsum), ptr<double>(ws->st)));
    PINS_CUDA(cudaMemcpyAsync(ws->h, ws->st.p, 11 * sizeof(double), cudaMemcpyDeviceToHost, st));
    PINS_CUDA(cudaStreamSynchronize(st));
    res_host[0] = e.gnorm;
    res_host[1] = std::max(0.0, pb->eta / s * e.maxz);
    res_host[2] = e.cost;
    res_host[3] = ws->h[8];
    res_host[4] = e.cost - ws->h[8];
    return PINS_OK;
}

extern "C" int pins_lp_certificate(pins_workspace *ws, const pins_problem *pb, const pins_params *prm,
                                   const double *phi, const double *psi, double s, const double *f, const double *g,
                                   double *u, double *v, double *cert_host, void *stream) {
    PINS_ARG(ws && prm && cert_host, "ws, prm, cert");
    PINS_TRY(check_problem(pb));
    invalidate_problem(ws);
    PINS_ARG(phi && psi && f && g && s > 0.0, "phi, psi, f, g, s > 0");
    cudaStream_t st = (cudaStream_t)stream;
    CertOut co;
    PINS_TRY(certify(ws, pb, phi, psi, s, f, g, true, &co, st));
    if (u) PINS_CUDA(cudaMemcpyAsync(u, ws->cbu.p, sizeof(double) * pb->m, cudaMemcpyDeviceToDevice, st));
    if (v) PINS_CUDA(cudaMemcpyAsync(v, ws->cbv.p, sizeof(double) * pb->n, cudaMemcpyDeviceToDevice, st));
    PINS_CUDA(cudaStreamSynchronize(st));
    cert_host[0] = co.primal;
    cert_host[1] = co.pobj;
    cert_host[2] = co.dobj;
    cert_host[3] = co.gap;
    cert_host[4] = co.dual_inf;
    cert_host[5] = (double)co.tree_edges;
    cert_host[6] = (double)co.used_tree;
    cert_host[7] = (double)co.nnz;
    return PINS_OK;
}

extern "C" int pins_plan(const pins_problem *pb, const double *phi, const double *psi, double s,
                         const double *f, const double *g, double *X, int64_t ldx, void *stream) {
    PINS_TRY(check_problem(pb));
    PINS_ARG(phi && psi && f && g && X && ldx >= pb->n && s > 0.0, "pointers / ldx");
    cudaStream_t st = (cudaStream_t)stream;
    // private exp table (same values as the workspace table)
    static DevBuf tab;
    if (!tab.p) {
        ExpTable t;
        for (int j = 0; j < 64; ++j) {
            long double v = exp2l((long double)j / 64.0L);
            t.hi[j] = (double)v;
            t.lo[j] = (double)(v - (long double)t.hi[j]);
        }
        PINS_TRY(ensure(tab, sizeof(ExpTable)));
        PINS_CUDA(cudaMemcpy(tab.p, &t, sizeof t, cudaMemcpyHostToDevice));
    }
    CostDesc cd = make_cd(pb);
    const double inv_eta = 1.0 / pb->eta, w = s * pb->cost_scale / pb->eta;
    const int G = grid_1d(pb->m * pb->n, 148, 16);
    if (pb->cost_kind == 0)
        LAUNCH(PINS_PROF_PLAN, st, plan_kernel<0><<<G, 256, 0, st>>>(pb->m, pb->n, cd, f, phi, g, psi, inv_eta, w, ptr<ExpTable>(tab), X, ldx));
    else if (pb->cost_kind == 1)
        LAUNCH(PINS_PROF_PLAN, st, plan_kernel<1><<<G, 256, 0, st>>>(pb->m, pb->n, cd, f, phi, g, psi, inv_eta, w, ptr<ExpTable>(tab), X, ldx));
    else
        LAUNCH(PINS_PROF_PLAN, st, plan_kernel<2><<<G, 256, 0, st>>>(pb->m, pb->n, cd, f, phi, g, psi, inv_eta, w, ptr<ExpTable>(tab), X, ldx));
    PINS_CUDA(cudaGetLastError());
    return PINS_OK;
}

static int solve_core(pins_workspace *ws, const pins_problem *pb, const pins_params *prm, pins_result *res,
                      void *stream) {
    auto t0 = std::chrono::steady_clock::now();
    cudaStream_t st = (cudaStream_t)stream;
    invalidate_problem(ws);
    ws->x0_enable = true;
    struct Reset {
        pins_workspace *w;
        ~Reset() { w->x0_enable = false; }
    } reset{ws};
    const long long m = pb->m, n = pb->n;
    double *f = res->f, *g = res->g, *phi = res->phi, *psi = res->psi;
    const double tau = prm->theta / ((double)m * (double)n);
    double s = 1.0;
    PINS_TRY(pins_center_init(pb, phi, psi, &s, stream));
    PINS_CUDA(cudaMemsetAsync(f, 0, sizeof(double) * m, st));
    PINS_CUDA(cudaMemsetAsync(g, 0, sizeof(double) * n, st));
    std::vector<double> objs;
    int sweeps = 0, newton_its = 0, cg_its = 0, k = 0;
    bool converged = false;
    EvalOut cur;
    CertOut cert;
    int cert_k = -1, next_cert = 0, n_certs = 0;
    const bool cert_trace = getenv("PINS_CERT_TRACE") != nullptr;
    bool halving_seen = false;
    FILE *trace = nullptr;
    if (const char *tp = getenv("PINS_TRACE")) trace = fopen(tp, "w");
    auto tk0 = std::chrono::steady_clock::now();
    for (k = 0; k < prm->K; ++k) {
        const int cg0 = cg_its;
        if (!prm->warm_start && k > 0) {
            PINS_CUDA(cudaMemsetAsync(f, 0, sizeof(double) * m, st));
            PINS_CUDA(cudaMemsetAsync(g, 0, sizeof(double) * n, st));
        }
        // warm_start 2 (reading R7): start from the linear extrapolation of the last two
        // subproblem solutions; fall back to the plain warm start if that would need Sinkhorn
        const bool extrap = prm->warm_start == 2 && k >= 2;
        if (prm->warm_start == 2) {
            PINS_TRY(ensure(ws->xprev, sizeof(double) * (m + n)));
            PINS_TRY(ensure(ws->xsave, sizeof(double) * (m + n)));
            double *xp = ptr<double>(ws->xprev), *xs = ptr<double>(ws->xsave);
            if (k == 1) {
                PINS_CUDA(cudaMemcpyAsync(xp, f, sizeof(double) * m, cudaMemcpyDeviceToDevice, st));
                PINS_CUDA(cudaMemcpyAsync(xp + m, g, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
            } else if (extrap) {
                LAUNCH(PINS_PROF_VEC, st, extrapolate_kernel<<<grid_1d(m, ws->nsm), 256, 0, st>>>(m, 1.0, 0, f, xp, xs));
                LAUNCH(PINS_PROF_VEC, st, extrapolate_kernel<<<grid_1d(n, ws->nsm), 256, 0, st>>>(n, 1.0, 0, g, xp + m, xs + m));
            }
        }
        PINS_TRY(run_eval(ws, pb, phi, psi, s, f, g, tau, false, st, &cur));
        if (extrap && !(cur.gnorm <= prm->sink_tol)) {
            double *xp = ptr<double>(ws->xprev), *xs = ptr<double>(ws->xsave);
            LAUNCH(PINS_PROF_VEC, st, extrapolate_kernel<<<grid_1d(m, ws->nsm), 256, 0, st>>>(m, 1.0, 1, f, xp, xs));
            LAUNCH(PINS_PROF_VEC, st, extrapolate_kernel<<<grid_1d(n, ws->nsm), 256, 0, st>>>(n, 1.0, 1, g, xp + m, xs + m));
            PINS_TRY(run_eval(ws, pb, phi, psi, s, f, g, tau, false, st, &cur));
        }
        int t = 0;
        if (!(cur.gnorm <= prm->sink_tol) && prm->T1 > 0) {
            PINS_TRY(sinkhorn_phase(ws, pb, prm, phi, psi, s, f, g, cur.gnorm, &t, st));
            PINS_TRY(run_eval(ws, pb, phi, psi, s, f, g, tau, false, st, &cur));
        }
        sweeps += t;
        const double g_sink = cur.gnorm;
        const double nnz0 = (double)ws->nnz;
        int tn = 0;
        while (cur.gnorm > prm->newton_tol && tn < prm->T2) {
            double info[8];
            PINS_TRY(newton_iter(ws, pb, prm, phi, psi, s, f, g, &cur, info, st));
            cg_its += (int)info[3];
            ++tn;
            if (info[2] == 0.0) break;
        }
        newton_its += tn;
        if (trace) {
            auto tk1 = std::chrono::steady_clock::now();
            fprintf(trace, "%d %d %d %d %.0f %.3e %.3e %.17g %.3f\n", k, t, tn, cg_its - cg0, nnz0, g_sink,
                    cur.gnorm, cur.cost, std::chrono::duration<double, std::milli>(tk1 - tk0).count());
            tk0 = tk1;
        }
        if (res->obj_trace_host) res->obj_trace_host[k] = cur.cost;
        objs.push_back(cur.cost);
        res->obj = cur.cost;
        res->kkt = cur.gnorm;
        res->dual_obj = cur.dualP;
        // outer stop (reading R6); rule 3 = certified (reading R11): the LP certificate of
        // X^{k+1} = X~(f, g) is built when the halving estimator first fires and on a
        // geometric schedule, and the solve stops once the primal residual is <= newton_tol
        // and the certified gap <= outer_tol |<C, X>|
        bool stop = false;
        const bool last = k + 1 >= prm->K;
        if (prm->outer_rule == 3) {
            pins_params p1 = *prm;
            p1.outer_rule = 1;
            const bool halving = outer_converged(objs, &p1);
            // first attempt when the halving estimator first fires, then every max(8, k/16)
            const bool trigger = (halving && !halving_seen) || (halving_seen && k + 1 >= next_cert);
            halving_seen = halving_seen || halving;
            if (trigger && cur.gnorm <= prm->newton_tol) {
                const double target = prm->outer_tol * std::fabs(cur.cost);
                PINS_TRY(certify(ws, pb, phi, psi, s, f, g, false, &cert, st, target));
                cert_k = k;
                ++n_certs;
                if (cert_trace)     // dev instrumentation (PINS_CERT_TRACE=1)
                    fprintf(stderr, "cert k %d obj %.17g dobj %.17g relgap %.3e primal %.3e tree %d comps %d "
                            "repairs %d viol %d used_tree %d nnz %lld\n",
                            k, cert.pobj, cert.dobj, cert.gap / std::fabs(cert.pobj), cert.primal, cert.tree_edges,
                            cert.components, cert.repairs, cert.violations, cert.used_tree, cert.nnz);
                if (cert.gap <= target) stop = true;
                else next_cert = k + 1 + std::max(8, (k + 1) / 16);
            }
        } else {
            stop = outer_converged(objs, prm);
        }
        if ((stop || last) && cert_k != k) {        // the returned plan's certificate (report)
            PINS_TRY(certify(ws, pb, phi, psi, s, f, g, false, &cert, st));
            cert_k = k;
            ++n_certs;
        }
        if (stop || last) PINS_TRY(measure_dual_inf(ws, pb, &cert, st));
        // X^{k+1} = X~(f, g): centre update (Alg. 2 line 16), then C^{k+1} (line 3)
        PINS_TRY(pins_center_update(pb, phi, psi, &s, f, g, stream));
        if (stop) {
            converged = true;
            ++k;
            break;
        }
    }
    if (trace) fclose(trace);
    if (k > prm->K) k = prm->K;
    // certified LP duals of the returned plan X^K (reading R11): dual feasible by
    // construction; lp_dual_obj <= LP* and gap = <C, X^K> - lp_dual_obj
    if (res->u) PINS_CUDA(cudaMemcpyAsync(res->u, ws->cbu.p, sizeof(double) * m, cudaMemcpyDeviceToDevice, st));
    if (res->v) PINS_CUDA(cudaMemcpyAsync(res->v, ws->cbv.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    res->lp_dual_obj = cert.dobj;
    res->gap = cert.gap;
    res->dual_inf = cert.dual_inf;
    res->certificates = n_certs;
    res->cert_tree = cert.used_tree;
    res->s = s;
    res->outer_iters = k;
    res->sweeps = sweeps;
    res->newton_iters = newton_its;
    res->cg_iters = cg_its;
    res->status = converged ? 0 : 1;
    if (getenv("PINS_SKIP_STATS") && ws->skipk && ws->skst.p) {   // dev instrumentation
        int h[64];
        PINS_CUDA(cudaMemcpyAsync(h, ws->skst.p, sizeof h, cudaMemcpyDeviceToHost, st));
        PINS_CUDA(cudaStreamSynchronize(st));
        const char *nm[4] = {"lse-row", "lse-col", "sum-row", "sum-col"};
        for (int q = 0; q < 4; ++q) {
            unsigned long long a2, b2;
            memcpy(&a2, h + 16 * q + 6, 8);
            memcpy(&b2, h + 16 * q + 8, 8);
            fprintf(stderr, "chunk skip %s: %llu of %llu tested chunks skipped (%.1f %%)\n", nm[q], a2, b2,
                    b2 ? 100.0 * (double)a2 / (double)b2 : 0.0);
        }
    }
    res->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return PINS_OK;
}

extern "C" int pins_solve_host(const pins_problem *pb_host, const pins_params *prm, pins_result *res_host,
                               int64_t *io_bytes_host, void *stream) {
    PINS_TRY(check_problem(pb_host));
    PINS_ARG(prm && res_host && io_bytes_host, "params / result / io_bytes");
    cudaStream_t st = (cudaStream_t)stream;
    const long long m = pb_host->m, n = pb_host->n;
    pins_problem pb = *pb_host;
    // one stream-ordered allocation for inputs and outputs
    const bool dense = pb_host->cost_kind == PINS_COST_DENSE;
    const long long nC = dense ? m * pb_host->ldc : 0;
    const long long nx = dense ? 0 : m * (long long)pb_host->d, ny = dense ? 0 : n * (long long)pb_host->d;
    const long long in_elems = nC + nx + ny + m + n;
    const long long out_elems = 3 * (m + n);     // f g phi psi u v
    double *buf = nullptr;
    PINS_CUDA(cudaMallocAsync((void **)&buf, sizeof(double) * (in_elems + out_elems), st));
    double *p = buf;
    long long h2d = 0, d2h = 0;
    auto up = [&](const double *src, long long cnt) -> double * {
        double *dst = p;
        p += cnt;
        if (cnt) cudaMemcpyAsync(dst, src, sizeof(double) * cnt, cudaMemcpyHostToDevice, st);
        h2d += sizeof(double) * cnt;
        return dst;
    };
    if (dense) pb.C = up(pb_host->C, nC);
    else {
        pb.x = up(pb_host->x, nx);
        pb.y = up(pb_host->y, ny);
    }
    pb.a = up(pb_host->a, m);
    pb.b = up(pb_host->b, n);
    PINS_CUDA(cudaGetLastError());
    pins_result r = *res_host;
    r.f = p; r.g = p + m; r.phi = p + m + n; r.psi = p + 2 * m + n; r.u = p + 2 * (m + n); r.v = p + 3 * m + 2 * n;
    int rc = pins_solve(&pb, prm, &r, stream);
    if (rc == PINS_OK) {
        double *const srcs[6] = {r.f, r.g, r.phi, r.psi, r.u, r.v};
        double *const dsts[6] = {res_host->f, res_host->g, res_host->phi, res_host->psi, res_host->u, res_host->v};
        const long long cnts[6] = {m, n, m, n, m, n};
        for (int q = 0; q < 6; ++q) {
            if (!dsts[q]) continue;
            cudaMemcpyAsync(dsts[q], srcs[q], sizeof(double) * cnts[q], cudaMemcpyDeviceToHost, st);
            d2h += sizeof(double) * cnts[q];
        }
        double *const keep[6] = {res_host->f, res_host->g, res_host->phi, res_host->psi, res_host->u, res_host->v};
        *res_host = r;
        res_host->f = keep[0]; res_host->g = keep[1]; res_host->phi = keep[2];
        res_host->psi = keep[3]; res_host->u = keep[4]; res_host->v = keep[5];
    }
    cudaFreeAsync(buf, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (rc != PINS_OK) return rc;
    PINS_CUDA(e);
    io_bytes_host[0] = h2d;
    io_bytes_host[1] = d2h;
    return PINS_OK;
}

// Morton permutation of one point set (pins_order.cuh): perm (device, np)
static int morton_order(long long np, int d, const double *pts, const double *lohi, int *perm, DevBuf &tmp,
                        cudaStream_t st) {
    PINS_TRY(ensure(tmp, sizeof(unsigned long long) * 2 * np + sizeof(int) * np));
    unsigned long long *k0 = ptr<unsigned long long>(tmp), *k1 = k0 + np;
    int *i0 = reinterpret_cast<int *>(k1 + np);
    LAUNCH(PINS_PROF_VEC, st, morton_kernel<<<grid_1d(np, 148), 256, 0, st>>>(np, d, pts, lohi, k0, i0));
    PINS_CUDA(cudaGetLastError());
    size_t tb = 0;
    PINS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, i0, perm, (int)np, 0, 64, st));
    DevBuf sortmp;
    PINS_TRY(ensure(sortmp, tb));
    PINS_CUDA(cub::DeviceRadixSort::SortPairs(sortmp.p, tb, k0, k1, i0, perm, (int)np, 0, 64, st));
    PINS_CUDA(cudaStreamSynchronize(st));
    return PINS_OK;
}

static int solve_entry(pins_workspace *ws, const pins_problem *pb, const pins_params *prm, pins_result *res,
                       void *stream) {
    PINS_TRY(check_problem(pb));
    PINS_ARG(prm && res && res->f && res->g && res->phi && res->psi, "params / result buffers");
    PINS_ARG(prm->K >= 1 && prm->T2 >= 0 && prm->T1 >= 0, "budgets");
    PINS_ARG(prm->outer_rule >= 0 && prm->outer_rule <= 3, "outer_rule in 0..3");
    auto t0 = std::chrono::steady_clock::now();
    cudaStream_t st = (cudaStream_t)stream;
    const long long m = pb->m, n = pb->n;
    const bool reorder = pb->cost_kind != PINS_COST_DENSE && (double)m * (double)n >= 65536.0 &&
                         getenv("PINS_NO_REORDER") == nullptr;
    if (!reorder) {
        int rc = solve_core(ws, pb, prm, res, stream);
        res->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return rc;
    }
    // permuted copy of the instance (points in Morton order), solve, scatter back
    const int d = pb->d;
    DevBuf buf, lohi, tmp;
    const long long nd = (long long)(m + n) * d + (m + n) + 6 * (m + n);
    PINS_TRY(ensure(buf, sizeof(double) * nd + sizeof(int) * (m + n)));
    PINS_TRY(ensure(lohi, sizeof(double) * 32));
    double *xp = ptr<double>(buf), *yp = xp + m * d, *ap = yp + n * d, *bp = ap + m;
    double *o = bp + n;                       // 6 (m+n) result slots
    int *px = reinterpret_cast<int *>(o + 6 * (m + n)), *py = px + m;
    LAUNCH(PINS_PROF_VEC, st, bbox_kernel<<<1, 1024, 0, st>>>(m, n, d, pb->x, pb->y, ptr<double>(lohi)));
    PINS_CUDA(cudaGetLastError());
    PINS_TRY(morton_order(m, d, pb->x, ptr<double>(lohi), px, tmp, st));
    PINS_TRY(morton_order(n, d, pb->y, ptr<double>(lohi), py, tmp, st));
    LAUNCH(PINS_PROF_VEC, st, gather_points_kernel<<<grid_1d(m, 148), 256, 0, st>>>(m, d, px, pb->x, pb->a, xp, ap));
    LAUNCH(PINS_PROF_VEC, st, gather_points_kernel<<<grid_1d(n, 148), 256, 0, st>>>(n, d, py, pb->y, pb->b, yp, bp));
    PINS_CUDA(cudaGetLastError());
    pins_problem q = *pb;
    q.x = xp; q.y = yp; q.a = ap; q.b = bp;
    pins_result r = *res;
    r.f = o; r.g = o + m; r.phi = o + (m + n); r.psi = o + (m + n) + m;
    r.u = res->u ? o + 2 * (m + n) : nullptr;
    r.v = res->v ? o + 2 * (m + n) + m : nullptr;
    PINS_TRY(solve_core(ws, &q, prm, &r, stream));
    double *const src[6] = {r.f, r.g, r.phi, r.psi, r.u, r.v};
    double *const dst[6] = {res->f, res->g, res->phi, res->psi, res->u, res->v};
    for (int t = 0; t < 6; ++t) {
        if (!src[t] || !dst[t]) continue;
        const bool rows = (t % 2) == 0;
        LAUNCH(PINS_PROF_VEC, st, scatter_kernel<<<grid_1d(rows ? m : n, 148), 256, 0, st>>>(
            rows ? m : n, rows ? px : py, src[t], dst[t]));
    }
    PINS_CUDA(cudaGetLastError());
    PINS_CUDA(cudaStreamSynchronize(st));
    double *const keep[6] = {res->f, res->g, res->phi, res->psi, res->u, res->v};
    *res = r;
    res->f = keep[0]; res->g = keep[1]; res->phi = keep[2]; res->psi = keep[3]; res->u = keep[4]; res->v = keep[5];
    res->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return PINS_OK;
}

extern "C" int pins_solve_ws(pins_workspace *ws, const pins_problem *pb, const pins_params *prm, pins_result *res,
                             void *stream) {
    PINS_ARG(ws != nullptr, "ws");
    return solve_entry(ws, pb, prm, res, stream);
}

extern "C" int pins_solve(const pins_problem *pb, const pins_params *prm, pins_result *res, void *stream) {
    pins_workspace *ws = nullptr;
    PINS_TRY(pins_workspace_create(&ws));
    const int rc = solve_entry(ws, pb, prm, res, stream);
    pins_workspace_destroy(ws);
    return rc;
}
