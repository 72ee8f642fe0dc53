// pins_pass.cuh -- the dense passes over the m x n plan block, v2 (sm_100a).
//
// One CUDA thread owns one row of the pass ("pass rows"), 128 rows per CTA,
// and streams over a contiguous column range (one of S column splits) in
// chunks of kCC columns staged in shared memory (column potentials, column
// points).  The same kernels run in both orientations: the row orientation
// (pass rows = the m rows of X, pass columns = the n columns) and the column
// orientation (roles swapped: x <-> y, f/phi <-> g/psi, a <-> b); the host
// fills a PassSide per orientation.
//
//  * lse_pass_kernel  -- Sinkhorn half-sweep, Alg. 2 line 5 (row orientation)
//    or line 6 (column orientation):  f_i <- eta(log a_i + 1) - phi_i
//    - eta LSE_j(Q_j - w D_ij),  Q_j = (g_j + psi_j)/eta,  w = s*scale/eta.
//    It also returns the residual ||a - X~ e||_1 of the iterate it starts
//    from (the row sums are exp(P_i + LSE_i)), which is how a sweep and its
//    stopping test share one read of the cost.
//  * sum_pass_kernel  -- evaluation of X~ of Eq. (7) in BOTH orientations in
//    one launch: row sums / column sums (gradient, Eq. (9)), <C, X~>, the
//    line-search trial sum (reading R4), and the sparsified plan block
//    (entries >= tau, reading R3) compacted per (row, split) -- row
//    orientation -> CSR, column orientation -> CSC, with bit-identical values.
//
// Negligible entries are skipped without evaluating the exponential (the
// plan of Eq. (7) is concentrated: Thm 4.3): in the LSE a
// term is skipped when x < M_lo - kLseCut, where M_lo is a running lower
// bound of the row maximum (seeded with the previous pass's argmax column),
// so each skipped term is < e^-36 of the largest; in the sums an entry is
// skipped when z < -kSumCut (X~ < 1.8e-35).  DESIGN.md §5 bounds the effect.
//
// Reductions are deterministic: per (split, row) partials, merged in split
// order by the last CTA of each row block (atomic ticket), then per-block
// scalars merged in block order by the last row block of the launch.
#pragma once
#include <cuda.h>

#include "pins_device.cuh"
#include "pins_tc.cuh"

#include <type_traits>

namespace pins {

constexpr int kPT = 128;            // threads per CTA = pass rows per CTA
constexpr int kCC = 32;             // columns per staged chunk
constexpr double kLseCut = 36.0;
constexpr double kSumCut = 80.0;

// cost evaluation variants (host picks, see pins_api.cu choose_cost)
enum : int {
    PC_DENSE_ROW = 0,   // dense C, row orientation: tile staged through smem
    PC_DENSE_COL = 1,   // dense C, column orientation: C[i*ldc + j] read directly (coalesced)
    PC_SQ32 = 2,        // integer points, exact in fp32: D = |x|^2 + |y|^2 - 2 x.y
    PC_L132 = 3,        // integer points, exact in fp32: D = sum |x - y|
    PC_SQ64 = 4,        // generic points, fp64: D = sum (x - y)^2
    PC_L164 = 5,        // generic points, fp64: D = sum |x - y|
    PC_SQTC = 6,        // integer points |x| <= 2048: x.y on the tensor cores (tcgen05, fp16 exact)
    PC_DENSE_ROW_T = 7, // dense C, row orientation: 128 x 32 tiles staged by TMA (SWIZZLE_128B)
    PC_DENSE_COL_T = 8, // dense C, column orientation: 32 x 128 tiles staged by TMA
};

// TMA staging of dense C (PC_DENSE_*_T): a ring of kNSt tiles of kTileB bytes in
// dynamic shared memory, one mbarrier per stage (pins_api.cu builds the tensor
// maps: row orientation boxes of {16 columns, 128 rows} with the 128-byte swizzle,
// so thread = row reads its 32 columns without bank conflicts; column orientation
// one box of {128 columns, 32 rows}, thread = column).
template <int COST>
constexpr bool kTma = COST == PC_DENSE_ROW_T || COST == PC_DENSE_COL_T;
constexpr int kNSt = 2;                      // ring stages
constexpr int kTileB = kCC * kPT * 8;        // 32 KB per stage
constexpr int kTmaSmem = kNSt * kTileB + 1024;   // + alignment slack (SWIZZLE_128B: 1024 B)

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *tm, int x, int y, uint64_t *mbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
        ::"r"(tc::smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(tc::smem_u32(mbar))
        : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(tc::smem_u32(mbar)), "r"(bytes)
                 : "memory");
}

// per-CTA TMA ring state
struct TmaRing {
    unsigned char *base;                     // 1024-aligned ring in dynamic shared memory
    uint64_t *full;                          // [kNSt] mbarriers (static shared memory)
    const CUtensorMap *tm;                   // the orientation's tensor map (kernel parameter)
    int x0;                                  // row orientation: unused; column orientation: first C column
    int y0;                                  // row orientation: first C row; column orientation: unused
};

// thread 0: load chunk c (columns jb + c kCC of the pass) into stage c % kNSt
template <int COST>
__device__ __forceinline__ void tma_issue(const TmaRing &R, long long jb, long long c) {
    const int s = (int)(c % kNSt);
    unsigned char *dst = R.base + s * kTileB;
    const int p = (int)(jb + c * kCC);      // first pass column of the chunk
    mbar_expect_tx(&R.full[s], kTileB);
    if constexpr (COST == PC_DENSE_ROW_T) {  // C rows y0.., columns p..p+31: two 16-column boxes
        tma_load_2d(dst, R.tm, p, R.y0, &R.full[s]);
        tma_load_2d(dst + kTileB / 2, R.tm, p + 16, R.y0, &R.full[s]);
    } else {                                 // C rows p..p+31, columns x0..x0+127
        tma_load_2d(dst, R.tm, R.x0, p, &R.full[s]);
    }
}

struct PassSide {
    long long M, N;                 // pass rows / pass columns
    int S, RB;                      // column splits, row blocks (RB = ceil(M / kPT))
    int dp;                         // padded point dimension (multiple of 4), points kinds
    // cost
    const double *C;                // dense: the caller's C (row-major m x n, ldc)
    long long ldc;
    const float *xr32, *yc32;       // fp32 points, M x dp / N x dp (zero padded)
    const float *nxr, *nyc;         // squared norms (PC_SQ32)
    const double *xr64, *yc64;      // fp64 points, M x dp / N x dp (zero padded)
    const __half *xrh, *ych;        // PC_SQTC: fp16 points, M x 16 / N x 16 (zero padded)
    // tile skipping (exact-fp32 point costs): bounding boxes [lo[dp], hi[dp]] of the
    // pass rows per row block (kPT rows) and of the pass columns per group of kCC
    // chunk skipping by drift certificates (SkipCtx; exact-fp32 point costs only)
    int skipk;                      // 0 off, 1 on
    int cps;                        // chunks per split (upper bound)
    float *gam;                     // [RB * S * cps * 4]: certificate per (row block, split, chunk, warp)
    float *gamD;                    // [RB * S * cps * 4]: min distance Df over the same (warp rows, chunk)
    float *tref;                    // [M]: reference-pass row thresholds
    float *qref;                    // [N]: reference-pass skip-test column values
    int *skst;                      // [0] age (< 0: next pass records), [1] skipped, [2] chunks,
                                    // [3] w_lo of the reference (float bits), [4] best skip fraction (ppm),
                                    // [5] passes left switched off, [6..9] totals skipped / chunks (u64, stats)
    // potentials: pass-row side (fr + phir), pass-column side (gc + psic)
    const double *fr, *phir, *gc, *psic;
    int m1_row;                     // SUM: the "-1" of Eq. (7) sits on the pass-row potential
    const double *ar;               // pass-row marginal
    // LSE outputs
    double *fout;                   // new pass-row potential (may alias fr)
    double *fsave;                  // LSE: copy of the old pass-row potential (rollback)
    int *jstar;                     // pass-row argmax column, in/out (-1 = unknown)
    // SUM outputs
    double *sum, *grad;             // pass-row sums, ar - sum
    const double *eu, *ev;          // trial factors (pass-row / pass-column), or NULL
    const double *bu, *bv;          // trial skip bumps >= 0 (pass-row / pass-column)
    int want_cx;                    // accumulate sum X D
    double tau;                     // sparsify threshold (0: off)
    long long cap;                  // per (row, split) buffer capacity
    int *cnt;                       // [M * S] counts (row-major: row, split)
    int *bcol;                      // [M * S * cap]
    double *bval;
    // partials
    double *pa, *pb;                // [S * M]: LSE (max, sum) / SUM (sum, -)
    double *psc;                    // SUM: [S * RB * 4] split-level scalars
    int *pj;                        // [S * M]: LSE split argmax
    double *blk;                    // [RB * 8] per row block scalars
    long long *blkoff;              // SUM: [RB + 1] exclusive scan of the block nnz totals
    unsigned *ticket;               // [RB]
    // Certified candidate lists of the Sinkhorn phase (LSE only; see lse_sparse_kernel).
    // Unit u = sp * M + i is (split sp, pass row i); its list holds, in column order, the
    // entries with test value v > lB[i] at the last record pass, unit-major at u * lcap.
    int lori;                       // orientation (0 rows, 1 columns): index into lctl
    int lrec;                       // dense pass: record the lists (conditional on lctl[lori])
    int lcap;                       // capacity per unit
    int *lcnt;                      // [S * M] entries per unit, -1 = overflow
    int *lj;                        // [S * M * lcap] columns
    void *lD;                       // [S * M * lcap] distances: float (exact-fp32 costs) or double
    float *lB;                      // [M] the record pass's list bound lB_i = thr0_i - margin
    float *lqref;                   // [N] the record pass's column test values qs_j
    const double *lqv;              // [N] sparse pass: column values q_j (written by the other side)
    const float *lqsv;              // [N] sparse pass: qs_of(q_j)
    const float *ldqs;              // [S] sparse pass: per split max_j (qs_j - lqref_j) since the record
    int *lperm;                     // [S * M] units by decreasing list length (after each record)
    int *lq;                        // [S * M] units whose certificate failed (fallback queue)
    int lstage;                     // sparse pass: the split's column values staged in shared memory
    // Absorbed kernel-matrix sweeps (lse_ksweep_kernel): the lists as a sliced-ELL matrix
    // K_ij = exp(x_ij(record) - r_u) per warp tile of 32 sorted ranks, tiles packed densely
    // in (split, rank) order (a sparse layout would touch every 2 MB page of the arrays)
    double *lqd;                    // [N] the record pass's column values q_j in fp64 (NULL: not kept)
    int *ellj;                      // [S * Mpad * lcap] column index inside the split (j - jb)
    double *ellK;                   // [S * Mpad * lcap] kernel values
    long long Mpad;                 // M rounded up to whole warp tiles
    int *ellL;                      // [S * Mpad / 32] k-steps stored per tile (a multiple of kKB)
    int *ellrel;                    // [S * Mpad / 32] first stage of the tile inside its split's block
    int *ellabs;                    // [S * Mpad / 32] first stage of the tile (tiles are packed densely:
                                    // entry k of lane l at (ellabs * kKB + k) * 32 + l)
    int *elltot;                    // [S] stages per split
    void *lunit;                    // [S * Mpad] KUnit per sorted rank: what a half-sweep needs of its unit
    // finalize: this side's new potentials are the other side's column values
    double *oqv;                    // [M] q of the other orientation, or NULL
    float *oqsv;                    // [M]
    const float *oqref;             // [M] the other side's lqref
    float *odqc;                    // [M / kCC + 1] scratch: per chunk drift of the other side's columns
    float *odqs;                    // [oS] the other side's ldqs
    int oS;                         // the other side's splits
    int *lctl;                      // [0..1] rebuild requested per side, [2..3] launch index of the
                                    // last record per side, [4] overflows, [5] max count, [6..7]
                                    // fallback units (stats), [8] fallback queue length, [12..13]
                                    // record passes (stats)
};

struct PassArgs {
    PassSide side[2];
    int nsides;
    int G0;                         // CTAs of side 0 (= S0 * RB0)
    int cost[2];                    // PC_* per side
    double eta, inv_eta, w;
    const ExpTable *tab;
    unsigned *gticket;              // launch-level ticket
    double *st;                     // launch stats (see finalize)
    const double *sink_tol;         // LSE: device copy of the tolerance, may be NULL
    int *ctl;                       // LSE control: [0] done flag, [1] sweeps done, [2] rollback
    int check_done;                 // LSE: exit immediately when ctl[0] is set
    int count_surv;                 // profiling: add the entries evaluated in phase 2 to g_surv
    int count_sweep;                // LSE col pass: ++ctl[1]
    int test_tol;                   // LSE row pass: set done (and rollback) when res <= tol
    const double *a_dot, *f_dot, *b_dot, *g_dot;   // SUM: <a,f> + <b,g> (global finalize)
    int lnosort;                    // candidate lists: keep the units in row order (experiments)
    int lt;                         // candidate lists: launch index of this half-sweep
    double lmargin;                 // candidate lists: record margin below the threshold
};

// candidate-list distance storage: the exact fp32 distance where phase 1 keeps one, else fp64
template <int COST>
using LDT = typename std::conditional<COST == PC_SQTC || COST == PC_SQ32 || COST == PC_L132, float, double>::type;

// Column range of split sp of S: whole kCC-column chunks (so every chunk starts at
// a multiple of kCC -- TMA box origins stay 256-byte aligned), the last split
// ending at N.
__device__ __forceinline__ void split_range(long long N, int S, int sp, long long &jb, long long &je) {
    const long long nch = (N + kCC - 1) / kCC;
    jb = kCC * (nch * sp / S);
    je = min(N, kCC * (nch * (sp + 1) / S));
}

// Profiling counters (pins_prof_read_work): entries evaluated in phase 2 (the
// survivors of the skip test), [0] half-sweeps, [1] sum passes.
__device__ unsigned long long g_surv[3];

__device__ __forceinline__ void count_survivors(int on, int slot, int nsurv) {
    if (!on) return;
    unsigned long long v = (unsigned long long)nsurv;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(g_surv + slot, v);
}

// Conservative fp32 form of the skip test  x = q - w D > thr  (phase 1 of a chunk):
// qs = q rounded up by 2^-20 |q|, w_lo = w (1 - 2^-19), thr_lo = thr - 2^-20 |thr|;
// fmaf(-w_lo, D, qs) > thr_lo holds whenever the fp64 test does (the margins cover
// every fp32 rounding), so no entry the fp64 test keeps is skipped (R10).
__device__ __forceinline__ float qs_of(double q) {
    return q == -INFINITY ? -INFINITY : (float)(q + fabs(q) * 0x1p-20);
}
// the spacing of floats at |x| (an upper bound of the rounding error of a value near x)
__device__ __forceinline__ float ulpf_of(float x) {
    const float a = fabsf(x);
    return a == INFINITY ? INFINITY : nextafterf(a, INFINITY) - a;
}
__device__ __forceinline__ float thr_lo_of(double t) { return (float)(t - fabs(t) * 0x1p-20 - 0x1p-30); }

// exact potential expressions (no FMA contraction: identical bits in both orientations)
__device__ __forceinline__ double pot_q(double g, double psi, double inv_eta) {
    return __dmul_rn(__dadd_rn(g, psi), inv_eta);
}
__device__ __forceinline__ double pot_p(double f, double phi, double inv_eta) {
    return __dsub_rn(__dmul_rn(__dadd_rn(f, phi), inv_eta), 1.0);
}

// ---------------------------------------------------------------- staging
// Chunks of kCC pass columns, double-buffered in shared memory (single-buffered
// for the dense row orientation, whose 128 x kCC tile is large).  Each thread
// prefetches its share of chunk c+2 into registers while chunk c is computed
// (Pref), and stores it into the free buffer at the next chunk boundary.
template <int COST, int DP>
struct Buf {
    static constexpr bool PTS32 = COST == PC_SQ32 || COST == PC_L132;
    static constexpr bool PTS64 = COST == PC_SQ64 || COST == PC_L164;
    double q[kCC];                               // column potential
    double qt[kCC];                              // skip-test column value (q + trial bump)
    double ev[kCC];                              // trial factor
    alignas(16) float qs[kCC];                   // fp32 skip-test value: qt rounded up by 2^-20 |qt|
    alignas(16) float ny[kCC];
    alignas(16) float y32[PTS32 ? kCC * DP : 4];
    double y64[PTS64 ? kCC * DP : 1];
    alignas(128) unsigned char yh[COST == PC_SQTC ? kCC * 32 : 16];   // UMMA B tile (kCC x 16 fp16)
    double tile[COST == PC_DENSE_ROW ? kCC * (kPT + 1) : 1];
};

template <int COST>
constexpr int kNBuf = COST == PC_DENSE_ROW ? 1 : 2;   // (the TMA ring stages dense C separately)

// Whole-chunk skip by drift certificates (R10, tile form).  An entry passes the
// per-entry fp32 test iff fl(qs_j - w_lo Df_ij) > thr32_i, i.e. (fl monotone,
// thr32 representable) only if the real value qs_j - w_lo Df_ij > thr32_i.  With
// integer points Df_ij is exact and the same in every pass.  A reference pass
// records, per (row block, split, chunk), gamma >= max_i (max_j v_ij + |v| 2^-22
// - T_i) with v the fp32 test values, T_i = the row's threshold then, and qref_j =
// the column values then, and Dmin = min Df_ij over the same tile.  In a later
// pass with w_lo >= w_lo(ref), dw = w_lo - w_lo(ref) >= 0,
//     qs_j - w_lo Df_ij = v_ij(real) + (qs_j - qref_j) - dw Df_ij
//                      <= gamma + T_i + max_j (qs_j - qref_j) - dw Dmin,
// so if  gamma - dw Dmin + max_j (qs_j - qref_j) <= min_i (thr32_i - T_i)  no entry
// of the chunk can pass and the chunk is skipped: results are bit-identical with
// and without skipping.  (The dw Dmin term matters across EPPA iterations: w grows
// with s_k, and the column values drift up by about as much as w D grows.)  The potentials drift slowly between passes, so certificates
// stay valid for many passes; a pass records fresh ones when the skip fraction
// falls (skip_switch).
struct SkipCtx {
    int kind;                   // 0 off, 1 test certificates, 2 record (reference pass)
    double dthr;                // kind 1: min over the CTA's rows of thr32_i - T_i (rounded down)
    long long jb;               // the CTA's first column
    float *gcta;                // the CTA's certificates [cps * 4]
    float *gDcta;               // the CTA's tile minimum distances [cps * 4]
    double dw;                  // kind 1: w_lo - w_lo(reference) >= 0
    float *qref;
    bool wq;                    // kind 2: this CTA writes qref (row block 0)
};

template <int COST, int DP>
struct Pref {
    static constexpr bool PTS32 = COST == PC_SQ32 || COST == PC_L132;
    static constexpr bool PTS64 = COST == PC_SQ64 || COST == PC_L164;
    static constexpr int NY = (PTS32 || PTS64) ? (kCC * DP + kPT - 1) / kPT : 1;
    double g, psi, ev, bv;
    float ny;
    float y32[PTS32 ? NY : 1];
    double y64[PTS64 ? NY : 1];
    uint2 yh;
    // global -> registers (this thread's share of columns j0 .. j0+nc-1)
    __device__ __forceinline__ void load(const PassSide &P, long long j0, int nc, bool trial, const SkipCtx &sk) {
        const int tid = threadIdx.x;
        if (tid < kCC) {
            const bool ok = tid < nc;
            g = ok ? P.gc[j0 + tid] : 0.0;
            psi = ok ? P.psic[j0 + tid] : 0.0;
        } else if (tid < 2 * kCC && trial) {
            const int c = tid - kCC;
            const bool ok = c < nc;
            ev = ok ? P.ev[j0 + c] : 0.0;
            bv = ok ? P.bv[j0 + c] : 0.0;
        }
        if (COST == PC_SQ32 && tid >= 2 * kCC && tid < 3 * kCC) {
            const int c = tid - 2 * kCC;
            ny = c < nc ? P.nyc[j0 + c] : 0.f;
        }
        if constexpr (PTS32) {
#pragma unroll
            for (int q = 0; q < NY; ++q) {
                const int t = tid + q * kPT;
                const int c = t / DP;
                y32[q] = (t < kCC * DP && c < nc) ? P.yc32[(j0 + c) * DP + (t - c * DP)] : 0.f;
            }
        } else if constexpr (PTS64) {
#pragma unroll
            for (int q = 0; q < NY; ++q) {
                const int t = tid + q * kPT;
                const int c = t / DP;
                y64[q] = (t < kCC * DP && c < nc) ? P.yc64[(j0 + c) * DP + (t - c * DP)] : 0.0;
            }
        } else if constexpr (COST == PC_SQTC) {
            const int c = tid >> 2, kq = (tid & 3) * 4;     // 4 fp16 of column c per thread
            yh = (c < nc) ? *reinterpret_cast<const uint2 *>(P.ych + (j0 + c) * 16 + kq) : make_uint2(0u, 0u);
            if (tid >= 2 * kCC && tid < 3 * kCC) {
                const int cc = tid - 2 * kCC;
                ny = cc < nc ? P.nyc[j0 + cc] : 0.f;
            }
        }
    }
    // owner warp, reference pass: record the chunk's column values
    __device__ __forceinline__ void decide(Buf<COST, DP> &B, const SkipCtx &sk, float qs, long long j0,
                                           int nc) const {
        const int lane = threadIdx.x & 31;
        if (sk.kind == 2 && sk.wq && lane < nc) sk.qref[j0 + lane] = qs;
    }
    // registers -> shared buffer.  qmode: 0 q = (g+psi)/eta, 1 q = (g+psi)/eta - 1
    __device__ __forceinline__ void store(Buf<COST, DP> &B, const PassSide &P, long long i0, long long j0, int nc,
                                          double inv_eta, int qmode, bool trial, const SkipCtx &sk) {
        const int tid = threadIdx.x;
        if (tid < kCC) {
            double q = -INFINITY;
            if (tid < nc) q = qmode ? pot_p(g, psi, inv_eta) : pot_q(g, psi, inv_eta);
            B.q[tid] = q;
            if (!trial) {
                const float qs = qs_of(q);
                B.qt[tid] = q;
                B.qs[tid] = qs;
                decide(B, sk, qs, j0, nc);
            }
        } else if (tid < 2 * kCC && trial) {
            B.ev[tid - kCC] = ev;
        }
        if (COST == PC_SQ32 || COST == PC_SQTC)
            if (tid >= 2 * kCC && tid < 3 * kCC) B.ny[tid - 2 * kCC] = ny;
        if constexpr (PTS32) {
#pragma unroll
            for (int q = 0; q < NY; ++q) {
                const int t = tid + q * kPT;
                if (t < kCC * DP) B.y32[t] = y32[q];
            }
        } else if constexpr (PTS64) {
#pragma unroll
            for (int q = 0; q < NY; ++q) {
                const int t = tid + q * kPT;
                if (t < kCC * DP) B.y64[t] = y64[q];
            }
        } else if constexpr (COST == PC_SQTC) {
            const int c = tid >> 2, kq = (tid & 3) * 4;
            *reinterpret_cast<uint2 *>(B.yh + tc::kmajor_off(c, kq)) = yh;
        } else if constexpr (COST == PC_DENSE_ROW) {
            // rows i0 .. i0+kPT-1 of C, columns j0 .. j0+kCC-1: warp w loads rows w, w+4, ...;
            // lane = column (coalesced 256 B per row); stored transposed with a pad column
            const int lane = tid & 31, warp = tid >> 5;
            const long long rows = P.M - i0;
            for (int r = warp; r < kPT; r += kPT / 32) {
                double v = 0.0;
                if (r < rows && lane < nc) v = __ldg(P.C + (i0 + r) * P.ldc + j0 + lane);
                B.tile[lane * (kPT + 1) + r] = v;
            }
        }
    }
    // trial: the skip-test value q + bv needs q, written by threads < kCC
    __device__ __forceinline__ void store_trial_qt(Buf<COST, DP> &B, const SkipCtx &sk, long long j0, int nc) {
        const int tid = threadIdx.x;
        if (tid >= kCC && tid < 2 * kCC) {
            const int c = tid - kCC;
            const double qt = B.q[c] + bv;
            const float qs = qs_of(qt);
            B.qt[c] = qt;
            B.qs[c] = qs;
            decide(B, sk, qs, j0, nc);
        }
    }
};

// distance of the thread's pass row to staged column c (as fp64)
template <int COST, int DP>
struct RowPt {
    float x32[DP > 0 ? DP : 1];
    float nx;
    double x64[DP > 0 ? DP : 1];
    __device__ __forceinline__ void load(const PassSide &P, long long i, bool valid) {
        if constexpr (COST == PC_SQ32 || COST == PC_L132 || COST == PC_SQTC) {
#pragma unroll
            for (int k = 0; k < DP; ++k) x32[k] = valid ? P.xr32[i * DP + k] : 0.f;
            nx = ((COST == PC_SQ32 || COST == PC_SQTC) && valid) ? P.nxr[i] : 0.f;
        } else if constexpr (COST == PC_SQ64 || COST == PC_L164) {
#pragma unroll
            for (int k = 0; k < DP; ++k) x64[k] = valid ? P.xr64[i * DP + k] : 0.0;
        }
    }
    __device__ __forceinline__ double dist(const Buf<COST, DP> &sg, int c) const {
        if constexpr (COST == PC_SQ32) {
            const float4 *yv = reinterpret_cast<const float4 *>(sg.y32 + c * DP);
            float dot = 0.f;
#pragma unroll
            for (int k = 0; k < DP / 4; ++k) {
                const float4 v = yv[k];
                dot = fmaf(x32[4 * k + 0], v.x, dot);
                dot = fmaf(x32[4 * k + 1], v.y, dot);
                dot = fmaf(x32[4 * k + 2], v.z, dot);
                dot = fmaf(x32[4 * k + 3], v.w, dot);
            }
            return (double)fmaf(-2.f, dot, nx + sg.ny[c]);
        } else if constexpr (COST == PC_L132) {
            const float4 *yv = reinterpret_cast<const float4 *>(sg.y32 + c * DP);
            float s = 0.f;
#pragma unroll
            for (int k = 0; k < DP / 4; ++k) {
                const float4 v = yv[k];
                s += fabsf(x32[4 * k + 0] - v.x);
                s += fabsf(x32[4 * k + 1] - v.y);
                s += fabsf(x32[4 * k + 2] - v.z);
                s += fabsf(x32[4 * k + 3] - v.w);
            }
            return (double)s;
        } else if constexpr (COST == PC_SQ64) {
            const double *yv = sg.y64 + c * DP;
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < DP; ++k) {
                const double t = x64[k] - yv[k];
                s = fma(t, t, s);
            }
            return s;
        } else {
            const double *yv = sg.y64 + c * DP;
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < DP; ++k) s += fabs(x64[k] - yv[k]);
            return s;
        }
    }
};

// single-entry distance straight from global memory (argmax seeding)
template <int COST, int DP>
__device__ __forceinline__ double dist_global(const PassSide &P, const RowPt<COST, DP> &rp, long long i,
                                              long long j) {
    if constexpr (COST == PC_DENSE_ROW || COST == PC_DENSE_ROW_T) return P.C[i * P.ldc + j];
    else if constexpr (COST == PC_DENSE_COL || COST == PC_DENSE_COL_T) return P.C[j * P.ldc + i];
    else if constexpr (COST == PC_SQ32 || COST == PC_SQTC) {
        float dot = 0.f;
#pragma unroll
        for (int k = 0; k < DP; ++k) dot = fmaf(rp.x32[k], P.yc32[j * DP + k], dot);
        return (double)fmaf(-2.f, dot, rp.nx + P.nyc[j]);
    } else if constexpr (COST == PC_L132) {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < DP; ++k) s += fabsf(rp.x32[k] - P.yc32[j * DP + k]);
        return (double)s;
    } else if constexpr (COST == PC_SQ64) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < DP; ++k) {
            const double t = rp.x64[k] - P.yc64[j * DP + k];
            s = fma(t, t, s);
        }
        return s;
    } else {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < DP; ++k) s += fabs(rp.x64[k] - P.yc64[j * DP + k]);
        return s;
    }
}

// Tensor-core state of a CTA (PC_SQTC): A tile (the CTA's 128 pass rows as
// fp16, UMMA K-major), TMEM double buffer of kCC fp32 columns, two mbarriers.
template <int AH>
struct TcStateT {
    alignas(128) unsigned char ah[AH];
    uint64_t mbar[2];
    uint32_t tbase;
};
using TcState = TcStateT<kPT * 32>;
template <int COST>
using TcFor = typename std::conditional<COST == PC_SQTC, TcState, TcStateT<16>>::type;

// Streams the column range [jb, je) through the staging buffers and calls
// body(c0, nc, buf, dots) per chunk: for PC_SQTC `dots` holds this thread's
// kCC dot products x_i.y_j from TMEM; for the other costs it is unused.
// Certificate test of every chunk of the CTA's column range at once (kind 1):
// warp w tests chunks w, w+4, ...; lane = column.  Sets bit c of bm for each
// chunk c that is skipped; returns the number skipped (valid in thread 0).
constexpr int kSkipWords = 256;     // chunk bitmap capacity: 8192 chunks per CTA
__device__ __forceinline__ int precheck_chunks(const PassSide &P, const SkipCtx &sk, long long jb, long long je,
                                               long long nch, double inv_eta, int qmode, bool trial,
                                               unsigned *bm) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nw = (int)((nch + 31) >> 5);
    for (int t = tid; t < nw; t += kPT) bm[t] = 0u;
    __syncthreads();
    for (long long c = warp; c < nch; c += kPT / 32) {
        const long long j = jb + c * kCC + lane;
        double d = -INFINITY;
        if (j < je) {
            double q = qmode ? pot_p(P.gc[j], P.psic[j], inv_eta) : pot_q(P.gc[j], P.psic[j], inv_eta);
            if (trial) q = q + P.bv[j];                 // the trial skip-test value (store_trial_qt)
            const float qs = qs_of(q);
            if (qs != -INFINITY) d = (double)qs - (double)__ldg(sk.qref + j);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
        if (lane == 0) {
            const float4 g4 = __ldg(reinterpret_cast<const float4 *>(sk.gcta + c * 4));
            const float4 d4 = __ldg(reinterpret_cast<const float4 *>(sk.gDcta + c * 4));
            const float gv[4] = {g4.x, g4.y, g4.z, g4.w}, dv[4] = {d4.x, d4.y, d4.z, d4.w};
            double g = -INFINITY, gmag = 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {        // per warp tile: gamma - dw Dmin
                if (gv[q] == -INFINITY) continue;
                const double t = (double)gv[q] - sk.dw * (double)dv[q];
                g = fmax(g, t);
                gmag = fmax(gmag, fabs((double)gv[q]) + sk.dw * (double)dv[q]);
            }
            const double lhs = g + d - sk.dthr;
            if (lhs + 1e-12 * (gmag + fabs(d) + fabs(sk.dthr)) <= 0.0) atomicOr(bm + (c >> 5), 1u << (c & 31));
        }
    }
    __syncthreads();
    int n = 0;
    if (tid == 0)
        for (int t = 0; t < nw; ++t) n += __popc(bm[t]);
    return n;
}

// Streams the kept chunks of the column range [jb, je) through the staging
// buffers and calls body(c0, nc, buf, dots) per chunk: for PC_SQTC `dots` holds
// this thread's kCC dot products x_i.y_j from TMEM; for the other costs it is
// unused.  Returns the number of chunks skipped by certificates (thread 0).
template <int COST, int DP, class TS, class Body>
__device__ __forceinline__ int stream_columns(const PassSide &P, long long i0, long long jb, long long je,
                                              double inv_eta, int qmode, bool trial, Buf<COST, DP> *bufs,
                                              TS *tcs, const SkipCtx &sk, const TmaRing &ring, Body body) {
    constexpr int NB = kNBuf<COST>;
    const long long nch = (je - jb + kCC - 1) / kCC;
    if (nch <= 0) return 0;
    const int tid = threadIdx.x, warp = tid >> 5;
    Pref<COST, DP> pf;
    constexpr uint32_t idesc = tc::make_idesc(kCC);
    auto nc_of = [&](long long c) { return (int)min((long long)kCC, je - (jb + c * kCC)); };
    __shared__ unsigned bm[kSkipWords];
    const bool pre = NB > 1 && !kTma<COST> && sk.kind == 1 && nch <= 32LL * kSkipWords;
    int nskip = 0;
    if (pre) nskip = precheck_chunks(P, sk, jb, je, nch, inv_eta, qmode, trial, bm);
    // next kept chunk after c (nch: none)
    auto next_of = [&](long long c) -> long long {
        long long t = c + 1;
        if (!pre) return t;
        while (t < nch) {
            const unsigned wv = ~bm[t >> 5] >> (t & 31);
            if (wv) return min(nch, t + __ffs(wv) - 1);
            t = (t | 31) + 1;
        }
        return nch;
    };
    long long cur = next_of(-1);
    if (cur >= nch) return nskip;
    long long nxt = next_of(cur);
    uint32_t par = 0u;                               // bit b: parity of buffer b's next phase
    // prologue: dense TMA tiles of the first kNSt - 1 chunks in flight (chunks are
    // consecutive: no skipping on dense costs), the first chunk into buffer 0,
    // prefetch the next
    if constexpr (kTma<COST>) {
        if (tid == 0)
            for (long long c = 0; c < kNSt - 1 && c < nch; ++c) tma_issue<COST>(ring, jb, c);
    }
    pf.load(P, jb + cur * kCC, nc_of(cur), trial, sk);
    pf.store(bufs[0], P, i0, jb + cur * kCC, nc_of(cur), inv_eta, qmode, trial, sk);
    if (trial) { __syncthreads(); pf.store_trial_qt(bufs[0], sk, jb + cur * kCC, nc_of(cur)); }
    if (NB > 1 && nxt < nch) pf.load(P, jb + nxt * kCC, nc_of(nxt), trial, sk);
    if constexpr (COST == PC_SQTC) tc::fence_proxy_async();
    __syncthreads();
    if constexpr (COST == PC_SQTC) {
        if (tid == 0) {
            tc::fence_after();
            tc::mma_f16(tcs->tbase, tc::make_desc(tcs->ah), tc::make_desc(bufs[0].yh), idesc);
            tc::commit(&tcs->mbar[0]);
        }
    }
    int b = 0;
    const long long first = cur;
    while (cur < nch) {
        long long nxt2 = nch;
        if (NB > 1) {
            if (nxt < nch) {
                const int nb = b ^ 1;
                if constexpr (COST == PC_SQTC) tc::fence_before();
                __syncthreads();                         // the previous chunk fully consumed
                if constexpr (kTma<COST>) {              // its stage is free: refill kNSt - 1 ahead
                    if (tid == 0 && cur + kNSt - 1 < nch) tma_issue<COST>(ring, jb, cur + kNSt - 1);
                }
                pf.store(bufs[nb], P, i0, jb + nxt * kCC, nc_of(nxt), inv_eta, qmode, trial, sk);
                if (trial) { __syncthreads(); pf.store_trial_qt(bufs[nb], sk, jb + nxt * kCC, nc_of(nxt)); }
                nxt2 = next_of(nxt);
                if (nxt2 < nch) pf.load(P, jb + nxt2 * kCC, nc_of(nxt2), trial, sk);
                if constexpr (COST == PC_SQTC) tc::fence_proxy_async();
                __syncthreads();
                if constexpr (COST == PC_SQTC) {
                    if (tid == 0) {
                        tc::fence_after();
                        tc::mma_f16(tcs->tbase + nb * kCC, tc::make_desc(tcs->ah), tc::make_desc(bufs[nb].yh), idesc);
                        tc::commit(&tcs->mbar[nb]);
                    }
                }
            }
        } else {
            if (cur != first) {                          // single buffer (never skipped): sequential chunks
                __syncthreads();
                pf.load(P, jb + cur * kCC, nc_of(cur), trial, sk);
                pf.store(bufs[0], P, i0, jb + cur * kCC, nc_of(cur), inv_eta, qmode, trial, sk);
                if (trial) { __syncthreads(); pf.store_trial_qt(bufs[0], sk, jb + cur * kCC, nc_of(cur)); }
                __syncthreads();
            }
            nxt2 = nxt + 1;
        }
        float dots[COST == PC_SQTC ? kCC : 1];
        if constexpr (COST == PC_SQTC) {
            tc::mbar_wait(&tcs->mbar[b], (par >> b) & 1u);
            par ^= 1u << b;
            tc::fence_after();
            tc::ld32(tcs->tbase + ((uint32_t)(32 * (warp & 3)) << 16) + b * kCC, dots);
        }
        const unsigned char *tile = nullptr;
        if constexpr (kTma<COST>) {                   // this chunk's C tile has landed
            tc::mbar_wait(&ring.full[cur % kNSt], (uint32_t)((cur / kNSt) & 1));
            tile = ring.base + (cur % kNSt) * kTileB;
        }
        body(jb + cur * kCC, nc_of(cur), bufs[b], dots, tile);
        cur = nxt;
        nxt = nxt2;
        if (NB > 1) b ^= 1;
    }
    return nskip;
}

// skip statistics of one CTA (thread 0), and the launch finalizer's switch: a pass
// that skipped < 5 % of its chunks turns skipping off for the next 16 passes
__device__ __forceinline__ void skip_count(const PassSide &P, const SkipCtx &sk, int nskip, long long jb,
                                           long long je) {
    if (threadIdx.x == 0 && sk.kind == 1) {
        atomicAdd(P.skst + 1, nskip);
        atomicAdd(P.skst + 2, (int)((je - jb + kCC - 1) / kCC));
    }
}
__device__ __forceinline__ bool skip_is_ref(const PassSide &P, float w_lo) {
    return P.skst[0] < 0 || !(w_lo >= __int_as_float(P.skst[3]));
}
// launch finalizer: after a reference pass start a new period; afterwards record fresh
// certificates once the skip fraction falls below 3/4 of the period's best (or at age
// 64); a pass that skipped < 5 % switches skipping off for 16 passes, then re-records
__device__ __forceinline__ void skip_switch(const PassSide &P, float w_lo) {
    if (!P.skipk) return;
    int *s = P.skst;
    if (s[5] > 0) {
        if (--s[5] == 0) s[0] = -1;
        return;
    }
    if (skip_is_ref(P, w_lo)) {
        s[0] = 1;
        s[3] = __float_as_int(w_lo);
        s[4] = -1;
    } else {
        const int frac = s[2] > 0 ? (int)(1e6 * (double)s[1] / (double)s[2]) : 0;
        s[4] = max(s[4], frac);
        s[0] += 1;
        if (frac < 50000) s[5] = 16;
        else if (4LL * frac < 3LL * s[4] || s[0] > 64) s[0] = -1;
        atomicAdd(reinterpret_cast<unsigned long long *>(s + 6), (unsigned long long)s[1]);   // totals (stats)
        atomicAdd(reinterpret_cast<unsigned long long *>(s + 8), (unsigned long long)s[2]);
    }
    s[1] = 0;
    s[2] = 0;
}

// CTA-level tensor-core setup / teardown (PC_SQTC only)
template <class TS>
__device__ __forceinline__ void tc_setup(TS &T, const PassSide &P, long long i0) {
    const int tid = threadIdx.x;
    const long long i = i0 + tid;
    uint4 lo = make_uint4(0, 0, 0, 0), hi = make_uint4(0, 0, 0, 0);
    if (i < P.M) {
        lo = *reinterpret_cast<const uint4 *>(P.xrh + i * 16);
        hi = *reinterpret_cast<const uint4 *>(P.xrh + i * 16 + 8);
    }
    *reinterpret_cast<uint4 *>(T.ah + tc::kmajor_off(tid, 0)) = lo;
    *reinterpret_cast<uint4 *>(T.ah + tc::kmajor_off(tid, 8)) = hi;
    if (tid < 32) tc::tmem_alloc(&T.tbase, 2 * kCC);
    if (tid == 0) {
        tc::mbar_init(&T.mbar[0], 1);
        tc::mbar_init(&T.mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
}
template <class TS>
__device__ __forceinline__ void tc_teardown(TS &T) {
    tc::fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc::fence_after();
        tc::tmem_free(T.tbase, 2 * kCC);
    }
}

// CTA-level TMA ring setup (dense costs staged by TMA): 1024-aligned ring in
// dynamic shared memory, one mbarrier per stage (contains __syncthreads)
template <int COST>
__device__ __forceinline__ TmaRing ring_setup(unsigned char *dyn, uint64_t *full, const CUtensorMap *tm, long long i0) {
    TmaRing R{nullptr, full, tm, (int)i0, (int)i0};
    if constexpr (kTma<COST>) {
        R.base = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(dyn) + 1023) & ~uintptr_t(1023));
        if (threadIdx.x == 0) {
            for (int s = 0; s < kNSt; ++s) tc::mbar_init(&full[s], 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
    }
    return R;
}

// D(i, j0 + c) for the non-tensor-core costs from the staged chunk
template <int COST, int DP>
__device__ __forceinline__ double chunk_dist(const Buf<COST, DP> &B, const PassSide &P, const RowPt<COST, DP> &rp,
                                             long long i, long long j0, int c, const unsigned char *tile) {
    if constexpr (COST == PC_DENSE_ROW_T) {       // swizzled {16 x 128} box c / 16, row = thread
        const int t = threadIdx.x, cc = c & 15;
        return *reinterpret_cast<const double *>(tile + (c >> 4) * (kTileB / 2) + t * 128 +
                                                 ((((cc >> 1) ^ (t & 7))) << 4) + (cc & 1) * 8);
    } else if constexpr (COST == PC_DENSE_COL_T) { // {128 x 32} box, column = thread
        return *reinterpret_cast<const double *>(tile + c * (kPT * 8) + threadIdx.x * 8);
    } else if constexpr (COST == PC_DENSE_ROW) return B.tile[c * (kPT + 1) + threadIdx.x];
    else if constexpr (COST == PC_DENSE_COL) return j0 + c < P.N ? __ldg(P.C + (j0 + c) * P.ldc + i) : 0.0;
    else if constexpr (COST == PC_SQTC) return 0.0;
    else return rp.dist(B, c);
}

// ----------------------------------------------------- ticket helpers
// returns true in exactly one CTA: the last of `total` arrivals on *t (then reset)
__device__ __forceinline__ bool last_arrival(unsigned *t, unsigned total, bool *sh_flag) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(t, 1u);
        *sh_flag = (prev == total - 1);
        if (*sh_flag) *t = 0u;
    }
    __syncthreads();
    if (*sh_flag) __threadfence();
    return *sh_flag;
}

__device__ __forceinline__ double block_reduce_sum(double v, double *sh) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double t = 0.0;
    for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) t += sh[w2];
    return t;
}
__device__ __forceinline__ double block_reduce_max(double v, double *sh) {
    v = warp_max(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double t = -INFINITY;
    for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) t = fmax(t, sh[w2]);
    return t;
}

// CTA setup of the chunk skip (block-wide; contains __syncthreads, call from all
// threads).  thr32 = the row's threshold at the start of the pass.
__device__ __forceinline__ SkipCtx skip_setup(const PassSide &P, int rb, int sp, long long i, bool valid,
                                              long long jb, float thr32, float w_lo, double *red) {
    SkipCtx sk{0, -INFINITY, jb, nullptr, nullptr, 0.0, P.qref, rb == 0};
    if (!P.skipk || P.skst[5] > 0) return sk;
    sk.gcta = P.gam + ((long long)rb * P.S + sp) * P.cps * 4;
    sk.gDcta = P.gamD + ((long long)rb * P.S + sp) * P.cps * 4;
    if (skip_is_ref(P, w_lo)) {
        sk.kind = 2;
        if (valid && sp == 0) P.tref[i] = thr32;
        return sk;
    }
    sk.kind = 1;
    sk.dw = (double)w_lo - (double)__int_as_float(P.skst[3]);     // exact; >= 0 (skip_is_ref)
    double d = INFINITY;
    if (valid) {
        const float t = P.tref[i];
        d = thr32 == -INFINITY ? -INFINITY : (double)thr32 - (double)t;
        d -= 1e-15 * (fabs((double)thr32) + fabs((double)t));
    }
    d = -block_reduce_max(-d, red);
    sk.dthr = d;
    return sk;
}

// reference pass: certificate of this chunk for the warp's rows (all 32 lanes)
// dmn: the row's minimum Df over the chunk (any lower bound is valid; columns past
// the end of a partial chunk may only lower it)
__device__ __forceinline__ void record_cert(const SkipCtx &sk, long long j0, float vmx, float T, bool valid,
                                            float dmn) {
    double e = -INFINITY;
    if (valid && vmx != -INFINITY) e = (double)vmx + fabs((double)vmx) * 0x1p-22 - (double)T;
    float dm = valid ? fmaxf(dmn, 0.f) : INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        e = fmax(e, __shfl_xor_sync(0xffffffffu, e, o));
        dm = fminf(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    }
    if ((threadIdx.x & 31) == 0) {
        const long long k = ((j0 - sk.jb) / kCC) * 4 + (threadIdx.x >> 5);
        sk.gcta[k] = __double2float_ru(e);
        sk.gDcta[k] = dm == INFINITY ? 0.f : dm;
    }
}

// phase 1 of a chunk (branch-free): the survivor mask of the fp32 test
// fl(qs_j - w_lo D_ij) > thr32, the fp32 distances (PC_SQTC) and the row's
// maximum test value (used by reference passes)
// costs whose exact fp32 distances phase 1 keeps (for phase 2 through shared memory)
template <int COST>
constexpr bool kDv = COST == PC_SQTC || COST == PC_SQ32 || COST == PC_L132;

// REF (reference passes of the chunk skip only): also the row's maximum test value
// vmx and minimum distance dmn over the chunk
template <int COST, int DP, bool REF, bool REC = false>
__device__ __forceinline__ unsigned phase1(const Buf<COST, DP> &B, const PassSide &P, const RowPt<COST, DP> &rp,
                                           long long i, long long j0, int nc, const float *dots, float w_lo,
                                           float thr32, float (&Dv)[kDv<COST> ? kCC : 1], float &vmx,
                                           float &dmn, const unsigned char *tile, float lb = 0.f,
                                           unsigned *rmask = nullptr) {
    unsigned mask = 0u;
#pragma unroll
    for (int c4 = 0; c4 < kCC; c4 += 4) {
        const float4 qs4 = *reinterpret_cast<const float4 *>(B.qs + c4);
        const float qsv[4] = {qs4.x, qs4.y, qs4.z, qs4.w};
        float nyv[4] = {0.f, 0.f, 0.f, 0.f};
        if constexpr (COST == PC_SQTC) {
            const float4 ny4 = *reinterpret_cast<const float4 *>(B.ny + c4);
            nyv[0] = ny4.x; nyv[1] = ny4.y; nyv[2] = ny4.z; nyv[3] = ny4.w;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = c4 + j;
            float Df;
            if constexpr (COST == PC_SQTC) {
                Df = fmaf(-2.f, dots[c], rp.nx + nyv[j]);
                Dv[c] = Df;
            } else {
                Df = (float)chunk_dist<COST, DP>(B, P, rp, i, j0, c, tile);
                if constexpr (kDv<COST>) Dv[c] = Df;
            }
            const float v = fmaf(-w_lo, Df, qsv[j]);
            // columns c >= nc of a partial chunk are staged with q = -inf, so v = -inf there:
            // no per-entry range test is needed
            if constexpr (REF) {
                vmx = fmaxf(vmx, v);
                dmn = fminf(dmn, Df);
            }
            if constexpr (REC) *rmask |= (v > lb) ? (1u << c) : 0u;
            mask |= (v > thr32) ? (1u << c) : 0u;
        }
    }
    return mask;
}

// =========================================================================
// LSE half-sweep.  One side per launch (A.side[0]).
// Stats written by the global finalizer: st[0] = residual ||a - X~ e||_1 of
// the starting iterate (pass-row side), st[1] = max |f_new - f_old|.
// =========================================================================
// Row-block and launch finalize of a half-sweep (the dense kernel after its split
// ticket, the sparse path's merge kernel directly): merge the S split partials of
// each pass row in split order, update the potential, residual of the starting
// iterate, argmax seed; for the candidate lists the new potentials become the other
// side's column values, with their drift since that side's record pass.
template <int NB = 8>
__device__ __forceinline__ void lse_rowblock_finalize(const PassArgs &A, const PassSide &P, int rb, long long i,
                                                      bool valid, const double *thi, const double *tlo, double *red,
                                                      bool *flag, float w_lo, bool rec_ran, bool sparse) {
    const int tid = threadIdx.x, lane = tid & 31;
    const double inv_eta = A.inv_eta;
    double res = 0.0, dmax = 0.0, dq = -INFINITY;
    if (valid) {
        // split partials in batches of NB (independent loads first; the max and the sum
        // then run in split order, whatever NB)
        double M = -INFINITY;
        int jbest = -1;
        for (int s0 = 0; s0 < P.S; s0 += NB) {
            double v[NB];
            int jj[NB];
#pragma unroll
            for (int q = 0; q < NB; ++q) {
                const int s = min(s0 + q, P.S - 1);
                v[q] = P.pa[(long long)s * P.M + i];
                jj[q] = P.pj[(long long)s * P.M + i];
            }
#pragma unroll
            for (int q = 0; q < NB; ++q)
                if (s0 + q < P.S && v[q] > M) { M = v[q]; jbest = jj[q]; }
        }
        double Ssum = 0.0;
        for (int s0 = 0; s0 < P.S; s0 += NB) {
            double v[NB], c[NB];
#pragma unroll
            for (int q = 0; q < NB; ++q) {
                const int s = min(s0 + q, P.S - 1);
                v[q] = P.pa[(long long)s * P.M + i];
                c[q] = P.pb[(long long)s * P.M + i];
            }
#pragma unroll
            for (int q = 0; q < NB; ++q)
                if (s0 + q < P.S && c[q] > 0.0) Ssum += c[q] * pexp(v[q] - M, thi, tlo);
        }
        const double L = M + log(Ssum);
        const double fo = P.fr[i], ph = P.phir[i], a = P.ar[i];
        // residual of the starting iterate: row sum = exp(P_i + L)
        const double r = exp(pot_p(fo, ph, inv_eta) + L);
        res = fabs(a - r);
        const double fn = A.eta * (log(a) + 1.0 - L) - ph;
        dmax = fabs(fn - fo);
        if (P.fsave) P.fsave[i] = fo;
        P.fout[i] = fn;
        if (jbest >= 0) P.jstar[i] = jbest;
        if (P.oqv) {                          // the other orientation's column value of this row
            const double q = pot_q(fn, ph, inv_eta);
            const float qs = qs_of(q);
            P.oqv[i] = q;
            P.oqsv[i] = qs;
            dq = qs == -INFINITY ? -INFINITY : (double)qs - (double)P.oqref[i];
        }
    }
    if (P.oqv) {      // a warp's 32 pass rows are one chunk of the other side's columns
        const double wq = warp_max(dq);
        if (lane == 0 && i < P.M) P.odqc[i >> 5] = wq == -INFINITY ? -INFINITY : __double2float_ru(wq);
    }
    const double bres = block_reduce_sum(res, red);
    const double bdm = block_reduce_max(dmax, red);
    if (tid == 0) {
        P.blk[rb * 8 + 0] = bres;
        P.blk[rb * 8 + 1] = bdm;
    }
    if (!last_arrival(A.gticket, (unsigned)P.RB, flag)) return;
    // ---- launch finalize ----
    double v0 = 0.0, v1 = 0.0;
    for (int b = tid; b < P.RB; b += kPT) {     // deterministic: fixed assignment + fixed tree
        v0 += P.blk[b * 8 + 0];
        v1 = fmax(v1, P.blk[b * 8 + 1]);
    }
    const double R = block_reduce_sum(v0, red);
    const double DM = block_reduce_max(v1, red);
    if (P.oqv) {      // per split of the other side: the largest chunk drift of its columns
        for (int sp = tid; sp < P.oS; sp += kPT) {
            long long jb, je;
            split_range(P.M, P.oS, sp, jb, je);
            float mx = -INFINITY;
            for (long long c = jb / kCC; c < (je + kCC - 1) / kCC; ++c) mx = fmaxf(mx, P.odqc[c]);
            P.odqs[sp] = mx;
        }
    }
    if (tid == 0) {
        A.st[0] = R;
        A.st[1] = DM;
        if (A.count_sweep) A.ctl[1] += 1;
        if (!sparse) skip_switch(P, w_lo);    // list passes stream no chunks: the skip period is not theirs
        if (rec_ran) {                        // lists recorded: the sparse path of this half-sweep exits
            P.lctl[P.lori] = 0;
            P.lctl[2 + P.lori] = A.lt;
            P.lctl[12 + P.lori] += 1;
        }
        if (sparse) {                         // record again once > 2 % of the units fell back
            const long long U = (long long)P.S * P.M;
            if (50LL * P.lctl[8] > U) P.lctl[P.lori] = 1;
            P.lctl[6 + P.lori] += P.lctl[8];
            P.lctl[8] = 0;
        }
        if (A.test_tol && A.sink_tol && R <= *A.sink_tol) {
            A.ctl[0] = 1;     // converged at the starting iterate: roll back this update
            A.ctl[2] = 1;
        }
    }
}

template <int COST, int DP>
__global__ void __launch_bounds__(kPT, 5) lse_pass_kernel(PassArgs A, const __grid_constant__ CUtensorMap tm0) {
    extern __shared__ __align__(1024) unsigned char dyn_smem[];   // TMA ring (dense costs) or unused
    __shared__ uint64_t ring_full[kNSt];
    __shared__ Buf<COST, DP> bufs[kNBuf<COST>];
    __shared__ TcFor<COST> tcs_storage[1];
    __shared__ float dscr[kDv<COST> ? kPT * (kCC + 1) : 1];
    __shared__ double thi[64], tlo[64];
    __shared__ double red[kPT / 32];
    __shared__ bool flag;
    if (A.check_done && A.ctl[0]) return;            // Sinkhorn phase already converged
    const PassSide &P = A.side[0];
    // candidate lists: this dense pass runs only when the lists must be (re)recorded
    const bool rec = P.lrec != 0;
    if (rec && P.lctl[P.lori] == 0) return;
    const int tid = threadIdx.x;
    const int rb = blockIdx.x % P.RB, sp = blockIdx.x / P.RB;
    const long long i0 = (long long)rb * kPT, i = i0 + tid;
    const bool valid = i < P.M;
    long long jb, je;
    split_range(P.N, P.S, sp, jb, je);
    load_exp_table(A.tab, thi, tlo);
    TcFor<COST> &tcs = tcs_storage[0];
    if constexpr (COST == PC_SQTC) tc_setup(tcs, P, i0);
    RowPt<COST, DP> rp;
    rp.load(P, i, valid);
    const double w = A.w, inv_eta = A.inv_eta;
    const float w_lo = (float)w * (1.f - 0x1p-19f);
    double mx = -INFINITY, sm = 0.0;       // the row's reference (a true entry) and sum exp(x - mx)
    int jm = -1;
    if (valid) {
        const int js = P.jstar[i];
        if (js >= 0 && js < P.N) {     // lower bound of the row max: one true entry
            const double D = dist_global<COST, DP>(P, rp, i, js);
            mx = fma(-w, D, pot_q(P.gc[js], P.psic[js], inv_eta));
            jm = js;
        }
    }
    float *dsc = dscr + tid * (kCC + 1);       // this thread's chunk distances (kDv costs)
    int nsurv = 0;
    const float thr0 = thr_lo_of(mx - kLseCut);
    // record pass: every entry with v > lb goes to the list (lb = thr0 - margin); the
    // chunk skip then certifies against lb, so skipped chunks hold no list entry either
    const float lb = rec ? (mx == -INFINITY ? -INFINITY : __double2float_rd((double)thr0 - A.lmargin)) : thr0;
    const long long lbase = ((long long)sp * P.M + i) * P.lcap;      // unit-major lists
    int lk = 0;
    if (rec && valid && sp == 0) P.lB[i] = lb;
    if (rec && rb == 0)             // the record's column test values (also of chunks skipped below)
        for (long long j = jb + tid; j < je; j += kPT) {
            const double qj = pot_q(P.gc[j], P.psic[j], inv_eta);
            P.lqref[j] = qs_of(qj);
            if (P.lqd) P.lqd[j] = qj;
        }
    const SkipCtx sk = skip_setup(P, rb, sp, i, valid, jb, lb, w_lo, red);
    const TmaRing ring = ring_setup<COST>(dyn_smem, ring_full, &tm0, i0);
    const int nskip = stream_columns<COST, DP>(P, i0, jb, je, inv_eta, 0, false, bufs, &tcs, sk, ring,
                             [&](long long j0, int nc, const Buf<COST, DP> &B, const float *dots,
                                 const unsigned char *tile) {
        // phase 1: skip test against the chunk-start bound of the row max
        const float thr32 = thr_lo_of(mx - kLseCut);
        unsigned mask = 0u, rmask = 0u;
        float vmx = -INFINITY, dmn = INFINITY;
        float Dv[kDv<COST> ? kCC : 1];
        if (valid) {
            if (rec) {
                if (sk.kind == 2)
                    mask = phase1<COST, DP, true, true>(B, P, rp, i, j0, nc, dots, w_lo, thr32, Dv, vmx, dmn, tile,
                                                        lb, &rmask);
                else
                    mask = phase1<COST, DP, false, true>(B, P, rp, i, j0, nc, dots, w_lo, thr32, Dv, vmx, dmn, tile,
                                                         lb, &rmask);
            } else if (sk.kind == 2) {
                mask = phase1<COST, DP, true>(B, P, rp, i, j0, nc, dots, w_lo, thr32, Dv, vmx, dmn, tile);
            } else {
                mask = phase1<COST, DP, false>(B, P, rp, i, j0, nc, dots, w_lo, thr32, Dv, vmx, dmn, tile);
            }
        }
        if (sk.kind == 2) record_cert(sk, j0, vmx, lb, valid, dmn);
        nsurv += __popc(mask);
        if constexpr (kDv<COST>) {
            // distances are needed only where some lane of the warp has a survivor
            if (__any_sync(0xffffffffu, (mask | rmask) != 0u)) {
#pragma unroll
                for (int c = 0; c < kCC; ++c) dsc[c] = Dv[c];
            }
        }
        if (!valid) return;
        if (rec) {                                 // append this chunk's list entries
            LDT<COST> *lD = reinterpret_cast<LDT<COST> *>(P.lD);
            while (rmask) {
                const int c = __ffs(rmask) - 1;
                rmask &= rmask - 1u;
                if (lk >= 0 && lk < P.lcap) {
                    const long long e = lbase + lk;
                    P.lj[e] = (int)(j0 + c);
                    if constexpr (kDv<COST>) lD[e] = dsc[c];
                    else lD[e] = (LDT<COST>)chunk_dist<COST, DP>(B, P, rp, i, j0, c, tile);
                    ++lk;
                } else {
                    lk = -1;                       // overflow: this (split, row) falls back to dense
                }
            }
        }
        // phase 2: the surviving entries of this row, two per iteration (independent
        // exponentials).  The reference mx is a true entry; sm accumulates exp(x - mx)
        // for x <= mx + 1 and a larger x (rare once the argmax seed is in place) becomes
        // the new reference with sm rescaled -- no per-entry max bookkeeping.
        while (mask) {
            const int c1 = __ffs(mask) - 1;
            mask &= mask - 1u;
            const bool two = mask != 0u;
            const int c2 = two ? __ffs(mask) - 1 : c1;
            mask &= two ? mask - 1u : mask;
            const double D1 = kDv<COST> ? (double)dsc[c1] : chunk_dist<COST, DP>(B, P, rp, i, j0, c1, tile);
            const double D2 = kDv<COST> ? (double)dsc[c2] : chunk_dist<COST, DP>(B, P, rp, i, j0, c2, tile);
            const double x1 = fma(-w, D1, B.q[c1]);
            const double x2 = fma(-w, D2, B.q[c2]);
            if (fmax(x1, x2) > mx + 1.0) {        // new reference: the larger entry
                const bool first = x1 >= x2;
                const double xn = first ? x1 : x2;
                sm = sm * pexp_lean(fmax(-745.0, mx - xn), thi, tlo);
                mx = xn;
                jm = (int)(j0 + (first ? c1 : c2));
            }
            const double e1 = pexp_lean(fmax(-745.0, x1 - mx), thi, tlo);
            const double e2 = pexp_lean(fmax(-745.0, x2 - mx), thi, tlo);
            sm += two ? e1 + e2 : e1;
        }
    });
    if constexpr (COST == PC_SQTC) tc_teardown(tcs);
    skip_count(P, sk, nskip, jb, je);
    count_survivors(A.count_surv, 0, nsurv);
    if (valid) {
        P.pa[(long long)sp * P.M + i] = mx;
        P.pb[(long long)sp * P.M + i] = sm;
        P.pj[(long long)sp * P.M + i] = jm;
        if (rec) {
            // pad the list to whole batches of 8 with entries that can never survive
            // (distance +inf: test value -inf), so the walk loads whole batches
            if (lk > 0 && (lk & 7)) {
                LDT<COST> *lD = reinterpret_cast<LDT<COST> *>(P.lD);
                const int jl = P.lj[lbase + lk - 1];
                for (int k = lk; k < ((lk + 7) & ~7); ++k) {
                    P.lj[lbase + k] = jl;
                    lD[lbase + k] = (LDT<COST>)INFINITY;
                }
            }
            P.lcnt[(long long)sp * P.M + i] = lk;
            if (lk < 0) atomicAdd(P.lctl + 4, 1);
            else {
                atomicMax(P.lctl + 5, lk);
                atomicAdd(P.lctl + 14 + P.lori, lk);      // entries of the last record (stats)
            }
        }
    }
    if (!last_arrival(P.ticket + rb, (unsigned)P.S, &flag)) return;
    lse_rowblock_finalize(A, P, rb, i, valid, thi, tlo, red, &flag, w_lo, rec, false);
}

// =========================================================================
// Sparse LSE half-sweep over the certified candidate lists (Sinkhorn phase).
//
// The record pass (lse_pass_kernel with lrec) lists, per unit (split sp, pass row i),
// every entry with fp32 test value v > lB_i = thr0_i - margin, in column order.
// Certificate of a unit in a later pass (same w: one Sinkhorn phase): an unlisted
// entry had fl(qs_j - w_lo D_ij) <= lB_i, so its real value now is at most
// lB_i + ulp(lB_i) + (qs_j(now) - qs_j(record)) <= lB_i + ulp + ldqs[sp].  If that is
// <= thr0_i (this pass's starting threshold, below every chunk threshold of the dense
// pass), no unlisted entry passes the dense pass's fp32 test, and walking the list
// with the dense pass's chunk-start thresholds, survivor pairing and reference updates
// gives bit-identical partials.  Units that fail go to a queue that
// lse_fallback_kernel scans densely (one warp per unit, same arithmetic);
// lse_merge_kernel then merges the split partials.  After each record, lse_sort_kernel
// orders the units by decreasing list length, so the threads of a warp walk lists of
// about the same length (no divergence) and the long ones start first.
// =========================================================================
constexpr int kKB = 16;                 // ELL k-steps per pipeline stage (32 lanes x kKB entries)
constexpr int kKNS = 2;                 // stages per warp
constexpr int kKStJ = kKB * 32 * 4;     // stage bytes: columns (int32)
constexpr int kKStK = kKB * 32 * 8;     // stage bytes: kernel values (fp64)
constexpr int kKRing = (kPT / 32) * kKNS * (kKStJ + kKStK);   // 96 KB per CTA

// per split, the pass rows by decreasing list length (counting sort in 64 length
// buckets, one CTA per split); only right after a record
__global__ void __launch_bounds__(1024) lse_sort_kernel(PassArgs A) {
    const PassSide &P = A.side[0];
    if (P.lctl[2 + P.lori] != A.lt) return;
    __shared__ int hist[64];
    const int sp = blockIdx.x, tid = threadIdx.x;
    const int *cnt = P.lcnt + (long long)sp * P.M;
    int *perm = P.lperm + (long long)sp * P.M;
    if (A.lnosort) {
        for (long long i = tid; i < P.M; i += 1024) perm[i] = (int)i;
    } else {
        if (tid < 64) hist[tid] = 0;
        __syncthreads();
        auto key = [&](long long i) {
            const int c = cnt[i];
            return c < 0 ? 0 : 63 - min(63, c >> 3);           // descending length; overflow first
        };
        for (long long i = tid; i < P.M; i += 1024) atomicAdd(hist + key(i), 1);
        __syncthreads();
        if (tid == 0) {
            int acc = 0;
            for (int k = 0; k < 64; ++k) { const int h = hist[k]; hist[k] = acc; acc += h; }
        }
        __syncthreads();
        for (long long i = tid; i < P.M; i += 1024) perm[atomicAdd(hist + key(i), 1)] = (int)i;
    }
    if (!P.ellL) return;
    // kernel-matrix mode: the ELL tile (32 consecutive ranks) lengths in whole stages of kKB
    // k-steps, and their dense packing offsets inside the split
    __syncthreads();
    const int ntile = (int)(P.Mpad / 32), lane = tid & 31, warp = tid >> 5;
    int *tl = P.ellL + (long long)sp * ntile, *to = P.ellrel + (long long)sp * ntile;
    for (int tt = warp; tt < ntile; tt += 32) {
        const long long r = (long long)tt * 32 + lane;
        const int c = r < P.M ? max(0, cnt[perm[r]]) : 0;
        const int L = (__reduce_max_sync(0xffffffffu, c) + kKB - 1) / kKB * kKB;
        if (lane == 0) tl[tt] = L;
    }
    __syncthreads();
    if (warp == 0) {
        int run = 0;
        for (int t0 = 0; t0 < ntile; t0 += 32) {
            const int tt = t0 + lane;
            const int v = tt < ntile ? tl[tt] / kKB : 0;
            int inc = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int nb = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += nb;
            }
            if (tt < ntile) to[tt] = run + inc - v;
            run += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) P.elltot[sp] = run;
    }
}

template <int COST, int DP, bool STG>
__global__ void __launch_bounds__(kPT) lse_sparse_kernel(PassArgs A) {
    constexpr int kLB = 8;                           // list entries per batch
    extern __shared__ __align__(16) unsigned char lsm[];   // the split's column values
    __shared__ double thi[64], tlo[64];
    __shared__ double sx[kLB * kPT], se[kLB * kPT];  // the batch, [entry][thread]
    __shared__ int sj[kLB * kPT];
    if (A.check_done && A.ctl[0]) return;            // Sinkhorn phase already converged
    const PassSide &P = A.side[0];
    if (P.lctl[2 + P.lori] == A.lt) return;          // the dense pass recorded this half-sweep
    // CTA = 128 consecutive ranks (by list length) of one split; the longest groups of
    // all splits come first (longest-first scheduling)
    const int sp = blockIdx.x % P.S;
    const long long t = (long long)(blockIdx.x / P.S) * kPT + threadIdx.x;
    long long jb, je;
    split_range(P.N, P.S, sp, jb, je);
    load_exp_table(A.tab, thi, tlo);
    // the split's column values in shared memory (STG: when they fit), else from global
    double *sq = reinterpret_cast<double *>(lsm);
    float *sqs = reinterpret_cast<float *>(sq + (STG ? je - jb : 0));
    if constexpr (STG)
        for (long long j = jb + threadIdx.x; j < je; j += kPT) {
            sq[j - jb] = __ldg(P.lqv + j);
            sqs[j - jb] = __ldg(P.lqsv + j);
        }
    __syncthreads();
    if (t >= P.M) return;
    const long long i = P.lperm[(long long)sp * P.M + t];
    const int u = (int)((long long)sp * P.M + i);
    RowPt<COST, DP> rp;
    rp.load(P, i, true);
    const double w = A.w;
    const float w_lo = (float)w * (1.f - 0x1p-19f);
    double mx = -INFINITY, sm = 0.0;
    int jm = -1;
    const int js = P.jstar[i];
    if (js >= 0 && js < P.N) {
        const double D = dist_global<COST, DP>(P, rp, i, js);
        mx = fma(-w, D, P.lqv[js]);
        jm = js;
    }
    const float thr0 = thr_lo_of(mx - kLseCut);
    const int cnt = P.lcnt[u];
    const float B = P.lB[i], dq = P.ldqs[sp];
    const double ub = (double)B + (double)ulpf_of(B) + (double)dq;
    if (!(cnt >= 0 && thr0 != -INFINITY && dq != INFINITY &&
          ub + 1e-12 * (fabs((double)B) + fabs((double)dq)) <= (double)thr0)) {
        P.lq[atomicAdd(P.lctl + 8, 1)] = u;          // certificate failed: dense scan (fallback kernel)
        return;
    }
    // the dense pass's sequence: per chunk the start threshold, survivors in column order
    // taken two at a time (a chunk's odd last survivor alone), reference updates
    long long cur = -1;
    float thr32 = thr0;
    int pj = -1, nsurv = 0;
    double px = 0.0;                                 // a pending survivor (first of a pair): its x
    auto step = [&](int j1, double x1, int j2, double x2, bool two) {
        if (fmax(x1, x2) > mx + 1.0) {
            const bool first = x1 >= x2;
            const double xn = first ? x1 : x2;
            sm = sm * pexp_lean(fmax(-745.0, mx - xn), thi, tlo);
            mx = xn;
            jm = first ? j1 : j2;
        }
        const double e1 = pexp_lean(fmax(-745.0, x1 - mx), thi, tlo);
        const double e2 = pexp_lean(fmax(-745.0, x2 - mx), thi, tlo);
        sm += two ? e1 + e2 : e1;
    };
    // Batches of kLB entries: the loads are independent of the running state and go
    // first; the fp32 test is branch-free (entries of a chunk that began in an earlier
    // batch keep its start threshold).  If no survivor of the batch (nor the pending one)
    // exceeds mx + 1, the reference cannot move inside the batch, so every exponential
    // is taken against the same mx -- independently, with full ILP -- and the survivors
    // are then summed in the dense pass's pair order.  Otherwise the batch runs the
    // sequential pair steps.  Both give the dense pass's bits.
    const LDT<COST> *lD = reinterpret_cast<const LDT<COST> *>(P.lD) + (long long)u * P.lcap;
    const int *lj = P.lj + (long long)u * P.lcap;
    int *tj = sj + threadIdx.x;
    double *tx = sx + threadIdx.x, *te = se + threadIdx.x;
    // whole batches (lists are padded to multiples of kLB), 16-byte loads, the next
    // batch's loads in flight while this one is processed
    int jn[kLB];
    LDT<COST> dn[kLB];
    auto load_batch = [&](int k0) {
        const int4 a0 = __ldg(reinterpret_cast<const int4 *>(lj + k0));
        const int4 a1 = __ldg(reinterpret_cast<const int4 *>(lj + k0) + 1);
        jn[0] = a0.x; jn[1] = a0.y; jn[2] = a0.z; jn[3] = a0.w;
        jn[4] = a1.x; jn[5] = a1.y; jn[6] = a1.z; jn[7] = a1.w;
        if constexpr (sizeof(LDT<COST>) == 4) {
            const float4 d0 = __ldg(reinterpret_cast<const float4 *>(lD + k0));
            const float4 d1 = __ldg(reinterpret_cast<const float4 *>(lD + k0) + 1);
            dn[0] = d0.x; dn[1] = d0.y; dn[2] = d0.z; dn[3] = d0.w;
            dn[4] = d1.x; dn[5] = d1.y; dn[6] = d1.z; dn[7] = d1.w;
        } else {
#pragma unroll
            for (int q = 0; q < kLB; q += 2) {
                const double2 d = __ldg(reinterpret_cast<const double2 *>(lD + k0 + q));
                dn[q] = d.x;
                dn[q + 1] = d.y;
            }
        }
    };
    if (cnt > 0) load_batch(0);
    for (int k0 = 0; k0 < cnt; k0 += kLB) {
        int jv[kLB];
        LDT<COST> dv[kLB];
        float qsv[kLB];
        double xv[kLB];
#pragma unroll
        for (int q = 0; q < kLB; ++q) { jv[q] = jn[q]; dv[q] = dn[q]; }
        if (k0 + kLB < cnt) load_batch(k0 + kLB);
#pragma unroll
        for (int q = 0; q < kLB; ++q) {
            if constexpr (STG) {
                qsv[q] = sqs[jv[q] - jb];
                xv[q] = fma(-w, (double)dv[q], sq[jv[q] - jb]);
            } else {
                qsv[q] = __ldg(P.lqsv + jv[q]);
                xv[q] = fma(-w, (double)dv[q], __ldg(P.lqv + jv[q]));
            }
        }
        const int nb = min(kLB, cnt - k0);
        unsigned mask = 0u;
        const float tnew = thr_lo_of(mx - kLseCut);
        double xmax = pj >= 0 ? px : -INFINITY;
#pragma unroll
        for (int q = 0; q < kLB; ++q) {
            const float v = fmaf(-w_lo, (float)dv[q], qsv[q]);
            const float th = (jv[q] >> 5) == cur ? thr32 : tnew;
            const bool sv = q < nb && v > th;
            mask |= sv ? (1u << q) : 0u;
            xmax = sv ? fmax(xmax, xv[q]) : xmax;
            tj[q * kPT] = jv[q];
            tx[q * kPT] = xv[q];
        }
        if (mask == 0u) continue;
        if (!(xmax > mx + 1.0)) {
            // fast path: the reference stays; all exponentials against mx
            double epend = 0.0;
            if (pj >= 0) epend = pexp_lean(fmax(-745.0, px - mx), thi, tlo);
#pragma unroll
            for (int q = 0; q < kLB; ++q) te[q * kPT] = pexp_lean(fmax(-745.0, xv[q] - mx), thi, tlo);
            nsurv += __popc(mask);
            while (mask) {
                const int q = __ffs(mask) - 1;
                mask &= mask - 1u;
                const int jq = tj[q * kPT];
                const double eq = te[q * kPT];
                if ((jq >> 5) != cur) {
                    if (pj >= 0) { sm += epend; pj = -1; }       // the previous chunk's odd survivor
                    cur = jq >> 5;
                    thr32 = tnew;
                }
                if (pj >= 0) { sm += epend + eq; pj = -1; }
                else { pj = jq; px = tx[q * kPT]; epend = eq; }
            }
            continue;
        }
        // a reference update may happen inside this batch: the dense pass's steps in order
        while (mask) {
            const int q = __ffs(mask) - 1;
            mask &= mask - 1u;
            const int jq = tj[q * kPT];
            if ((jq >> 5) != cur) {
                if (pj >= 0) { step(pj, px, pj, px, false); pj = -1; }
                cur = jq >> 5;
                thr32 = thr_lo_of(mx - kLseCut);
                if (thr32 != tnew) {
                    // mx moved: this and the later entries of the batch are tested against
                    // the new chunk thresholds, as the dense pass does
                    unsigned m2 = 0u;
#pragma unroll
                    for (int r = 0; r < kLB; ++r) {
                        const float v = fmaf(-w_lo, (float)dv[r], qsv[r]);
                        m2 |= (r < nb && r >= q && v > thr32) ? (1u << r) : 0u;
                    }
                    mask = m2 & ~((2u << q) - 1u);
                    if (!((m2 >> q) & 1u)) continue;
                }
            }
            ++nsurv;
            const double xq = tx[q * kPT];
            if (pj >= 0) { step(pj, px, jq, xq, true); pj = -1; }
            else { pj = jq; px = xq; }
        }
    }
    if (pj >= 0) step(pj, px, pj, px, false);
    if (A.count_surv && nsurv) atomicAdd(g_surv, (unsigned long long)nsurv);
    P.pa[(long long)sp * P.M + i] = mx;
    P.pb[(long long)sp * P.M + i] = sm;
    P.pj[(long long)sp * P.M + i] = jm;
}

// Dense scan of the units whose certificate failed: one warp per unit, lane = column
// of a chunk; the survivors of a chunk are taken in order, two at a time, by every
// lane alike (values broadcast by shuffles) -- the dense pass's arithmetic.
template <int COST, int DP>
__global__ void __launch_bounds__(kPT) lse_fallback_kernel(PassArgs A) {
    __shared__ double thi[64], tlo[64];
    if (A.check_done && A.ctl[0]) return;
    const PassSide &P = A.side[0];
    if (P.lctl[2 + P.lori] == A.lt) return;
    const int nq = P.lctl[8];
    if (nq == 0) return;
    load_exp_table(A.tab, thi, tlo);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long gw = ((long long)blockIdx.x * kPT + threadIdx.x) >> 5, nw = (long long)gridDim.x * (kPT / 32);
    const double w = A.w;
    const float w_lo = (float)w * (1.f - 0x1p-19f);
    for (long long qi = gw; qi < nq; qi += nw) {
        const int u = P.lq[qi];
        const long long i = u % P.M;
        const int sp = (int)(u / P.M);
        long long jb, je;
        split_range(P.N, P.S, sp, jb, je);
        RowPt<COST, DP> rp;
        rp.load(P, i, true);
        double mx = -INFINITY, sm = 0.0;
        int jm = -1, nsurv = 0;
        const int js = P.jstar[i];
        if (js >= 0 && js < P.N) {
            const double D = dist_global<COST, DP>(P, rp, i, js);
            mx = fma(-w, D, P.lqv[js]);
            jm = js;
        }
        for (long long j0 = jb; j0 < je; j0 += kCC) {
            const long long j = j0 + lane;
            double D = 0.0, q = 0.0;
            float v = -INFINITY;
            if (j < je) {
                D = dist_global<COST, DP>(P, rp, i, j);
                q = __ldg(P.lqv + j);
                v = fmaf(-w_lo, (float)D, __ldg(P.lqsv + j));
            }
            const float thr32 = thr_lo_of(mx - kLseCut);
            unsigned mask = __ballot_sync(0xffffffffu, v > thr32);
            nsurv += __popc(mask);
            while (mask) {
                const int c1 = __ffs(mask) - 1;
                mask &= mask - 1u;
                const bool two = mask != 0u;
                const int c2 = two ? __ffs(mask) - 1 : c1;
                mask &= two ? mask - 1u : mask;
                const double D1 = __shfl_sync(0xffffffffu, D, c1), q1 = __shfl_sync(0xffffffffu, q, c1);
                const double D2 = __shfl_sync(0xffffffffu, D, c2), q2 = __shfl_sync(0xffffffffu, q, c2);
                const double x1 = fma(-w, D1, q1);
                const double x2 = fma(-w, D2, q2);
                if (fmax(x1, x2) > mx + 1.0) {
                    const bool first = x1 >= x2;
                    const double xn = first ? x1 : x2;
                    sm = sm * pexp_lean(fmax(-745.0, mx - xn), thi, tlo);
                    mx = xn;
                    jm = (int)(j0 + (first ? c1 : c2));
                }
                const double e1 = pexp_lean(fmax(-745.0, x1 - mx), thi, tlo);
                const double e2 = pexp_lean(fmax(-745.0, x2 - mx), thi, tlo);
                sm += two ? e1 + e2 : e1;
            }
        }
        if (lane == 0) {
            if (A.count_surv && nsurv) atomicAdd(g_surv, (unsigned long long)nsurv);
            P.pa[(long long)sp * P.M + i] = mx;
            P.pb[(long long)sp * P.M + i] = sm;
            P.pj[(long long)sp * P.M + i] = jm;
        }
    }
}

// the sparse path's merge: one CTA per row block, then the launch finalize
__global__ void __launch_bounds__(kPT) lse_merge_kernel(PassArgs A) {
    __shared__ double thi[64], tlo[64];
    __shared__ double red[kPT / 32];
    __shared__ bool flag;
    if (A.check_done && A.ctl[0]) return;
    const PassSide &P = A.side[0];
    if (P.lctl[2 + P.lori] == A.lt) return;
    load_exp_table(A.tab, thi, tlo);
    __syncthreads();
    const int rb = blockIdx.x;
    const long long i = (long long)rb * kPT + threadIdx.x;
    const float w_lo = (float)A.w * (1.f - 0x1p-19f);
    lse_rowblock_finalize<32>(A, P, rb, i, i < P.M, thi, tlo, red, &flag, w_lo, false, true);
}

// =========================================================================
// Absorbed kernel-matrix half-sweeps over the certified candidate lists.
//
// Inside one Sinkhorn phase the cost term w D_ij of x_ij = q_j - w D_ij is fixed; only
// the column values q_j move.  With the record pass's values q_j^rec and a per-unit
// reference r_u (that pass's final mx), every listed entry is
//     exp(x_ij - r_u - c) = K_ij u_j,   K_ij = exp(q_j^rec - w D_ij - r_u),
//                                       u_j  = exp(q_j - q_j^rec - c),
// c = the split's largest column drift (any constant: it only keeps u_j <= ~1).  K is
// computed once per record (lse_kbuild_kernel, one exponential per listed entry) and
// stored as a sliced-ELL matrix per warp tile of 32 length-sorted ranks; a half-sweep is
// then one exponential per COLUMN and one FMA per listed entry -- a sparse
// matrix-vector product that streams 12 B per entry -- with partials (r_u + c, sum),
// merged like any other split partial.  The unit certificate of lse_sparse_kernel
// (unlisted entries are below the LSE cut, R10) is checked per pass; failed units go to
// lse_fallback_kernel.  Same mathematics as the log-domain pass, different rounding:
// every term carries a few ulps of relative error instead of the error of x - mx
// (DESIGN.md section 5).
// =========================================================================
// 1D bulk copy global -> shared by the TMA unit (SASS UBLKCP), completion on an mbarrier
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *mbar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
        ::"r"(tc::smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(tc::smem_u32(mbar))
        : "memory");
}

// per sorted rank: the unit's row, list length, certificate data (list bound lB, argmax seed
// column js with its distance -- the seed stays put between records: kernel-matrix passes
// leave jstar alone) and reference, one 32-byte record read by every half-sweep
struct __align__(16) KUnit {
    int i, cnt, js;
    float lB;
    double Dseed, mref;
};

template <int COST, int DP>
__global__ void __launch_bounds__(kPT) lse_kbuild_kernel(PassArgs A) {
    using DT = LDT<COST>;
    __shared__ double thi[64], tlo[64];
    const PassSide &P = A.side[0];
    if (P.lctl[2 + P.lori] != A.lt) return;          // only right after a record
    const int sp = blockIdx.x % P.S, lane = threadIdx.x & 31;
    const long long t = (long long)(blockIdx.x / P.S) * kPT + threadIdx.x;
    long long jb, je;
    split_range(P.N, P.S, sp, jb, je);
    load_exp_table(A.tab, thi, tlo);
    __syncthreads();
    const bool act = t < P.M;
    long long u = 0;
    int cnt = 0;
    double mref = 0.0;
    if (act) {
        const long long i = P.lperm[(long long)sp * P.M + t];
        u = (long long)sp * P.M + i;
        cnt = max(0, P.lcnt[u]);
        mref = P.pa[u];                              // the record pass's reference of this unit
        KUnit un;
        un.i = (int)i;
        un.cnt = P.lcnt[u];
        un.js = P.jstar[i];
        un.lB = P.lB[i];
        un.Dseed = 0.0;
        if (un.js >= 0 && un.js < P.N) {
            RowPt<COST, DP> rp;
            rp.load(P, i, true);
            un.Dseed = dist_global<COST, DP>(P, rp, i, un.js);
        } else {
            un.js = -1;
        }
        un.mref = mref;
        reinterpret_cast<KUnit *>(P.lunit)[(long long)sp * P.Mpad + t] = un;
    }
    // the tile is zero-padded to whole stages of kKB k-steps (lse_sort_kernel: lengths and
    // packing offsets)
    const bool tile = (t & ~31LL) < P.M;
    const long long te = (long long)sp * (P.Mpad / 32) + (t >> 5);
    int sbase = 0;
    for (int q = 0; q < sp; ++q) sbase += P.elltot[q];
    const int L = tile ? P.ellL[te] : 0;
    const int tabs = tile ? sbase + P.ellrel[te] : 0;
    const long long base = (long long)tabs * (kKB * 32) + lane;
    if (lane == 0 && tile) {
        P.ellabs[te] = tabs;
        atomicAdd(P.lctl + 10 + P.lori, L / kKB);       // stats: stages stored (512 entries each)
    }
    const DT *lD = reinterpret_cast<const DT *>(P.lD) + u * P.lcap;
    const int *lj = P.lj + u * P.lcap;
    const double w = A.w;
    for (int k = 0; k < L; ++k) {
        int jl = 0;
        double K = 0.0;
        if (k < cnt) {
            const int j = lj[k];
            const double x = fma(-w, (double)lD[k], P.lqd[j]);
            K = pexp(x - mref, thi, tlo);
            jl = (int)(j - jb);
        }
        P.ellj[base + (long long)k * 32] = jl;
        P.ellK[base + (long long)k * 32] = K;
    }
}

__global__ void __launch_bounds__(kPT) lse_ksweep_kernel(PassArgs A) {
    // dynamic shared memory: the ring (per warp kKNS stages of kKB k-steps), then u_j of
    // the split's columns
    extern __shared__ __align__(128) unsigned char lsm[];
    __shared__ double thi[64], tlo[64];
    __shared__ uint64_t kbar[kPT / 32][kKNS];
    if (A.check_done && A.ctl[0]) return;            // Sinkhorn phase already converged
    const PassSide &P = A.side[0];
    if (P.lctl[2 + P.lori] == A.lt) return;          // the dense pass recorded this half-sweep
    const int sp = blockIdx.x % P.S, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long t = (long long)(blockIdx.x / P.S) * kPT + threadIdx.x;
    long long jb, je;
    split_range(P.N, P.S, sp, jb, je);
    load_exp_table(A.tab, thi, tlo);
    // The warp's tile is one contiguous block of L x 32 entries per array: stages of kKB
    // k-steps are brought into the warp's ring by 1D bulk copies (lane 0 issues, the TMA
    // unit completes on the stage's mbarrier), kKNS stages in flight -- memory-level
    // parallelism without registers.  The first stages are issued before anything else,
    // so the certificate and the column factors below overlap their latency.
    const bool tile = (t & ~31LL) < P.M;
    const long long te = (long long)sp * (P.Mpad / 32) + (t >> 5);
    const long long tile0 = tile ? (long long)P.ellabs[te] * (kKB * 32) : 0;
    unsigned char *ring = lsm + warp * (kKNS * (kKStJ + kKStK));
    uint64_t *bar = kbar[warp];
    const int nb = tile ? P.ellL[te] / kKB : 0;
    auto issue = [&](int b) {
        const int st = b % kKNS;
        unsigned char *dst = ring + st * (kKStJ + kKStK);
        mbar_expect_tx(&bar[st], kKStJ + kKStK);
        bulk_load(dst, P.ellK + tile0 + (long long)b * (kKB * 32), kKStK, &bar[st]);
        bulk_load(dst + kKStK, P.ellj + tile0 + (long long)b * (kKB * 32), kKStJ, &bar[st]);
    };
    if (lane == 0) {
        for (int st = 0; st < kKNS; ++st) tc::mbar_init(&kbar[warp][st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        for (int b = 0; b < min(nb, kKNS); ++b) issue(b);
    }
    KUnit kun;
    kun.i = 0; kun.cnt = 0; kun.js = -1; kun.lB = 0.f; kun.Dseed = 0.0; kun.mref = 0.0;
    if (t < P.M) kun = reinterpret_cast<const KUnit *>(P.lunit)[(long long)sp * P.Mpad + t];
    const double qseed = kun.js >= 0 ? __ldg(P.lqv + kun.js) : 0.0;
    __syncthreads();
    const float dq = P.ldqs[sp];
    const double shift = (dq == dq && fabsf(dq) != INFINITY) ? (double)dq : 0.0;
    double *su = reinterpret_cast<double *>(lsm + kKRing);
    for (long long j = jb + threadIdx.x; j < je; j += kPT) {
        const double q = __ldg(P.lqv + j), qr = __ldg(P.lqd + j);
        su[j - jb] = (q == -INFINITY || qr == -INFINITY) ? 0.0 : pexp(q - qr - shift, thi, tlo);
    }
    __syncthreads();
    long long u = 0;
    int cnt = 0;
    double mref = 0.0;
    bool ok = false;
    if (t < P.M) {
        const KUnit un = kun;
        u = (long long)sp * P.M + un.i;
        cnt = un.cnt;
        mref = un.mref;
        // the unit certificate of lse_sparse_kernel: no unlisted entry can pass the LSE cut
        const double mx = un.js >= 0 ? fma(-A.w, un.Dseed, qseed) : -INFINITY;
        const float thr0 = thr_lo_of(mx - kLseCut);
        const float B = un.lB;
        const double ub = (double)B + (double)ulpf_of(B) + (double)dq;
        ok = cnt >= 0 && thr0 != -INFINITY && dq != INFINITY &&
             ub + 1e-12 * (fabs((double)B) + fabs((double)dq)) <= (double)thr0;
        if (!ok) P.lq[atomicAdd(P.lctl + 8, 1)] = (int)u;     // dense scan (fallback kernel)
    }
    // lanes past their own list read the tile's zero padding (K = 0, column 0)
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    for (int b = 0; b < nb; ++b) {
        const int st = b % kKNS;
        tc::mbar_wait(&bar[st], (uint32_t)((b / kKNS) & 1));
        const double *sK = reinterpret_cast<const double *>(ring + st * (kKStJ + kKStK)) + lane;
        const int *sj = reinterpret_cast<const int *>(ring + st * (kKStJ + kKStK) + kKStK) + lane;
#pragma unroll
        for (int q = 0; q < kKB; q += 4) {
            s0 = fma(sK[(q + 0) * 32], su[sj[(q + 0) * 32]], s0);
            s1 = fma(sK[(q + 1) * 32], su[sj[(q + 1) * 32]], s1);
            s2 = fma(sK[(q + 2) * 32], su[sj[(q + 2) * 32]], s2);
            s3 = fma(sK[(q + 3) * 32], su[sj[(q + 3) * 32]], s3);
        }
        __syncwarp();                                // every lane is done with this stage
        if (lane == 0 && b + kKNS < nb) issue(b + kKNS);
    }
    count_survivors(A.count_surv, 2, ok && cnt > 0 ? cnt : 0);       // ELL entries walked (profiling)
    if (!ok) return;
    const double sm = (s0 + s1) + (s2 + s3);
    if (cnt > 0 && !(sm > 1e-280)) {                 // every listed term underflowed: exact dense scan
        P.lq[atomicAdd(P.lctl + 8, 1)] = (int)u;
        return;
    }
    P.pa[u] = cnt > 0 ? mref + shift : -INFINITY;
    P.pb[u] = sm;
    P.pj[u] = -1;
}

// Dense scan of the units whose certificate failed, kernel-matrix mode: one warp per
// unit, every lane an online log-sum-exp over its columns (j = jb + lane, + 32, ...),
// combined in lane order.  (The list-walk mode needs the dense pass's survivor sequence
// -- lse_fallback_kernel; here only the sums matter.)
template <int COST, int DP>
__global__ void __launch_bounds__(kPT) lse_fallback_k_kernel(PassArgs A) {
    __shared__ double thi[64], tlo[64];
    if (A.check_done && A.ctl[0]) return;
    const PassSide &P = A.side[0];
    if (P.lctl[2 + P.lori] == A.lt) return;
    const int nq = P.lctl[8];
    if (nq == 0) return;
    load_exp_table(A.tab, thi, tlo);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long gw = ((long long)blockIdx.x * kPT + threadIdx.x) >> 5, nw = (long long)gridDim.x * (kPT / 32);
    const double w = A.w;
    for (long long qi = gw; qi < nq; qi += nw) {
        const int u = P.lq[qi];
        const long long i = u % P.M;
        const int sp = (int)(u / P.M);
        long long jb, je;
        split_range(P.N, P.S, sp, jb, je);
        RowPt<COST, DP> rp;
        rp.load(P, i, true);
        double mx = -INFINITY, sm = 0.0;
        for (long long j0 = jb + lane; j0 < je; j0 += 256) {      // 8 columns per lane and step: loads first
            double x[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const long long j = j0 + 32 * q;
                x[q] = j < je ? fma(-w, dist_global<COST, DP>(P, rp, i, j), __ldg(P.lqv + j)) : -INFINITY;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (x[q] == -INFINITY) continue;
                if (x[q] > mx) {
                    sm = fma(sm, pexp(mx - x[q], thi, tlo), 1.0);
                    mx = x[q];
                } else {
                    sm += pexp(x[q] - mx, thi, tlo);
                }
            }
        }
        const double Mx = warp_max(mx);
        const double tot = warp_sum(mx == -INFINITY ? 0.0 : sm * pexp(mx - Mx, thi, tlo));
        if (lane == 0) {
            P.pa[(long long)sp * P.M + i] = Mx;
            P.pb[(long long)sp * P.M + i] = tot;
            P.pj[(long long)sp * P.M + i] = -1;
        }
    }
}

// =========================================================================
// Evaluation pass, both orientations in one launch.
// Block scalars (per side, row block rb): [0] sum|grad| [1] sum of sums
// [2] sum X D [3] sum X em1 [4] max z [5] max count [6] sum min(count, cap).
// Launch stats st[]: 0 |grad_f|_1, 1 |grad_g|_1, 2 sum X, 3 sum X D (unscaled),
// 4 trial sum, 5 max z, 6 max count, 7 nnz side 0, 8 <a,f>+<b,g>,
// 9 max row sum, 10 max column sum, 11 nnz side 1.
// =========================================================================
template <int COST, int DP, class TS>
__device__ __forceinline__ void sum_side(const PassArgs &A, const PassSide &P, int bid, Buf<COST, DP> *bufs,
                                         TS &tcs, float *dscr, double *thi, double *tlo, double *red,
                                         bool *flag, int side, unsigned char *dyn, uint64_t *ring_full,
                                         const CUtensorMap *tm) {
    const int tid = threadIdx.x;
    const int rb = bid % P.RB, sp = bid / P.RB;
    const long long i0 = (long long)rb * kPT, i = i0 + tid;
    const bool valid = i < P.M;
    long long jb, je;
    split_range(P.N, P.S, sp, jb, je);
    if constexpr (COST == PC_SQTC) tc_setup(tcs, P, i0);
    RowPt<COST, DP> rp;
    rp.load(P, i, valid);
    const double w = A.w, inv_eta = A.inv_eta;
    double Pi = 0.0, eu = 0.0, bu = 0.0;
    if (valid) {
        Pi = P.m1_row ? pot_p(P.fr[i], P.phir[i], inv_eta) : pot_q(P.fr[i], P.phir[i], inv_eta);
        if (P.eu) { eu = P.eu[i]; bu = P.bu[i]; }
    }
    const bool trial = P.eu != nullptr, sparse = P.tau > 0.0;
    // skip test in the form fma(-w, D, qt_j) > thr_i (qt = q + bump_j): the exact z is
    // only formed for entries that pass (R10); near the cut the two orientations may
    // decide differently, which changes sums by < e^-80 and never the kept pattern
    const double thr = -kSumCut - Pi - bu;
    const float thr32 = thr_lo_of(thr);
    const float w_lo = (float)w * (1.f - 0x1p-19f);
    double acc = 0.0, cx = 0.0, em = 0.0, mz = -INFINITY;
    int cnt = 0;
    const long long bufbase = (i * P.S + sp) * P.cap;
    float *dsc = dscr + tid * (kCC + 1);
    int nsurv = 0;
    const SkipCtx sk = skip_setup(P, rb, sp, i, valid, jb, thr32, w_lo, red);
    const TmaRing ring = ring_setup<COST>(dyn, ring_full, tm, i0);
    const int nskip = stream_columns<COST, DP>(P, i0, jb, je, inv_eta, P.m1_row ? 0 : 1, trial, bufs, &tcs, sk, ring,
                             [&](long long j0, int nc, const Buf<COST, DP> &B, const float *dots,
                                 const unsigned char *tile) {
        unsigned mask = 0u;
        float vmx = -INFINITY, dmn = INFINITY;
        float Dv[kDv<COST> ? kCC : 1];
        if (valid) {
            if (sk.kind == 2) mask = phase1<COST, DP, true>(B, P, rp, i, j0, nc, dots, w_lo, thr32, Dv, vmx, dmn, tile);
            else mask = phase1<COST, DP, false>(B, P, rp, i, j0, nc, dots, w_lo, thr32, Dv, vmx, dmn, tile);
        }
        if (sk.kind == 2) record_cert(sk, j0, vmx, thr32, valid, dmn);
        nsurv += __popc(mask);
        if (!valid) return;
        if constexpr (COST == PC_SQTC) {
            // distances are needed only where some lane of the warp has a survivor
            if (__any_sync(__activemask(), mask != 0u)) {
#pragma unroll
                for (int c = 0; c < kCC; ++c) dsc[c] = Dv[c];
            }
        }
        while (mask) {
            const int c = __ffs(mask) - 1;
            mask &= mask - 1u;
            double D;
            if constexpr (COST == PC_SQTC) D = (double)dsc[c];
            else D = chunk_dist<COST, DP>(B, P, rp, i, j0, c, tile);
            const double z = fma(-w, D, __dadd_rn(Pi, B.q[c]));
            const double X = pexp_lean(fmin(709.0, fmax(-745.0, z)), thi, tlo);
            acc += X;
            mz = fmax(mz, z);
            if (P.want_cx) cx = fma(X, D, cx);
            if (trial) {
                const double ev = B.ev[c];
                em = fma(X, fma(eu, ev, eu + ev), em);
            }
            if (sparse && X >= P.tau) {
                if (cnt < P.cap) {
                    P.bcol[bufbase + cnt] = (int)(j0 + c);
                    P.bval[bufbase + cnt] = X;
                }
                ++cnt;
            }
        }
    });
    if constexpr (COST == PC_SQTC) tc_teardown(tcs);
    skip_count(P, sk, nskip, jb, je);
    count_survivors(A.count_surv, 1, nsurv);
    if (valid) {
        P.pa[(long long)sp * P.M + i] = acc;
        if (sparse) P.cnt[i * P.S + sp] = cnt;
    }
    // split-level scalars (per CTA)
    const double bcx = block_reduce_sum(cx, red);
    const double bem = block_reduce_sum(em, red);
    const double bmz = block_reduce_max(mz, red);
    if (tid == 0) {
        P.psc[((long long)sp * P.RB + rb) * 4 + 0] = bcx;
        P.psc[((long long)sp * P.RB + rb) * 4 + 1] = bem;
        P.psc[((long long)sp * P.RB + rb) * 4 + 2] = bmz;
    }
    if (!last_arrival(P.ticket + rb, (unsigned)P.S, flag)) return;
    // ---- row-block finalize ----
    double g1 = 0.0, sr = 0.0, mc = 0.0, nn = 0.0;
    if (valid) {
        double s = 0.0;
        for (int q = 0; q < P.S; ++q) s += P.pa[(long long)q * P.M + i];
        P.sum[i] = s;
        const double gr = P.ar[i] - s;
        P.grad[i] = gr;
        g1 = fabs(gr);
        sr = s;
        if (sparse) {
            for (int q = 0; q < P.S; ++q) {
                const int c = P.cnt[i * P.S + q];
                mc = fmax(mc, (double)c);
                nn += (double)min((long long)c, P.cap);
            }
        }
    }
    double tcx = 0.0, tem = 0.0, tmz = -INFINITY;
    if (tid == 0) {
        for (int q = 0; q < P.S; ++q) {
            tcx += P.psc[((long long)q * P.RB + rb) * 4 + 0];
            tem += P.psc[((long long)q * P.RB + rb) * 4 + 1];
            tmz = fmax(tmz, P.psc[((long long)q * P.RB + rb) * 4 + 2]);
        }
    }
    const double bg = block_reduce_sum(g1, red);
    const double bs = block_reduce_sum(sr, red);
    const double bmc = block_reduce_max(mc, red);
    const double bnn = block_reduce_sum(nn, red);
    if (tid == 0) {
        double *o = P.blk + rb * 8;
        o[0] = bg;
        o[1] = bs;
        o[2] = tcx;
        o[3] = tem;
        o[4] = tmz;
        o[5] = bmc;
        o[6] = bnn;
        o[7] = 0.0;
    }
    (void)side;
}

template <int COST0, int COST1, int DP>
__global__ void __launch_bounds__(kPT) sum_pass_kernel(PassArgs A, const __grid_constant__ CUtensorMap tm0,
                                                       const __grid_constant__ CUtensorMap tm1) {
    extern __shared__ __align__(1024) unsigned char dyn_smem[];   // TMA ring (dense costs) or unused
    __shared__ uint64_t ring_full[kNSt];
    constexpr size_t kB0 = sizeof(Buf<COST0, DP>) * kNBuf<COST0>, kB1 = sizeof(Buf<COST1, DP>) * kNBuf<COST1>;
    __shared__ __align__(128) unsigned char smraw[kB0 > kB1 ? kB0 : kB1];
    __shared__ TcFor<(COST0 == PC_SQTC || COST1 == PC_SQTC) ? PC_SQTC : COST0> tcs;
    __shared__ float dscr[(COST0 == PC_SQTC || COST1 == PC_SQTC) ? kPT * (kCC + 1) : 1];
    __shared__ double thi[64], tlo[64];
    __shared__ double red[kPT / 32];
    __shared__ bool flag;
    load_exp_table(A.tab, thi, tlo);
    const int side = (blockIdx.x < (unsigned)A.G0) ? 0 : 1;
    const int bid = side == 0 ? blockIdx.x : blockIdx.x - A.G0;
    if (side == 0)
        sum_side<COST0, DP>(A, A.side[0], bid, reinterpret_cast<Buf<COST0, DP> *>(smraw), tcs, dscr, thi, tlo, red,
                            &flag, 0, dyn_smem, ring_full, &tm0);
    else
        sum_side<COST1, DP>(A, A.side[1], bid, reinterpret_cast<Buf<COST1, DP> *>(smraw), tcs, dscr, thi, tlo, red,
                            &flag, 1, dyn_smem, ring_full, &tm1);
    // only row-block finalizers continue past here with flag set
    if (!flag) return;
    const unsigned tot = (unsigned)(A.side[0].RB + (A.nsides > 1 ? A.side[1].RB : 0));
    if (!last_arrival(A.gticket, tot, &flag)) return;
    // ---- launch finalize (one CTA): deterministic merges ----
    const int tid = threadIdx.x;
    double v[2][7];
    for (int s2 = 0; s2 < 2; ++s2) {
        double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = -INFINITY, a5 = 0, a6 = 0;
        if (s2 < A.nsides) {
            const PassSide &P = A.side[s2];
            for (int b = tid; b < P.RB; b += kPT) {
                const double *o = P.blk + b * 8;
                a0 += o[0]; a1 += o[1]; a2 += o[2]; a3 += o[3];
                a4 = fmax(a4, o[4]); a5 = fmax(a5, o[5]); a6 += o[6];
            }
        }
        v[s2][0] = block_reduce_sum(a0, red);
        v[s2][1] = block_reduce_sum(a1, red);
        v[s2][2] = block_reduce_sum(a2, red);
        v[s2][3] = block_reduce_sum(a3, red);
        v[s2][4] = block_reduce_max(a4, red);
        v[s2][5] = block_reduce_max(a5, red);
        v[s2][6] = block_reduce_sum(a6, red);
    }
    // <a,f> + <b,g>, max row / column sums
    double dot = 0.0, mr = 0.0, mcol = 0.0;
    if (A.a_dot) {
        const PassSide &P0 = A.side[0];
        for (long long k = tid; k < P0.M; k += kPT) dot = fma(A.a_dot[k], A.f_dot[k], dot);
        for (long long k = tid; k < P0.N; k += kPT) dot = fma(A.b_dot[k], A.g_dot[k], dot);
    }
    for (long long k = tid; k < A.side[0].M; k += kPT) mr = fmax(mr, A.side[0].sum[k]);
    if (A.nsides > 1)
        for (long long k = tid; k < A.side[1].M; k += kPT) mcol = fmax(mcol, A.side[1].sum[k]);
    const double Dt = block_reduce_sum(dot, red);
    const double Mr = block_reduce_max(mr, red);
    const double Mc = block_reduce_max(mcol, red);
    if (tid == 0) {
        A.st[0] = v[0][0];
        A.st[1] = A.nsides > 1 ? v[1][0] : 0.0;
        A.st[2] = v[0][1];
        A.st[3] = v[0][2];
        A.st[4] = v[0][3];
        A.st[5] = fmax(v[0][4], A.nsides > 1 ? v[1][4] : -INFINITY);
        A.st[6] = fmax(v[0][5], A.nsides > 1 ? v[1][5] : 0.0);
        A.st[7] = v[0][6];
        A.st[8] = Dt;
        A.st[9] = Mr;
        A.st[10] = Mc;
        A.st[11] = A.nsides > 1 ? v[1][6] : 0.0;
        const float wl = (float)A.w * (1.f - 0x1p-19f);
        for (int s2 = 0; s2 < A.nsides; ++s2) skip_switch(A.side[s2], wl);
        // row-block bases of the CSR / CSC (sequential scan, RB is small)
        for (int s2 = 0; s2 < A.nsides; ++s2) {
            const PassSide &P = A.side[s2];
            if (!P.blkoff) continue;
            long long acc = 0;
            for (int b = 0; b < P.RB; ++b) {
                P.blkoff[b] = acc;
                acc += (long long)P.blk[b * 8 + 6];
            }
            P.blkoff[P.RB] = acc;
        }
    }
}

}  // namespace pins

namespace pins {

// CSR (side 0) / CSC (side 1) assembly from the per-(row, split) buffers.
// blkoff[b] (exclusive scan of the row-block nnz totals, written by the sum
// pass's launch finalizer) gives each row block its base; inside the block a
// shared-memory scan over the 128 rows gives each row its start.  Thread =
// pass row; columns stay ascending (splits are ascending column ranges).
struct CsrOut {
    long long *ptr;
    int *idx;
    double *val;
    const long long *blkoff;
};

__global__ void __launch_bounds__(kPT) csr_build_kernel(PassSide P0, PassSide P1, int nsides, CsrOut O0,
                                                        CsrOut O1, int warpcopy) {
    __shared__ long long sc[kPT];
    const int side = (blockIdx.x < (unsigned)P0.RB) ? 0 : 1;
    if (side == 1 && nsides < 2) return;
    const PassSide &P = side == 0 ? P0 : P1;
    const CsrOut &O = side == 0 ? O0 : O1;
    const int rb = side == 0 ? blockIdx.x : blockIdx.x - P0.RB;
    const int tid = threadIdx.x;
    const long long i = (long long)rb * kPT + tid;
    long long tot = 0;
    if (i < P.M) {
#pragma unroll 8
        for (int s = 0; s < P.S; ++s) tot += min((long long)P.cnt[i * P.S + s], P.cap);
    }
    sc[tid] = tot;
    __syncthreads();
    for (int o = 1; o < kPT; o <<= 1) {
        const long long t = tid >= o ? sc[tid - o] : 0;
        __syncthreads();
        sc[tid] += t;
        __syncthreads();
    }
    const long long start = O.blkoff[rb] + sc[tid] - tot;
    __shared__ long long rstart_s[kPT];
    rstart_s[tid] = start;
    if (i < P.M && i == P.M - 1) O.ptr[P.M] = start + tot;
    if (i < P.M) O.ptr[i] = start;
    if (!warpcopy) {                                   // short rows: thread per row
        if (i < P.M) {
            long long dst = start;
            for (int s0 = 0; s0 < P.S; s0 += 8) {
                int len[8];
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    len[j] = s0 + j < P.S ? (int)min((long long)P.cnt[i * P.S + s0 + j], P.cap) : 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const long long src = (i * P.S + s0 + j) * P.cap;
                    for (int k = 0; k < len[j]; ++k) {
                        O.idx[dst + k] = P.bcol[src + k];
                        O.val[dst + k] = P.bval[src + k];
                    }
                    dst += len[j];
                }
            }
        }
        return;
    }
    __syncthreads();
    // copy: one warp per row, lane = split segment (exclusive scan of the segment
    // lengths across the lanes gives each segment's offset inside the row)
    const int lane = tid & 31, warp = tid >> 5;
    for (int rr = warp; rr < kPT; rr += kPT / 32) {
        const long long ii = (long long)rb * kPT + rr;
        if (ii >= P.M) break;
        long long dst = rstart_s[rr];
        for (int s0 = 0; s0 < P.S; s0 += 32) {
            const int s = s0 + lane;
            const int len = s < P.S ? (int)min((long long)P.cnt[ii * P.S + s], P.cap) : 0;
            int x = len;
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += t;
            }
            const long long my = dst + x - len;
            const long long src = (ii * P.S + s) * P.cap;
            for (int k = 0; k < len; ++k) {
                O.idx[my + k] = P.bcol[src + k];
                O.val[my + k] = P.bval[src + k];
            }
            dst += __shfl_sync(0xffffffffu, x, 31);
        }
    }
}

// fp16 copy of padded fp32 points (rows of 16; exact for integers |x| <= 2048)
__global__ void to_half16_kernel(long long np, int dp, const float *x32, __half *xh) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < np * 16;
         t += (long long)gridDim.x * blockDim.x) {
        const long long p = t >> 4;
        const int k = (int)(t & 15);
        xh[t] = __float2half_rn(k < dp ? x32[p * dp + k] : 0.f);
    }
}

// Point preparation: zero-padded fp32 / fp64 copies (row stride dp), fp32
// squared norms, and the exactness facts the host needs to pick the fp32 path:
// info[0] = max |coord| (as ordered bits), info[1] = max squared norm,
// info[2] = number of non-integer coordinates.
__global__ void prep_points_kernel(long long np, int d, int dp, const double *x, float *x32, double *x64,
                                   float *n32, unsigned long long *info) {
    double amax = 0.0, nmax = 0.0;
    unsigned long long nonint = 0;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < np;
         p += (long long)gridDim.x * blockDim.x) {
        double nr = 0.0;
        for (int k = 0; k < dp; ++k) {
            const double v = k < d ? x[p * d + k] : 0.0;
            x32[p * dp + k] = (float)v;
            x64[p * dp + k] = v;
            nr = fma(v, v, nr);
            amax = fmax(amax, fabs(v));
            nonint += (v != rint(v)) ? 1ull : 0ull;
        }
        n32[p] = (float)nr;
        nmax = fmax(nmax, nr);
    }
    amax = warp_max(amax);
    nmax = warp_max(nmax);
    for (int o = 16; o > 0; o >>= 1) nonint += __shfl_xor_sync(0xffffffffu, nonint, o);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(info + 0, (unsigned long long)__double_as_longlong(amax));
        atomicMax(info + 1, (unsigned long long)__double_as_longlong(nmax));
        atomicAdd(info + 2, nonint);
    }
}

// Dense plan materialisation X~(f, g) (Eq. (7); pins_plan).  The exponent is
// formed exactly as in sum_pass_kernel -- z = fma(-w, D, pot_p(f, phi) +
// pot_q(g, psi)), no FMA contraction of the potentials, D in the same operation
// order -- and pexp agrees with pexp_lean bit for bit on the pass's clamp range,
// so every entry the sum pass keeps (X~ >= tau) has the same bits here: the
// sparsifier's parity test thresholds this plan on the host.
template <int KIND>
__global__ void plan_kernel(long long m, long long n, CostDesc cd, const double *f,
                            const double *phi, const double *g, const double *psi,
                            double inv_eta, double w, const ExpTable *tab, double *X, long long ldx) {
    __shared__ double thi[64], tlo[64];
    load_exp_table(tab, thi, tlo);
    __syncthreads();
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m * n;
         e += (long long)gridDim.x * blockDim.x) {
        const long long i = e / n, j = e % n;
        double D;
        if constexpr (KIND == 0) {
            D = cd.C[i * cd.ldc + j];
        } else {
            double s = 0.0;
            for (int k = 0; k < cd.d; ++k) {
                const double t = cd.x[i * cd.d + k] - cd.y[j * cd.d + k];
                s = (KIND == 1) ? fma(t, t, s) : s + fabs(t);
            }
            D = s;
        }
        const double z = fma(-w, D, __dadd_rn(pot_p(f[i], phi[i], inv_eta), pot_q(g[j], psi[j], inv_eta)));
        X[i * ldx + j] = pexp(z, thi, tlo);
    }
}

}  // namespace pins
