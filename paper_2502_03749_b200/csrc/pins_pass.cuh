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
// so each skipped term is < e^-50 of the largest; in the sums an entry is
// skipped when z < -kSumCut (X~ < 1.8e-35).  DESIGN.md §5 bounds the effect.
//
// Reductions are deterministic: per (split, row) partials, merged in split
// order by the last CTA of each row block (atomic ticket), then per-block
// scalars merged in block order by the last row block of the launch.
#pragma once
#include "pins_device.cuh"

namespace pins {

constexpr int kPT = 128;            // threads per CTA = pass rows per CTA
constexpr int kCC = 32;             // columns per staged chunk
constexpr double kLseCut = 50.0;
constexpr double kSumCut = 80.0;

// cost evaluation variants (host picks, see pins_api.cu choose_cost)
enum : int {
    PC_DENSE_ROW = 0,   // dense C, row orientation: tile staged through smem
    PC_DENSE_COL = 1,   // dense C, column orientation: C[i*ldc + j] read directly (coalesced)
    PC_SQ32 = 2,        // integer points, exact in fp32: D = |x|^2 + |y|^2 - 2 x.y
    PC_L132 = 3,        // integer points, exact in fp32: D = sum |x - y|
    PC_SQ64 = 4,        // generic points, fp64: D = sum (x - y)^2
    PC_L164 = 5,        // generic points, fp64: D = sum |x - y|
};

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
    int count_sweep;                // LSE col pass: ++ctl[1]
    int test_tol;                   // LSE row pass: set done (and rollback) when res <= tol
    const double *a_dot, *f_dot, *b_dot, *g_dot;   // SUM: <a,f> + <b,g> (global finalize)
};

// exact potential expressions (no FMA contraction: identical bits in both orientations)
__device__ __forceinline__ double pot_q(double g, double psi, double inv_eta) {
    return __dmul_rn(__dadd_rn(g, psi), inv_eta);
}
__device__ __forceinline__ double pot_p(double f, double phi, double inv_eta) {
    return __dsub_rn(__dmul_rn(__dadd_rn(f, phi), inv_eta), 1.0);
}

// ---------------------------------------------------------------- staging
// Per chunk: kCC pass columns j0 .. j0+kCC-1 (tail-padded).
template <int COST, int DP>
struct Stage {
    static constexpr int NY32 = (COST == PC_SQ32 || COST == PC_L132) ? kCC * DP : 4;
    static constexpr int NY64 = (COST == PC_SQ64 || COST == PC_L164) ? kCC * DP : 1;
    static constexpr int NT = (COST == PC_DENSE_ROW) ? kCC * (kPT + 1) : 1;
    double q[kCC];                  // column potential
    double ev[kCC], bv[kCC];        // trial factors / bumps
    double y64[NY64];               // fp64 points
    double tile[NT];                // dense row orientation: C[i0 + r][j0 + c] -> tile[c * (kPT+1) + r]
    alignas(16) float y32[NY32];    // fp32 points
    float ny[kCC];
};

template <int COST, int DP>
__device__ __forceinline__ void stage_cost(Stage<COST, DP> &sg, const PassSide &P, long long i0, long long j0,
                                           int nc) {
    const int tid = threadIdx.x;
    if constexpr (COST == PC_SQ32 || COST == PC_L132) {
        for (int t = tid; t < kCC * DP; t += kPT) {
            const int c = t / DP;
            sg.y32[t] = (c < nc) ? P.yc32[(j0 + c) * DP + (t - c * DP)] : 0.f;
        }
        if (COST == PC_SQ32)
            for (int c = tid; c < kCC; c += kPT) sg.ny[c] = (c < nc) ? P.nyc[j0 + c] : 0.f;
    } else if constexpr (COST == PC_SQ64 || COST == PC_L164) {
        for (int t = tid; t < kCC * DP; t += kPT) {
            const int c = t / DP;
            sg.y64[t] = (c < nc) ? P.yc64[(j0 + c) * DP + (t - c * DP)] : 0.0;
        }
    } else if constexpr (COST == PC_DENSE_ROW) {
        // rows i0 .. i0+kPT-1 of C, columns j0 .. j0+kCC-1: warp w loads rows w, w+4, ...;
        // lane = column (coalesced 256 B per row); stored transposed with a pad column
        const int lane = tid & 31, warp = tid >> 5;
        const long long rows = P.M - i0;
        for (int r = warp; r < kPT; r += kPT / 32) {
            double v = 0.0;
            if (r < rows && lane < nc) v = __ldg(P.C + (i0 + r) * P.ldc + j0 + lane);
            sg.tile[lane * (kPT + 1) + r] = v;
        }
    }
}

// distance of the thread's pass row to staged column c (as fp64)
template <int COST, int DP>
struct RowPt {
    float x32[DP > 0 ? DP : 1];
    float nx;
    double x64[DP > 0 ? DP : 1];
    __device__ __forceinline__ void load(const PassSide &P, long long i, bool valid) {
        if constexpr (COST == PC_SQ32 || COST == PC_L132) {
#pragma unroll
            for (int k = 0; k < DP; ++k) x32[k] = valid ? P.xr32[i * DP + k] : 0.f;
            nx = (COST == PC_SQ32 && valid) ? P.nxr[i] : 0.f;
        } else if constexpr (COST == PC_SQ64 || COST == PC_L164) {
#pragma unroll
            for (int k = 0; k < DP; ++k) x64[k] = valid ? P.xr64[i * DP + k] : 0.0;
        }
    }
    // D(i, j) from the staged chunk (points kinds)
    __device__ __forceinline__ double dist(const Stage<COST, DP> &sg, int c) const {
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
    if constexpr (COST == PC_DENSE_ROW) return P.C[i * P.ldc + j];
    else if constexpr (COST == PC_DENSE_COL) return P.C[j * P.ldc + i];
    else if constexpr (COST == PC_SQ32) {
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

template <int COST, int DP>
__device__ __forceinline__ double chunk_dist(const Stage<COST, DP> &sg, const PassSide &P,
                                             const RowPt<COST, DP> &rp, long long i, long long j, int c,
                                             bool valid) {
    if constexpr (COST == PC_DENSE_ROW) return sg.tile[c * (kPT + 1) + threadIdx.x];
    else if constexpr (COST == PC_DENSE_COL) return valid ? __ldg(P.C + j * P.ldc + i) : 0.0;
    else return rp.dist(sg, c);
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

// =========================================================================
// LSE half-sweep.  One side per launch (A.side[0]).
// Stats written by the global finalizer: st[0] = residual ||a - X~ e||_1 of
// the starting iterate (pass-row side), st[1] = max |f_new - f_old|.
// =========================================================================
template <int COST, int DP>
__global__ void __launch_bounds__(kPT) lse_pass_kernel(PassArgs A) {
    __shared__ Stage<COST, DP> sg;
    __shared__ double thi[64], tlo[64];
    __shared__ double red[kPT / 32];
    __shared__ bool flag;
    if (A.check_done && A.ctl[0]) return;            // Sinkhorn phase already converged
    const PassSide &P = A.side[0];
    const int tid = threadIdx.x;
    const int rb = blockIdx.x % P.RB, sp = blockIdx.x / P.RB;
    const long long i0 = (long long)rb * kPT, i = i0 + tid;
    const bool valid = i < P.M;
    const long long jb = P.N * sp / P.S, je = P.N * (sp + 1) / P.S;
    load_exp_table(A.tab, thi, tlo);
    RowPt<COST, DP> rp;
    rp.load(P, i, valid);
    const double w = A.w, inv_eta = A.inv_eta;
    double mx = -INFINITY, sm = 0.0;
    int jm = -1;
    if (valid) {
        const int js = P.jstar[i];
        if (js >= 0 && js < P.N) {     // lower bound of the row max: one true entry
            const double D = dist_global<COST, DP>(P, rp, i, js);
            mx = fma(-w, D, pot_q(P.gc[js], P.psic[js], inv_eta));
        }
    }
    for (long long j0 = jb; j0 < je; j0 += kCC) {
        const int nc = (int)min((long long)kCC, je - j0);
        __syncthreads();
        for (int c = tid; c < kCC; c += kPT) sg.q[c] = (c < nc) ? pot_q(P.gc[j0 + c], P.psic[j0 + c], inv_eta) : -INFINITY;
        stage_cost<COST, DP>(sg, P, i0, j0, nc);
        __syncthreads();
        if (valid) {
#pragma unroll 4
            for (int c = 0; c < kCC; ++c) {
                if (c < nc) {
                    const double D = chunk_dist<COST, DP>(sg, P, rp, i, j0 + c, c, valid);
                    const double x = fma(-w, D, sg.q[c]);
                    if (x > mx - kLseCut) {
                        if (x > mx) {
                            sm = fma(sm, pexp(mx - x, thi, tlo), 1.0);
                            mx = x;
                            jm = (int)(j0 + c);
                        } else {
                            sm += pexp(x - mx, thi, tlo);
                        }
                    }
                }
            }
        }
    }
    if (valid) {
        P.pa[(long long)sp * P.M + i] = mx;
        P.pb[(long long)sp * P.M + i] = sm;
        P.pj[(long long)sp * P.M + i] = jm;
    }
    if (!last_arrival(P.ticket + rb, (unsigned)P.S, &flag)) return;
    // ---- row-block finalize: merge the S splits (in split order) ----
    double res = 0.0, dmax = 0.0;
    if (valid) {
        double M = -INFINITY;
        int jbest = -1;
        for (int s = 0; s < P.S; ++s) {
            const double v = P.pa[(long long)s * P.M + i];
            if (v > M) { M = v; jbest = P.pj[(long long)s * P.M + i]; }
        }
        double Ssum = 0.0;
        for (int s = 0; s < P.S; ++s) {
            const double v = P.pa[(long long)s * P.M + i];
            const double c = P.pb[(long long)s * P.M + i];
            if (c > 0.0) Ssum += c * pexp(v - M, thi, tlo);
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
    }
    const double bres = block_reduce_sum(res, red);
    const double bdm = block_reduce_max(dmax, red);
    if (tid == 0) {
        P.blk[rb * 8 + 0] = bres;
        P.blk[rb * 8 + 1] = bdm;
    }
    if (!last_arrival(A.gticket, (unsigned)P.RB, &flag)) return;
    // ---- launch finalize ----
    double v0 = 0.0, v1 = 0.0;
    for (int b = tid; b < P.RB; b += kPT) {     // deterministic: fixed assignment + fixed tree
        v0 += P.blk[b * 8 + 0];
        v1 = fmax(v1, P.blk[b * 8 + 1]);
    }
    const double R = block_reduce_sum(v0, red);
    const double DM = block_reduce_max(v1, red);
    if (tid == 0) {
        A.st[0] = R;
        A.st[1] = DM;
        if (A.count_sweep) A.ctl[1] += 1;
        if (A.test_tol && A.sink_tol && R <= *A.sink_tol) {
            A.ctl[0] = 1;     // converged at the starting iterate: roll back this update
            A.ctl[2] = 1;
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
template <int COST, int DP>
__device__ __forceinline__ void sum_side(const PassArgs &A, const PassSide &P, int bid, Stage<COST, DP> &sg,
                                         double *thi, double *tlo, double *red, bool *flag, int side) {
    const int tid = threadIdx.x;
    const int rb = bid % P.RB, sp = bid / P.RB;
    const long long i0 = (long long)rb * kPT, i = i0 + tid;
    const bool valid = i < P.M;
    const long long jb = P.N * sp / P.S, je = P.N * (sp + 1) / P.S;
    RowPt<COST, DP> rp;
    rp.load(P, i, valid);
    const double w = A.w, inv_eta = A.inv_eta;
    double Pi = 0.0, eu = 0.0, bu = 0.0;
    if (valid) {
        Pi = P.m1_row ? pot_p(P.fr[i], P.phir[i], inv_eta) : pot_q(P.fr[i], P.phir[i], inv_eta);
        if (P.eu) { eu = P.eu[i]; bu = P.bu[i]; }
    }
    const bool trial = P.eu != nullptr, sparse = P.tau > 0.0;
    double acc = 0.0, cx = 0.0, em = 0.0, mz = -INFINITY;
    int cnt = 0;
    const long long bufbase = (i * P.S + sp) * P.cap;
    for (long long j0 = jb; j0 < je; j0 += kCC) {
        const int nc = (int)min((long long)kCC, je - j0);
        __syncthreads();
        for (int c = tid; c < kCC; c += kPT) {
            double q = -INFINITY;
            if (c < nc) q = P.m1_row ? pot_q(P.gc[j0 + c], P.psic[j0 + c], inv_eta)
                                     : pot_p(P.gc[j0 + c], P.psic[j0 + c], inv_eta);
            sg.q[c] = q;
            if (trial) {
                sg.ev[c] = (c < nc) ? P.ev[j0 + c] : 0.0;
                sg.bv[c] = (c < nc) ? P.bv[j0 + c] : 0.0;
            }
        }
        stage_cost<COST, DP>(sg, P, i0, j0, nc);
        __syncthreads();
        if (valid) {
#pragma unroll 4
            for (int c = 0; c < kCC; ++c) {
                if (c < nc) {
                    const double D = chunk_dist<COST, DP>(sg, P, rp, i, j0 + c, c, valid);
                    const double z = fma(-w, D, __dadd_rn(Pi, sg.q[c]));
                    const double zt = trial ? z + bu + sg.bv[c] : z;
                    if (zt > -kSumCut) {
                        const double X = pexp(z, thi, tlo);
                        acc += X;
                        mz = fmax(mz, z);
                        if (P.want_cx) cx = fma(X, D, cx);
                        if (trial) {
                            const double ev = sg.ev[c];
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
                }
            }
        }
    }
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
__global__ void __launch_bounds__(kPT) sum_pass_kernel(PassArgs A) {
    constexpr size_t kB0 = sizeof(Stage<COST0, DP>), kB1 = sizeof(Stage<COST1, DP>);
    __shared__ __align__(16) unsigned char smraw[kB0 > kB1 ? kB0 : kB1];
    __shared__ double thi[64], tlo[64];
    __shared__ double red[kPT / 32];
    __shared__ bool flag;
    load_exp_table(A.tab, thi, tlo);
    const int side = (blockIdx.x < (unsigned)A.G0) ? 0 : 1;
    const int bid = side == 0 ? blockIdx.x : blockIdx.x - A.G0;
    if (side == 0)
        sum_side<COST0, DP>(A, A.side[0], bid, *reinterpret_cast<Stage<COST0, DP> *>(smraw), thi, tlo, red, &flag, 0);
    else
        sum_side<COST1, DP>(A, A.side[1], bid, *reinterpret_cast<Stage<COST1, DP> *>(smraw), thi, tlo, red, &flag, 1);
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

// CSR (or CSC) from the per-(row, split) buffers: rowptr from an exclusive
// scan of min(cnt, cap) over (row, split) in row-major order (done by
// scan_counts_kernel), then one warp per pass row copies its S segments.
__global__ void seg_copy_kernel(long long M, int S, long long cap, const long long *segptr,
                                const int *bcol, const double *bval, long long *rowptr, int *colidx,
                                double *val) {
    const int lane = threadIdx.x & 31;
    const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = gw; i < M; i += nw) {
        if (lane == 0) rowptr[i] = segptr[i * S];
        if (i == M - 1 && lane == 0) rowptr[M] = segptr[M * S];
        for (int s = 0; s < S; ++s) {
            const long long seg = i * S + s;
            const long long dst = segptr[seg], len = segptr[seg + 1] - dst;
            const long long src = seg * cap;
            for (long long k = lane; k < len; k += 32) {
                colidx[dst + k] = bcol[src + k];
                val[dst + k] = bval[src + k];
            }
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
                                                        CsrOut O1) {
    __shared__ long long sc[kPT];
    const int side = (blockIdx.x < (unsigned)P0.RB) ? 0 : 1;
    if (side == 1 && nsides < 2) return;
    const PassSide &P = side == 0 ? P0 : P1;
    const CsrOut &O = side == 0 ? O0 : O1;
    const int rb = side == 0 ? blockIdx.x : blockIdx.x - P0.RB;
    const int tid = threadIdx.x;
    const long long i = (long long)rb * kPT + tid;
    long long tot = 0;
    if (i < P.M)
        for (int s = 0; s < P.S; ++s) tot += min((long long)P.cnt[i * P.S + s], P.cap);
    sc[tid] = tot;
    __syncthreads();
    for (int o = 1; o < kPT; o <<= 1) {
        const long long t = tid >= o ? sc[tid - o] : 0;
        __syncthreads();
        sc[tid] += t;
        __syncthreads();
    }
    const long long start = O.blkoff[rb] + sc[tid] - tot;
    if (i < P.M) {
        O.ptr[i] = start;
        long long dst = start;
        for (int s = 0; s < P.S; ++s) {
            const long long len = min((long long)P.cnt[i * P.S + s], P.cap);
            const long long src = (i * P.S + s) * P.cap;
            for (long long k = 0; k < len; ++k) {
                O.idx[dst + k] = P.bcol[src + k];
                O.val[dst + k] = P.bval[src + k];
            }
            dst += len;
        }
        if (i == P.M - 1) O.ptr[P.M] = dst;
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

}  // namespace pins
