// pins_kernels.cuh -- the PINS dense passes, sparsification, CSR/CSC builders
// and the cooperative CG kernel.  Included once by pins_api.cu.
#pragma once
#include <cooperative_groups.h>

#include "pins_device.cuh"

namespace pins {
namespace cgx = cooperative_groups;

// =========================================================================
// Evaluation pass: X~_ij = exp(z_ij), z_ij = R_i + S_j - w D_ij with
//   R_i = (f_i + phi_i)/eta - 1,  S_j = (g_j + psi_j)/eta,  w = s*cost_scale/eta
// (Eq. (7) with the factored centre).
// Layout: CTA b owns rows [m b/G, m (b+1)/G) (<= kRMax rows); thread t owns
// columns j = c0 + 2t, c0 + 2t + 1 of each 512-column chunk, for all the
// CTA's rows.  Row sums live in per-thread registers and are block-reduced
// once at the end; column sums over the CTA's rows are complete per chunk
// and written as one partial row per CTA (coalesced).
// SPARSE: entries X~ >= tau are compacted per row into rb_* (row-major,
//   columns ascending) with warp ballots + a cross-warp prefix in smem.
// TRIAL:  also accumulates sum_ij X~_ij * expm1(-alpha(df_i+dg_j)/eta) from
//   the separable factors eu_i, ev_j (line-search identity, reading R4).
// =========================================================================
struct EvalArgs {
    long long m, n;
    CostDesc cd;
    const double *f, *phi, *g, *psi, *a;
    double inv_eta, w, tau;
    long long cap;
    const double *eu, *ev;
    const ExpTable *tab;
    double *rowsum, *gradf;
    double *colpart;               // G x n
    double *blk;                   // G x 4: [sum C X (unscaled D), sum X em1, max z, spare]
    int *rowcnt;
    int *rb_col;
    double *rb_val;
};

template <int KIND, int DMAX, bool SPARSE, bool TRIAL>
__global__ void __launch_bounds__(kThreads) eval_kernel(EvalArgs A) {
    __shared__ double thi[64], tlo[64];
    __shared__ double xs[kRMax * (DMAX > 0 ? DMAX : 1)];
    __shared__ double sR[kRMax], sEU[kRMax];
    __shared__ int cnt_sm[kRMax][kWarps];
    __shared__ int run_sm[kRMax];
    __shared__ double red[kWarps][kRMax];
    __shared__ double redb[kWarps][3];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long G = gridDim.x, b = blockIdx.x;
    const long long r0 = (A.m * b) / G, r1 = (A.m * (b + 1)) / G;
    const int nr = (int)(r1 - r0);
    load_exp_table(A.tab, thi, tlo);
    for (int t = tid; t < nr; t += kThreads) {
        sR[t] = (A.f[r0 + t] + A.phi[r0 + t]) * A.inv_eta - 1.0;
        if (TRIAL) sEU[t] = A.eu[r0 + t];
        if (SPARSE) run_sm[t] = 0;
    }
    if (KIND == 1 || KIND == 2) {
        for (int t = tid; t < nr * A.cd.d; t += kThreads) xs[t] = A.cd.x[r0 * A.cd.d + t];
    }
    __syncthreads();

    double rs[kRMax];
#pragma unroll
    for (int r = 0; r < kRMax; ++r) rs[r] = 0.0;
    double acc_cx = 0.0, acc_em = 0.0, acc_mz = -INFINITY;
    const double w = A.w, tau = A.tau;

    for (long long c0 = 0; c0 < A.n; c0 += kChunk) {
        const long long j = c0 + 2 * tid;
        const bool v0 = j < A.n, v1 = j + 1 < A.n;
        double S0 = 0.0, S1 = 0.0, ev0 = 0.0, ev1 = 0.0;
        if (v0) S0 = (A.g[j] + A.psi[j]) * A.inv_eta;
        if (v1) S1 = (A.g[j + 1] + A.psi[j + 1]) * A.inv_eta;
        if (TRIAL) {
            if (v0) ev0 = A.ev[j];
            if (v1) ev1 = A.ev[j + 1];
        }
        ColPts<KIND, DMAX> cp;
        cp.load(A.cd, j, A.n);
        double cs0 = 0.0, cs1 = 0.0;
        unsigned kb0 = 0u, kb1 = 0u;     // SPARSE: keep bits per row
#pragma unroll
        for (int r = 0; r < kRMax; ++r) {
            if (r < nr) {
                double D0, D1;
                if constexpr (KIND == 0 || KIND == 3) dense_load2(A.cd, r0 + r, j, A.n, D0, D1);
                else pts_dist2<KIND, DMAX>(xs + r * A.cd.d, cp, A.cd.d, D0, D1);
                const double R = sR[r];
                double z0 = fma(-w, D0, R + S0);
                double z1 = fma(-w, D1, R + S1);
                double X0, X1;
                if constexpr (KIND == 3) {
                    X0 = v0 ? D0 : 0.0;
                    X1 = v1 ? D1 : 0.0;
                } else {
                    X0 = v0 ? pexp(z0, thi, tlo) : 0.0;
                    X1 = v1 ? pexp(z1, thi, tlo) : 0.0;
                }
                rs[r] += X0 + X1;
                cs0 += X0;
                cs1 += X1;
                acc_cx = fma(X0, D0, acc_cx);
                acc_cx = fma(X1, D1, acc_cx);
                if (v0) acc_mz = fmax(acc_mz, z0);
                if (v1) acc_mz = fmax(acc_mz, z1);
                if (TRIAL) {
                    const double eu = sEU[r];
                    acc_em = fma(X0, fma(eu, ev0, eu + ev0), acc_em);
                    acc_em = fma(X1, fma(eu, ev1, eu + ev1), acc_em);
                }
                if (SPARSE) {
                    const bool k0 = v0 && X0 >= tau, k1 = v1 && X1 >= tau;
                    kb0 |= (unsigned)k0 << r;
                    kb1 |= (unsigned)k1 << r;
                    const unsigned b0 = __ballot_sync(0xffffffffu, k0);
                    const unsigned b1 = __ballot_sync(0xffffffffu, k1);
                    if (lane == 0) cnt_sm[r][warp] = __popc(b0) + __popc(b1);
                }
            }
        }
        if (SPARSE) {
            __syncthreads();
            // write phase: columns ascending inside a row = warp-major, then
            // lane-major, sub 0 before sub 1.  Only kept entries recompute X
            // (same arithmetic -> identical bits).
#pragma unroll 1
            for (int r = 0; r < nr; ++r) {
                const bool k0 = (kb0 >> r) & 1u, k1 = (kb1 >> r) & 1u;
                const unsigned b0 = __ballot_sync(0xffffffffu, k0);
                const unsigned b1 = __ballot_sync(0xffffffffu, k1);
                if ((b0 | b1) == 0u) continue;
                if (!(k0 || k1)) continue;
                int base = run_sm[r];
                for (int w2 = 0; w2 < warp; ++w2) base += cnt_sm[r][w2];
                const unsigned lt = (1u << lane) - 1u;
                const int rank0 = __popc(b0 & lt) + __popc(b1 & lt);
                double D0, D1;
                if constexpr (KIND == 0 || KIND == 3) dense_load2(A.cd, r0 + r, j, A.n, D0, D1);
                else pts_dist2<KIND, DMAX>(xs + r * A.cd.d, cp, A.cd.d, D0, D1);
                const double R = sR[r];
                const long long row = r0 + r;
                if constexpr (KIND == 3) {
                    if (k0) { const long long pos = base + rank0;
                        if (pos < A.cap) { A.rb_col[row * A.cap + pos] = (int)j; A.rb_val[row * A.cap + pos] = D0; } }
                    if (k1) { const long long pos = base + rank0 + (k0 ? 1 : 0);
                        if (pos < A.cap) { A.rb_col[row * A.cap + pos] = (int)(j + 1); A.rb_val[row * A.cap + pos] = D1; } }
                    continue;
                }
                if (k0) {
                    const long long pos = base + rank0;
                    if (pos < A.cap) {
                        A.rb_col[row * A.cap + pos] = (int)j;
                        A.rb_val[row * A.cap + pos] = pexp(fma(-w, D0, R + S0), thi, tlo);
                    }
                }
                if (k1) {
                    const long long pos = base + rank0 + (k0 ? 1 : 0);
                    if (pos < A.cap) {
                        A.rb_col[row * A.cap + pos] = (int)(j + 1);
                        A.rb_val[row * A.cap + pos] = pexp(fma(-w, D1, R + S1), thi, tlo);
                    }
                }
            }
            __syncthreads();
            for (int r = tid; r < nr; r += kThreads) {
                int tot = 0;
                for (int w2 = 0; w2 < kWarps; ++w2) tot += cnt_sm[r][w2];
                run_sm[r] += tot;
            }
            // cnt_sm is rewritten in the next chunk only after this barrier
            __syncthreads();
        }
        if (v0) A.colpart[b * A.n + j] = cs0;
        if (v1) A.colpart[b * A.n + j + 1] = cs1;
    }

    // ---- row reductions (block) ----
#pragma unroll
    for (int r = 0; r < kRMax; ++r) {
        if (r < nr) {
            double v = warp_sum(rs[r]);
            if (lane == 0) red[warp][r] = v;
        }
    }
    {
        double cx = warp_sum(acc_cx);
        double em = warp_sum(acc_em);
        double mz = warp_max(acc_mz);
        if (lane == 0) {
            redb[warp][0] = cx;
            redb[warp][1] = em;
            redb[warp][2] = mz;
        }
    }
    __syncthreads();
    for (int r = tid; r < nr; r += kThreads) {
        double v = 0.0;
        for (int w2 = 0; w2 < kWarps; ++w2) v += red[w2][r];
        A.rowsum[r0 + r] = v;
        A.gradf[r0 + r] = A.a[r0 + r] - v;
        if (SPARSE) A.rowcnt[r0 + r] = run_sm[r];
    }
    if (tid == 0) {
        double cx = 0.0, em = 0.0, mz = -INFINITY;
        for (int w2 = 0; w2 < kWarps; ++w2) {
            cx += redb[w2][0];
            em += redb[w2][1];
            mz = fmax(mz, redb[w2][2]);
        }
        A.blk[b * 4 + 0] = cx;
        A.blk[b * 4 + 1] = em;
        A.blk[b * 4 + 2] = mz;
        A.blk[b * 4 + 3] = 0.0;
    }
}

// column sums from the per-CTA partials, gradient g-part
__global__ void colsum_kernel(long long n, int G, const double *__restrict__ colpart,
                              const double *__restrict__ bvec, double *__restrict__ colsum,
                              double *__restrict__ gradg) {
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
         j += (long long)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < G; ++b) s += colpart[(long long)b * n + j];
        colsum[j] = s;
        gradg[j] = bvec[j] - s;
    }
}

// Deterministic scalar reductions after an evaluation pass (single block of 1024):
// st[0] ||gradf||_1  [1] ||gradg||_1  [2] sum X  [3] sum X D  [4] sum X em1
// [5] max z  [6] max rowcnt  [7] sum min(rowcnt, cap)  [8] sum a.f + b.g (optional)
__global__ void __launch_bounds__(1024) stats_kernel(long long m, long long n, int G,
                                                     const double *gradf, const double *gradg,
                                                     const double *rowsum, const double *blk,
                                                     const int *rowcnt, long long cap,
                                                     double *st) {
    __shared__ double sh[32][6];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double v0 = 0, v1 = 0, v2 = 0, v3 = 0, v4 = 0, v5 = -INFINITY, c6 = 0, c7 = 0;
    for (long long i = tid; i < m; i += 1024) {
        v0 += fabs(gradf[i]);
        v2 += rowsum[i];
        if (rowcnt) {
            double c = (double)rowcnt[i];
            c6 = fmax(c6, c);
            c7 += fmin(c, (double)cap);
        }
    }
    for (long long j = tid; j < n; j += 1024) v1 += fabs(gradg[j]);
    for (int b = tid; b < G; b += 1024) {
        v3 += blk[b * 4 + 0];
        v4 += blk[b * 4 + 1];
        v5 = fmax(v5, blk[b * 4 + 2]);
    }
    double vals[8] = {v0, v1, v2, v3, v4, v5, c6, c7};
    // two-level: warp then block (max for 5,6; sum otherwise)
    double outv[8];
    for (int q = 0; q < 8; ++q) outv[q] = (q == 5 || q == 6) ? warp_max(vals[q]) : warp_sum(vals[q]);
    __shared__ double sh8[32][8];
    if (lane == 0)
        for (int q = 0; q < 8; ++q) sh8[warp][q] = outv[q];
    __syncthreads();
    if (tid < 8) {
        double acc = (tid == 5 || tid == 6) ? -INFINITY : 0.0;
        for (int w2 = 0; w2 < 32; ++w2)
            acc = (tid == 5 || tid == 6) ? fmax(acc, sh8[w2][tid]) : acc + sh8[w2][tid];
        st[tid] = acc;
    }
    (void)sh;
}

// =========================================================================
// Sinkhorn sweep (Alg. 2 lines 5-6), robust log-domain form:
//   f_i <- eta(log a_i + 1) - phi_i - eta LSE_j(S_j - w D_ij),  S_j=(g_j+psi_j)/eta
//   g_j <- eta(log b_j + 1) - psi_j - eta LSE_i(R'_i - w D_ij), R'_i=(f_i+phi_i)/eta
// (DESIGN.md §2 expansion of Eq. (7)).  Row kernel: one warp per row, online
// (max, sum) per lane, shuffle merge.  Column kernel: one CTA per 32 columns,
// lane = column, warps stride the rows, smem merge.
// =========================================================================
struct SweepArgs {
    long long m, n;
    CostDesc cd;
    const double *phi, *psi, *a, *b;
    double *f, *g;
    double eta, inv_eta, w;
    const ExpTable *tab;
};

template <int KIND, int DMAX>
__global__ void __launch_bounds__(kThreads) sweep_row_kernel(SweepArgs A) {
    __shared__ double thi[64], tlo[64];
    load_exp_table(A.tab, thi, tlo);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = gw; i < A.m; i += nw) {
        double xr[DMAX > 0 ? DMAX : 1];
        if (KIND != 0) {
#pragma unroll
            for (int k = 0; k < DMAX; ++k) xr[k] = (k < A.cd.d) ? A.cd.x[i * A.cd.d + k] : 0.0;
        }
        double mx = -INFINITY, sm = 0.0;
        for (long long j = lane; j < A.n; j += 32) {
            double D;
            if constexpr (KIND == 0) {
                D = __ldg(A.cd.C + i * A.cd.ldc + j);
            } else {
                double s = 0.0;
#pragma unroll
                for (int k = 0; k < DMAX; ++k) {
                    if (k < A.cd.d) {
                        double t = xr[k] - __ldg(A.cd.y + j * A.cd.d + k);
                        s = (KIND == 1) ? fma(t, t, s) : s + fabs(t);
                    }
                }
                D = s;
            }
            const double x = fma(-A.w, D, (A.g[j] + A.psi[j]) * A.inv_eta);
            lse_push(mx, sm, x, thi, tlo);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            double m2 = __shfl_xor_sync(0xffffffffu, mx, o);
            double s2 = __shfl_xor_sync(0xffffffffu, sm, o);
            lse_merge(mx, sm, m2, s2, thi, tlo);
        }
        if (lane == 0) {
            const double L = mx + log(sm);
            A.f[i] = A.eta * (log(A.a[i]) + 1.0 - L) - A.phi[i];
        }
    }
}

template <int KIND, int DMAX>
__global__ void __launch_bounds__(kThreads) sweep_col_kernel(SweepArgs A) {
    __shared__ double thi[64], tlo[64];
    __shared__ double smx[kWarps][32], ssm[kWarps][32];
    load_exp_table(A.tab, thi, tlo);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (long long j0 = blockIdx.x * 32LL; j0 < A.n; j0 += 32LL * gridDim.x) {
        const long long j = j0 + lane;
        const bool vj = j < A.n;
        double yr[DMAX > 0 ? DMAX : 1];
        if (KIND != 0) {
#pragma unroll
            for (int k = 0; k < DMAX; ++k) yr[k] = (vj && k < A.cd.d) ? A.cd.y[j * A.cd.d + k] : 0.0;
        }
        double mx = -INFINITY, sm = 0.0;
        if (vj) {
            for (long long i = warp; i < A.m; i += kWarps) {
                double D;
                if constexpr (KIND == 0) {
                    D = __ldg(A.cd.C + i * A.cd.ldc + j);
                } else {
                    double s = 0.0;
#pragma unroll
                    for (int k = 0; k < DMAX; ++k) {
                        if (k < A.cd.d) {
                            double t = __ldg(A.cd.x + i * A.cd.d + k) - yr[k];
                            s = (KIND == 1) ? fma(t, t, s) : s + fabs(t);
                        }
                    }
                    D = s;
                }
                const double x = fma(-A.w, D, (A.f[i] + A.phi[i]) * A.inv_eta);
                lse_push(mx, sm, x, thi, tlo);
            }
        }
        smx[warp][lane] = mx;
        ssm[warp][lane] = sm;
        __syncthreads();
        if (warp == 0 && vj) {
            double M = smx[0][lane], S = ssm[0][lane];
            for (int w2 = 1; w2 < kWarps; ++w2) lse_merge(M, S, smx[w2][lane], ssm[w2][lane], thi, tlo);
            const double L = M + log(S);
            A.g[j] = A.eta * (log(A.b[j]) + 1.0 - L) - A.psi[j];
        }
        __syncthreads();
    }
}

// =========================================================================
// CSR from the row buffers; CSC (transpose) with per-column row sort.
// =========================================================================
// exclusive scan of min(cnt, cap) -> ptr (len+1), single block of 1024
__global__ void __launch_bounds__(1024) scan_counts_kernel(long long len, const int *cnt,
                                                          long long cap, long long *ptr) {
    __shared__ long long part[1024];
    __shared__ long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (long long base = 0; base < len; base += 1024) {
        long long i = base + threadIdx.x;
        long long v = (i < len) ? (long long)min((long long)cnt[i], cap) : 0;
        part[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            long long t = (threadIdx.x >= (unsigned)o) ? part[threadIdx.x - o] : 0;
            __syncthreads();
            part[threadIdx.x] += t;
            __syncthreads();
        }
        if (i < len) ptr[i] = carry + part[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry += part[1023];
        __syncthreads();
    }
    if (threadIdx.x == 0) ptr[len] = carry;
}

__global__ void csr_copy_kernel(long long m, long long cap, const long long *rowptr,
                                const int *rb_col, const double *rb_val, int *colidx, double *val) {
    const int lane = threadIdx.x & 31;
    const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = gw; i < m; i += nw) {
        const long long s = rowptr[i], e = rowptr[i + 1];
        for (long long k = lane; k < e - s; k += 32) {
            colidx[s + k] = rb_col[i * cap + k];
            val[s + k] = rb_val[i * cap + k];
        }
    }
}

__global__ void csc_count_kernel(long long m, const long long *rowptr, const int *colidx, int *colcnt) {
    const int lane = threadIdx.x & 31;
    const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = gw; i < m; i += nw)
        for (long long k = rowptr[i] + lane; k < rowptr[i + 1]; k += 32) atomicAdd(colcnt + colidx[k], 1);
}

__global__ void csc_fill_kernel(long long m, const long long *rowptr, const int *colidx,
                                const double *val, const long long *colptr, int *cursor,
                                int *rowidx, double *valT) {
    const int lane = threadIdx.x & 31;
    const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = gw; i < m; i += nw)
        for (long long k = rowptr[i] + lane; k < rowptr[i + 1]; k += 32) {
            const int jj = colidx[k];
            const long long pos = colptr[jj] + atomicAdd(cursor + jj, 1);
            rowidx[pos] = (int)i;
            valT[pos] = val[k];
        }
}

// insertion sort of each column segment by row index (segments are short)
__global__ void csc_sort_kernel(long long n, const long long *colptr, int *rowidx, double *valT) {
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
         j += (long long)gridDim.x * blockDim.x) {
        const long long s = colptr[j], e = colptr[j + 1];
        for (long long p = s + 1; p < e; ++p) {
            int r = rowidx[p];
            double v = valT[p];
            long long q = p - 1;
            while (q >= s && rowidx[q] > r) {
                rowidx[q + 1] = rowidx[q];
                valT[q + 1] = valT[q];
                --q;
            }
            rowidx[q + 1] = r;
            valT[q + 1] = v;
        }
    }
}

// =========================================================================
// Jacobi-preconditioned CG, one cooperative persistent launch.
//   M = [[diag(dr), Xs], [Xs^T, diag(dc)]] + mu I
// Per iteration two grid barriers: (A) w = M z, q = w + beta q, p = z + beta p,
// <p,q>; (B) alpha, x += alpha p, r -= alpha q, z = r ./ diag, <r,z>, <r,r>.
// (q = M p maintained through M p = M z + beta M p_prev.)  All blocks reduce
// the per-block partials in the same order, so every block takes the same
// branch.  At exit: st[0]=iters, st[1]=relres, st[2]=<grad, x>, st[3]=<a,x_f>+<b,x_g>
// computed with gvec (gradient) and wa (a, b) when given.
// =========================================================================
struct CGArgs {
    long long m, n;
    const long long *rowptr;
    const int *colidx;
    const double *val;
    const long long *colptr;
    const int *rowidx;
    const double *valT;
    const double *dr, *dc;
    double mu;
    const double *rhs;
    double *x, *r, *z, *p, *q;
    double *part;       // 4 * gridDim.x
    double rtol;
    int maxit;
    const double *gradf, *gradg, *a, *b;   // optional: slope / a.d terms
    double *st;
    int vec;                               // 1: warp-per-row products (mean degree > 8)
};

__device__ __forceinline__ double block_sum(double v, double *sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0) {
        for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) t += sh[w2];
    }
    return t;   // valid in thread 0
}

// sum of the per-block partials, read by warp 0 (lanes stride the blocks,
// fixed shuffle tree: the same value in every block), broadcast through smem
__device__ __forceinline__ double grid_reduce(const double *part, int slot, int G) {
    __shared__ double bcast;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = 0.0;
#pragma unroll 8
        for (int b2 = threadIdx.x; b2 < G; b2 += 32) t += __ldcg(part + b2 * 4 + slot);
        t = warp_sum(t);
        if (threadIdx.x == 0) bcast = t;
    }
    __syncthreads();
    return bcast;
}

__global__ void __launch_bounds__(kThreads) cg_kernel(CGArgs A) {
    cgx::grid_group grid = cgx::this_grid();
    __shared__ double sh[32];
    const long long N = A.m + A.n;
    const long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long gs = (long long)gridDim.x * blockDim.x;
    const int G = gridDim.x;
    auto diag = [&](long long k) {
        return (k < A.m ? A.dr[k] : A.dc[k - A.m]) + A.mu;
    };
    // init: x = 0, r = rhs, z = r/d, q = 0, p = 0
    double l_rz = 0.0, l_rr = 0.0;
    for (long long k = gt; k < N; k += gs) {
        double rv = A.rhs[k];
        double zv = rv / diag(k);
        A.x[k] = 0.0;
        A.r[k] = rv;
        A.z[k] = zv;
        A.p[k] = 0.0;
        A.q[k] = 0.0;
        l_rz += rv * zv;
        l_rr += rv * rv;
    }
    double t0 = block_sum(l_rz, sh);
    double t1 = block_sum(l_rr, sh);
    if (threadIdx.x == 0) {
        A.part[blockIdx.x * 4 + 0] = t0;
        A.part[blockIdx.x * 4 + 1] = t1;
    }
    grid.sync();
    double rz = grid_reduce(A.part, 0, G);
    double rr = grid_reduce(A.part, 1, G);
    const double bb = rr;
    double beta = 0.0;
    int it = 0;
    double relres = bb > 0.0 ? 1.0 : 0.0;
    while (bb > 0.0) {
        relres = sqrt(rr / bb);
        if (relres <= A.rtol || it >= A.maxit) break;
        // (A) w = M z ; q = w + beta q ; p = z + beta p ; <p,q>
        double l_pq = 0.0;
        if (A.vec) {                       // dense-ish rows: one warp per row, lanes over entries
            const int lane = threadIdx.x & 31;
            const long long gw = gt >> 5, nw = gs >> 5;
            for (long long k = gw; k < N; k += nw) {
                double wv = 0.0;
                if (k < A.m) {
                    for (long long e = A.rowptr[k] + lane; e < A.rowptr[k + 1]; e += 32)
                        wv = fma(A.val[e], A.z[A.m + A.colidx[e]], wv);
                } else {
                    const long long jj = k - A.m;
                    for (long long e = A.colptr[jj] + lane; e < A.colptr[jj + 1]; e += 32)
                        wv = fma(A.valT[e], A.z[A.rowidx[e]], wv);
                }
                wv = warp_sum(wv);
                if (lane == 0) {
                    wv = fma(diag(k), A.z[k], wv);
                    const double qv = fma(beta, A.q[k], wv);
                    const double pv = fma(beta, A.p[k], A.z[k]);
                    A.q[k] = qv;
                    A.p[k] = pv;
                    l_pq = fma(pv, qv, l_pq);
                }
            }
        } else
        for (long long k = gt; k < N; k += gs) {
            double wv;
            if (k < A.m) {
                wv = diag(k) * A.z[k];
                for (long long e = A.rowptr[k]; e < A.rowptr[k + 1]; ++e)
                    wv = fma(A.val[e], A.z[A.m + A.colidx[e]], wv);
            } else {
                const long long jj = k - A.m;
                wv = diag(k) * A.z[k];
                for (long long e = A.colptr[jj]; e < A.colptr[jj + 1]; ++e)
                    wv = fma(A.valT[e], A.z[A.rowidx[e]], wv);
            }
            const double qv = fma(beta, A.q[k], wv);
            const double pv = fma(beta, A.p[k], A.z[k]);
            A.q[k] = qv;
            A.p[k] = pv;
            l_pq = fma(pv, qv, l_pq);
        }
        double tpq = block_sum(l_pq, sh);
        if (threadIdx.x == 0) A.part[blockIdx.x * 4 + 2] = tpq;
        grid.sync();
        const double pq = grid_reduce(A.part, 2, G);
        if (!(pq > 0.0)) break;
        const double alpha = rz / pq;
        // (B)
        double l_rz2 = 0.0, l_rr2 = 0.0;
        for (long long k = gt; k < N; k += gs) {
            double xv = fma(alpha, A.p[k], A.x[k]);
            double rv = fma(-alpha, A.q[k], A.r[k]);
            double zv = rv / diag(k);
            A.x[k] = xv;
            A.r[k] = rv;
            A.z[k] = zv;
            l_rz2 = fma(rv, zv, l_rz2);
            l_rr2 = fma(rv, rv, l_rr2);
        }
        double u0 = block_sum(l_rz2, sh);
        double u1 = block_sum(l_rr2, sh);
        if (threadIdx.x == 0) {
            A.part[blockIdx.x * 4 + 0] = u0;
            A.part[blockIdx.x * 4 + 1] = u1;
        }
        grid.sync();
        const double rz_new = grid_reduce(A.part, 0, G);
        rr = grid_reduce(A.part, 1, G);
        beta = rz_new / rz;
        rz = rz_new;
        ++it;
    }
    // slope terms for the line search
    double l_s = 0.0, l_a = 0.0;
    if (A.gradf) {
        for (long long k = gt; k < N; k += gs) {
            const double xv = A.x[k];
            if (k < A.m) {
                l_s = fma(A.gradf[k], xv, l_s);
                l_a = fma(A.a[k], xv, l_a);
            } else {
                l_s = fma(A.gradg[k - A.m], xv, l_s);
                l_a = fma(A.b[k - A.m], xv, l_a);
            }
        }
    }
    double v0 = block_sum(l_s, sh);
    double v1 = block_sum(l_a, sh);
    grid.sync();
    if (threadIdx.x == 0) {
        A.part[blockIdx.x * 4 + 0] = v0;
        A.part[blockIdx.x * 4 + 1] = v1;
    }
    grid.sync();
    const double s0 = grid_reduce(A.part, 0, G);   // every thread: grid_reduce synchronises the block
    const double s1 = grid_reduce(A.part, 1, G);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        A.st[0] = (double)it;
        A.st[1] = relres;
        A.st[2] = s0;
        A.st[3] = s1;
    }
}

// =========================================================================
// small vector kernels
// =========================================================================
// trial point (f + alpha df, g + alpha dg) and the separable expm1 factors
// bu / bv = max(0, -alpha d / eta): X~ at the old point is X~ at the trial point
// times exp(bu_i + bv_j) at most, which keeps the sum pass's skip test safe for
// the trial term (pins_pass.cuh)
__global__ void trial_prep_kernel(long long m, long long n, double alpha, double inv_eta,
                                  const double *f, const double *g, const double *d,
                                  double *ft, double *gt, double *eu, double *ev, double *bu, double *bv) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < m + n;
         k += (long long)gridDim.x * blockDim.x) {
        const double dk = alpha * d[k];
        if (k < m) {
            ft[k] = f[k] + dk;
            eu[k] = expm1(-dk * inv_eta);
            bu[k] = fmax(0.0, -dk * inv_eta);
        } else {
            gt[k - m] = g[k - m] + dk;
            ev[k - m] = expm1(-dk * inv_eta);
            bv[k - m] = fmax(0.0, -dk * inv_eta);
        }
    }
}

__global__ void scale_concat_kernel(long long m, long long n, double s, const double *u,
                                    const double *v, double *out) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < m + n;
         k += (long long)gridDim.x * blockDim.x)
        out[k] = s * (k < m ? u[k] : v[k - m]);
}

__global__ void center_init_kernel(long long m, long long n, double eta, const double *a,
                                   const double *b, double *phi, double *psi) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < m + n;
         k += (long long)gridDim.x * blockDim.x) {
        if (k < m) phi[k] = eta * log(a[k]);
        else psi[k - m] = eta * log(b[k - m]);
    }
}

// warm start by linear extrapolation (warm_start = 2): x_prev <- x, x <- x + gamma (x - x_prev);
// with undo = 1 restores x <- x_prev (the saved value)
__global__ void extrapolate_kernel(long long len, double gamma, int undo, double *x, double *xprev,
                                   double *xsave) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < len;
         k += (long long)gridDim.x * blockDim.x) {
        if (undo) {
            x[k] = xsave[k];
        } else {
            const double cur = x[k];
            xsave[k] = cur;
            x[k] = fma(gamma, cur - xprev[k], cur);
            xprev[k] = cur;
        }
    }
}

__global__ void center_update_kernel(long long m, long long n, double eta, const double *f,
                                     const double *g, double *phi, double *psi) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < m + n;
         k += (long long)gridDim.x * blockDim.x) {
        if (k < m) phi[k] += f[k];
        else psi[k - m] += g[k - m] - eta;
    }
}

__global__ void lp_duals_kernel(long long m, long long n, double eta, double inv_s,
                                const double *f, const double *g, const double *phi,
                                const double *psi, double *u, double *v) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < m + n;
         k += (long long)gridDim.x * blockDim.x) {
        if (k < m) u[k] = (f[k] + phi[k]) * inv_s;
        else v[k - m] = (g[k - m] + psi[k - m] - eta) * inv_s;
    }
}

// dense plan materialisation (same z and pexp as eval_kernel -> identical bits)
template <int KIND, int DMAX>
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
                double t = cd.x[i * cd.d + k] - cd.y[j * cd.d + k];
                s = (KIND == 1) ? fma(t, t, s) : s + fabs(t);
            }
            D = s;
        }
        const double R = (f[i] + phi[i]) * inv_eta - 1.0;
        const double S = (g[j] + psi[j]) * inv_eta;
        X[i * ldx + j] = pexp(fma(-w, D, R + S), thi, tlo);
    }
}

}  // namespace pins
