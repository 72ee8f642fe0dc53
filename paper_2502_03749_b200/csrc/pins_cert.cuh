// pins_cert.cuh -- LP optimality certificate of a PINS plan (reading R11,
// DESIGN.md §3): certified duals and the LP KKT residuals of Eq. (1),
// PAPER.md:41-46.
//
//  1. basis: the maximum-weight spanning forest T of the sparsified support
//     of X~ -- built by tree_pcg_kernel's Boruvka (pins_tree.cuh, setup mode),
//     which also leaves an O(log N)-round tree-contraction schedule: records
//     (u eliminated, neighbours v1, v2 at that time, slot sources s1, s2 =
//     tree edge t >= 0 or the fill edge of record -(s+1)).
//  2. tree_duals_kernel: the complementary-slackness equations u_i + v_j =
//     C_ij on T, solved exactly by replaying that schedule with a different
//     payload.  With z = (u, -v) every equation is a difference z_a - z_b =
//     d_ab (d = C_ij for row -> column).  Eliminating u with neighbours v1, v2
//     (z_u - z_v1 = d1, z_u - z_v2 = d2) leaves the fill equation
//     z_v1 - z_v2 = d2 - d1; back substitution z_u = z_v1 + d1; the last node
//     of each component gets z = 0 (gauge).  O(log N) rounds, one CTA.
//  3. ctrans_*: c-transforms u'_i = min_j (C_ij - v_j), v'_j = min_i (C_ij -
//     u'_i) (dense passes over the cost; fp64, C_ij = cost_scale * D_ij with D
//     as the plan kernel forms it), and the measured dual infeasibility
//     max_ij (u_i + v_j - C_ij).  (u', v') is dual feasible by construction,
//     so <a,u'> + <b,v'> <= LP* and gap = <C,X> - <a,u'> - <b,v'> bounds the
//     objective error of X from above.
#pragma once
#include "pins_device.cuh"
#include "pins_tree.cuh"

namespace pins {

constexpr int kCtT = 128;              // threads of the c-transform / component passes
constexpr int kCtC = 32;               // staged pass columns per chunk (points)

struct TreeDualArgs {
    int m, n;
    const int *ctr;                    // [1] rounds, [2] tree edges
    const int *rstart;                 // round boundaries
    const int *fu, *fv1, *fv2, *fs1, *fs2;
    const int *tei, *tej;              // tree edges (row, column)
    CostDesc cd;
    double scale;                      // cost_scale
    double *dd;                        // [N] per record: d1 (its own equation to v1)
    double *df;                        // [N] per record: fill payload d2 - d1 (z_v1 - z_v2)
    double *tc;                        // [N] per tree edge: C_ij
    double *z;                         // [N] output: z = (u, -v)
    int *comp;                         // [N] output: component root of each node
};

__device__ __forceinline__ double cost_entry(const CostDesc &cd, double scale, long long i, long long j) {
    double D;
    if (cd.kind == 0) {
        D = cd.C[i * cd.ldc + j];
    } else {
        double s = 0.0;
        for (int k = 0; k < cd.d; ++k) {
            const double t = cd.x[i * cd.d + k] - cd.y[j * cd.d + k];
            s = cd.kind == 1 ? fma(t, t, s) : s + fabs(t);
        }
        D = s;
    }
    return __dmul_rn(scale, D);
}

__global__ void __launch_bounds__(1024, 1) tree_duals_kernel(TreeDualArgs A) {
    const int tid = threadIdx.x;
    const int N = A.m + A.n;
    const int nr = A.ctr[1], ne = A.ctr[2];
    for (int t = tid; t < ne; t += blockDim.x) A.tc[t] = cost_entry(A.cd, A.scale, A.tei[t], A.tej[t]);
    for (int v = tid; v < N; v += blockDim.x) A.z[v] = 0.0;
    __syncthreads();
    // payload of slot source s seen from node u: z_u - z_other = d
    auto payload = [&](int s, int u) -> double {
        if (s >= 0) {
            const double c = A.tc[s];
            return u == A.tei[s] ? c : -c;           // row -> column: +C, column -> row: -C
        }
        const int p = -s - 1;                        // fill edge of record p: z_v1(p) - z_v2(p) = df[p]
        return u == A.fv1[p] ? A.df[p] : -A.df[p];
    };
    for (int r = 0; r < nr; ++r) {                  // forward: payloads in elimination order
        const int q1 = A.rstart[r + 1];
        for (int q = A.rstart[r] + tid; q < q1; q += blockDim.x) {
            const int u = A.fu[q];
            double d1 = 0.0;
            if (A.fv1[q] >= 0) d1 = payload(A.fs1[q], u);
            A.dd[q] = d1;
            if (A.fv2[q] >= 0) A.df[q] = payload(A.fs2[q], u) - d1;
        }
        __syncthreads();
    }
    for (int v = tid; v < N; v += blockDim.x) A.comp[v] = v;    // never eliminated: own root
    __syncthreads();
    for (int r = nr - 1; r >= 0; --r) {             // backward: z_u = z_v1 + d1
        const int q1 = A.rstart[r + 1];
        for (int q = A.rstart[r] + tid; q < q1; q += blockDim.x) {
            const int v1 = A.fv1[q], u = A.fu[q];
            A.z[u] = v1 >= 0 ? A.z[v1] + A.dd[q] : 0.0;
            A.comp[u] = v1 >= 0 ? A.comp[v1] : u;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------- basis repair (R11)
// Reduced costs of the support edges under the tree duals: an edge with
// C_ij - u_i - v_j < -tol violates dual feasibility; it is forced into the
// next forest (weight 4 > any plan entry), so the next maximum spanning forest
// drops the lightest edge of the cycle it closes (a dual-simplex-like pivot).
// Forced edges stay forced.  cnt[0] += violations.
__global__ void support_rc_kernel(long long nnz, const int *erow, const int *colidx, const double *val,
                                  CostDesc cd, double scale, const double *u, const double *v, double tol,
                                  double *w, int first, int *cnt) {
    int nv = 0;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
         e += (long long)gridDim.x * blockDim.x) {
        const int i = erow[e], j = colidx[e];
        const double r = cost_entry(cd, scale, i, j) - u[i] - v[j];
        const bool viol = r < -tol;
        nv += viol ? 1 : 0;
        const bool forced = !first && w[e] == 4.0;
        w[e] = (viol || forced) ? 4.0 : val[e];
    }
    nv = warp_sum_int(nv);
    if ((threadIdx.x & 31) == 0 && nv) atomicAdd(cnt, nv);
}

// ------------------------------------------------- component gauges (R11)
// A disconnected support leaves one free gauge per component (u + d, v - d).
// The shifts d_A must satisfy d_A - d_B <= R_AB = min_{i in A, j in B}
// (C_ij - u_i - v_j) (rows of A, columns of B); with balanced components
// (no optimal flow between them) every feasible choice gives the same bound,
// and shortest-path distances are one.  ncomp <= kMaxComp.
constexpr int kMaxComp = 64;

__device__ __forceinline__ unsigned long long ord_key(double x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_val(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

// one CTA: component ids (roots -> 0..K-1), K in cid_info[0] (-1 if > kMaxComp)
__global__ void __launch_bounds__(1024) comp_ids_kernel(int N, const int *comp, int *cid, int *cid_info,
                                                        unsigned long long *R) {
    __shared__ int cnt;
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    for (int x = threadIdx.x; x < N; x += blockDim.x)
        if (comp[x] == x) cid[x] = atomicAdd(&cnt, 1);        // any numbering works (shortest paths)
    __syncthreads();
    if (threadIdx.x == 0) cid_info[0] = cnt <= kMaxComp ? cnt : -1;
    for (int t = threadIdx.x; t < kMaxComp * kMaxComp; t += blockDim.x) R[t] = ~0ull;
}

// R_AB over all pairs (i, j) in different components: thread per row, columns staged
__global__ void __launch_bounds__(kCtT) comp_rmin_kernel(long long m, long long n, CostDesc cd, double scale,
                                                         const double *u, const double *v, const int *comp,
                                                         const int *cid, const int *cid_info,
                                                         unsigned long long *R) {
    __shared__ unsigned long long Rs[kMaxComp * kMaxComp];
    __shared__ int cc[256];
    __shared__ double vs[256];
    const int K = cid_info[0];
    if (K <= 1) return;
    for (int t = threadIdx.x; t < K * K; t += blockDim.x) Rs[t] = ~0ull;
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const bool valid = i < m;
    const int A = valid ? cid[comp[i]] : 0;
    const double ui = valid ? u[i] : 0.0;
    for (long long j0 = 0; j0 < n; j0 += 256) {
        const int nc = (int)min(256LL, n - j0);
        __syncthreads();
        for (int t = threadIdx.x; t < nc; t += blockDim.x) {
            cc[t] = cid[comp[m + j0 + t]];
            vs[t] = v[j0 + t];
        }
        __syncthreads();
        if (!valid) continue;
        for (int c = 0; c < nc; ++c) {
            const int B = cc[c];
            if (B == A) continue;
            const double r = cost_entry(cd, scale, i, j0 + c) - ui - vs[c];
            atomicMin(Rs + A * K + B, ord_key(r));
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < K * K; t += blockDim.x)
        if (Rs[t] != ~0ull) atomicMin(R + t, Rs[t]);
}

// one thread: Bellman-Ford from a virtual source (d = 0 for all), edges B -> A of
// weight R_AB (d_A <= d_B + R_AB); then shift u_i += d_{A(i)}, v_j -= d_{B(j)}.
// A negative cycle (no feasible shifts) leaves the duals unshifted.
__global__ void comp_shift_solve_kernel(const int *cid_info, const unsigned long long *R, double *dsh, int *ok) {
    const int K = cid_info[0];
    *ok = 0;
    if (K <= 1) return;
    double d[kMaxComp];
    for (int a = 0; a < K; ++a) d[a] = 0.0;
    bool changed = true;
    for (int it = 0; it <= K && changed; ++it) {
        changed = false;
        for (int a = 0; a < K; ++a)
            for (int b = 0; b < K; ++b) {
                const unsigned long long key = R[a * K + b];
                if (a == b || key == ~0ull) continue;
                const double nd = d[b] + ord_val(key);
                if (nd < d[a]) { d[a] = nd; changed = true; }
            }
    }
    if (changed) return;                             // negative cycle
    for (int a = 0; a < K; ++a) dsh[a] = d[a];
    *ok = 1;
}

__global__ void comp_shift_apply_kernel(long long m, long long n, const int *comp, const int *cid, const int *ok,
                                        const double *dsh, double *u, double *v) {
    if (!*ok) return;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < m + n;
         k += (long long)gridDim.x * blockDim.x) {
        const double d = dsh[cid[comp[k]]];
        if (k < m) u[k] += d;
        else v[k - m] -= d;
    }
}

// z = (u, -v) -> u (m), v (n)
__global__ void split_duals_kernel(long long m, long long n, const double *z, double *u, double *v) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < m + n;
         k += (long long)gridDim.x * blockDim.x) {
        if (k < m) u[k] = z[k];
        else v[k - m] = -z[k];
    }
}

// --------------------------------------------------------------- c-transforms
// Pass rows p (M of them), pass columns q (N): row orientation p = i, q = j;
// column orientation p = j, q = i.  mode 0: out_p = min_q (C_pq - pin_q);
// mode 1: out_p = max_q (self_p + pin_q - C_pq) (dual infeasibility).
// Column splits S write partials part[s * M + p]; ctrans_finalize merges.
struct CtArgs {
    long long M, N;
    int S, orient, mode;
    CostDesc cd;                       // points: x = pass-row points, y = pass-column points
    double scale;
    const double *pin;                 // [N]
    const double *self;                // [M] (mode 1)
    double *part;                      // [S * M]
};


__device__ __forceinline__ double ct_fold(int mode, double acc, double v) {
    return mode == 0 ? fmin(acc, v) : fmax(acc, v);
}

// points, either orientation: thread per pass row, column chunks staged in smem
template <int KIND>
__global__ void __launch_bounds__(kCtT) ctrans_points_kernel(CtArgs A) {
    __shared__ double ys[kCtC * 16];
    __shared__ double ps[kCtC];
    const int tid = threadIdx.x, d = A.cd.d;
    const long long RB = (A.M + kCtT - 1) / kCtT;
    const long long rb = blockIdx.x % RB, sp = blockIdx.x / RB;
    const long long p = rb * kCtT + tid;
    const bool valid = p < A.M;
    const long long qb = A.N * sp / A.S, qe = A.N * (sp + 1) / A.S;
    double x[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = (valid && k < d) ? A.cd.x[p * d + k] : 0.0;
    const double self = (A.mode == 1 && valid) ? A.self[p] : 0.0;
    double acc = A.mode == 0 ? INFINITY : -INFINITY;
    for (long long q0 = qb; q0 < qe; q0 += kCtC) {
        const int nc = (int)min((long long)kCtC, qe - q0);
        __syncthreads();
        for (int t = tid; t < nc * d; t += kCtT) ys[t] = A.cd.y[q0 * d + t];
        if (tid < nc) ps[tid] = A.pin[q0 + tid];
        __syncthreads();
        if (!valid) continue;
        for (int c = 0; c < nc; ++c) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                if (k < d) {
                    const double t = x[k] - ys[c * d + k];
                    s = KIND == 1 ? fma(t, t, s) : s + fabs(t);
                }
            }
            const double C = __dmul_rn(A.scale, s);
            acc = ct_fold(A.mode, acc, A.mode == 0 ? C - ps[c] : (self + ps[c]) - C);
        }
    }
    if (valid) A.part[sp * A.M + p] = acc;
}

// dense C, row orientation: warp per pass row, lanes along the (contiguous) columns
__global__ void __launch_bounds__(kCtT) ctrans_dense_rows_kernel(CtArgs A) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long RB = (A.M + 3) / 4;
    const long long rb = blockIdx.x % RB, sp = blockIdx.x / RB;
    const long long p = rb * 4 + warp;
    if (p >= A.M) return;
    const long long qb = A.N * sp / A.S, qe = A.N * (sp + 1) / A.S;
    const double *row = A.cd.C + p * A.cd.ldc;
    const double self = A.mode == 1 ? A.self[p] : 0.0;
    double acc = A.mode == 0 ? INFINITY : -INFINITY;
    for (long long q = qb + lane; q < qe; q += 32) {
        const double C = __dmul_rn(A.scale, __ldg(row + q));
        acc = ct_fold(A.mode, acc, A.mode == 0 ? C - __ldg(A.pin + q) : (self + __ldg(A.pin + q)) - C);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = ct_fold(A.mode, acc, __shfl_xor_sync(0xffffffffu, acc, o));
    if (lane == 0) A.part[sp * A.M + p] = acc;
}

// dense C, column orientation: thread per pass row (= column j of C), adjacent
// threads read adjacent columns of each row of C (coalesced)
__global__ void __launch_bounds__(kCtT) ctrans_dense_cols_kernel(CtArgs A) {
    const int tid = threadIdx.x;
    const long long RB = (A.M + kCtT - 1) / kCtT;
    const long long rb = blockIdx.x % RB, sp = blockIdx.x / RB;
    const long long p = rb * kCtT + tid;
    if (p >= A.M) return;
    const long long qb = A.N * sp / A.S, qe = A.N * (sp + 1) / A.S;
    const double self = A.mode == 1 ? A.self[p] : 0.0;
    double acc = A.mode == 0 ? INFINITY : -INFINITY;
    for (long long q = qb; q < qe; ++q) {
        const double C = __dmul_rn(A.scale, __ldg(A.cd.C + q * A.cd.ldc + p));
        acc = ct_fold(A.mode, acc, A.mode == 0 ? C - __ldg(A.pin + q) : (self + __ldg(A.pin + q)) - C);
    }
    A.part[sp * A.M + p] = acc;
}

// merge the splits: out_p = min_s / max_s part[s * M + p]
__global__ void ctrans_finalize_kernel(long long M, int S, int mode, const double *part, double *out) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < M;
         p += (long long)gridDim.x * blockDim.x) {
        double acc = mode == 0 ? INFINITY : -INFINITY;
        for (int s = 0; s < S; ++s) acc = ct_fold(mode, acc, part[s * M + p]);
        out[p] = acc;
    }
}

// single CTA: st[slot] = max(0, max_k x[k])
__global__ void __launch_bounds__(1024) vec_max_kernel(long long len, const double *x, double *st, int slot) {
    __shared__ double sh[32];
    double v = 0.0;
    for (long long k = threadIdx.x; k < len; k += 1024) v = fmax(v, x[k]);
    v = warp_max(v);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = warp_max(sh[threadIdx.x]);
        if (threadIdx.x == 0) st[slot] = v;
    }
}

}  // namespace pins
