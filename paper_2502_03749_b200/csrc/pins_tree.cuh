// pins_tree.cuh -- CG on the sparsified Newton system with a maximum-spanning-
// tree preconditioner (support-graph preconditioning), one CTA per system.
//
// System (Alg. 2 line 12, reading R5):  M d = rhs,
//     M = [[Dr, X],[X^T, Dc]],  Dr = diag(X~ e) + mu,  Dc = diag(X~^T e) + mu,
// X = the sparsified plan block.  M is the "signless Laplacian" of the
// bipartite support graph (rows + columns, edge (i, j) of weight X_ij) plus a
// positive diagonal excess (dropped mass, mu).  The preconditioner keeps the
// diagonal and the edges of a MAXIMUM-WEIGHT SPANNING FOREST T of that graph:
//     M_T = diag(Dr, Dc) + T,
// which is SPD and is factorised EXACTLY with zero fill by tree contraction.
// Late in EPPA the plan approaches a vertex of the transport polytope, whose
// support is a spanning tree (Thm 4.3), so M_T ~ M and CG
// needs a handful of iterations instead of hundreds.
//
//  1. Boruvka: every component takes its heaviest outgoing edge (64-bit atomic
//     max of (float weight bits, edge id): a strict total order, hence no
//     cycles), components merge by hooking + pointer jumping; O(log N) rounds.
//  2. Tree contraction: each round eliminates an independent set of nodes of
//     degree <= 2 (random priorities; leaves = rake, degree 2 = compress, which
//     rewires the two neighbours to each other with the fill weight
//     -w1 w2 / d).  O(log N) rounds; the eliminated nodes of a round are
//     stored contiguously with their neighbours and multipliers.
//  3. PCG (Jacobi-free: z = M_T^-1 r): forward elimination round by round,
//     back substitution in reverse, on a shared-memory copy of the vector.
//
// Everything runs in ONE CTA of kTT threads with __syncthreads between phases
// (no grid synchronisation); graph state lives in a workspace in global
// memory (L2-resident at these sizes), the tree-solve vector in shared memory.
#pragma once
#include "pins_device.cuh"

namespace pins {

constexpr int kTT = 1024;              // threads of the tree-CG CTA

// one entry of a record's pull list: a child's node and its forward multiplier
struct alignas(16) PullE {
    int node, pad;
    double coef;
};
constexpr int kTreeMaxRounds = 256;

struct TreeArgs {
    int m, n;                          // rows / columns (N = m + n nodes)
    long long nnz;
    const long long *rowptr;           // CSR of X (m rows)
    const int *colidx;
    const double *val;
    const long long *colptr;           // CSC of X (n columns)
    const int *rowidx;
    const double *valT;
    const double *dr, *dc;             // diagonals (without mu)
    double mu;
    const double *rhs;                 // N
    double *x;                         // N (output)
    double rtol;
    int maxit;
    const double *gradf, *gradg, *a, *b;   // optional slope terms
    double *st;                        // [0] its [1] relres [2] slope [3] <(a,b),d> [4] rounds [5] tree edges
    // workspace (global)
    int *erow;                         // [nnz] row of each CSR entry
    int *comp, *hook;                  // [N]
    unsigned long long *best;          // [N]
    unsigned char *tmark;              // [nnz]
    int *tptr;                         // [N + 1]
    int *tnbr;                         // [2 (N - 1)] (rewired during contraction)
    double *tw;                        // [2 (N - 1)]
    int *deg;                          // [N]
    unsigned char *alive, *sel;        // [N]
    double *dcur;                      // [N]
    int *fu, *fv1, *fv2;               // [N] factor in elimination order
    double *fc1, *fc2, *finv;          // [N]
    int *rstart;                       // [kTreeMaxRounds + 1]
    double *r, *z, *p, *q;             // [N] CG vectors (z unused: kept in shared memory)
    double *frec;                      // [5 N] packed factor records (40 B each)
    int *ctr;                          // [8] counters: [0] records [1] rounds [2] tree edges [3] valid
    int tail_cap;                      // factor records cached in shared memory
    // reuse across Newton steps: tree edge list, slot sources, weights
    int *tei, *tej;                    // [N] tree edges (row, column)
    double *tval;                      // [N] current weights X_ij of the tree edges
    int *tsrc;                         // [2 (N - 1)] adjacency slot source: edge t >= 0, fill -(pos+1)
    int *fs1, *fs2;                    // [N] record slot sources
    double *fw1, *fw2;                 // [N] record slot weights
    int reuse;                         // 1: try the stored tree / schedule first
    int setup_only;                    // 1: stop after the factor is packed (cluster PCG follows)
    // pull form of the elimination (deterministic, no atomics): for record q the records
    // p eliminated next to it ("children": fv1[p] or fv2[p] is fu[q]), sorted by node
    int *cptr;                         // [N + 1] child-list offsets per record
    int *cent;                         // [2 N] child entries 2 p + slot (slot 0: v1, 1: v2)
    int *ppos;                         // [2 N] list position of (p, slot)
    int4 *pk;                          // [N] per record: {node, first entry, entries, 0}
    int *rpos;                         // [N] record of each node
    int *cur;                          // [N] fill cursors
    struct PullE *pe;                  // [2 N] entries {child node, multiplier fc1 / fc2 of p}
};

__device__ __forceinline__ unsigned hash_prio(unsigned u, unsigned r) {
    unsigned h = u * 0x9E3779B1u ^ (r + 1u) * 0x85EBCA6Bu;
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    h *= 0x297A2D39u;
    h ^= h >> 15;
    return h;
}

__device__ __forceinline__ double tree_block_sum(double v, double *sh) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (warp == 0) t = warp_sum(sh[lane]);
    if (threadIdx.x == 0) sh[32] = t;
    __syncthreads();
    return sh[32];
}

// packed factor record of one eliminated node (forward: y_v -= c * y_u; backward:
// x_u = y_u inv - c1 x_v1 - c2 x_v2)
struct Rec { int u, v1, v2, pad; double c1, c2, inv; };
__device__ __forceinline__ Rec ldg_rec(const Rec *p) {
    Rec r;
    const int2 h0 = __ldg(reinterpret_cast<const int2 *>(p));        // 40-byte records: 8-byte aligned
    const int2 h1 = __ldg(reinterpret_cast<const int2 *>(p) + 1);
    r.u = h0.x; r.v1 = h0.y; r.v2 = h1.x; r.pad = 0;
    r.c1 = __ldg(&p->c1);
    r.c2 = __ldg(&p->c2);
    r.inv = __ldg(&p->inv);
    return r;
}


// block-wide exclusive scan of per-thread counts (kTT threads); returns the
// thread's offset, *total gets the sum
__device__ __forceinline__ int block_excl_scan(int v, int *wsc, int *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += t;
    }
    __syncthreads();
    if (lane == 31) wsc[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = wsc[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += t;
        }
        wsc[lane] = w;
    }
    __syncthreads();
    *total = wsc[31];
    return x - v + (warp > 0 ? wsc[warp - 1] : 0);
}

__global__ void __launch_bounds__(kTT, 1) tree_pcg_kernel(TreeArgs A) {
    extern __shared__ __align__(16) unsigned char dyn[];   // 8 N bytes, reused by phase
    __shared__ double red[40];
    __shared__ int wsc[32];
    __shared__ int rs[kTreeMaxRounds + 1];     // round boundaries (copy of A.rstart)
    __shared__ int s_flag, s_cnt;
    const int tid = threadIdx.x;
    const int m = A.m, n = A.n, N = m + n;
    const long long nnz = A.nnz;
    const double mu = A.mu;
    const long long t_start = clock64();
    long long t_mst = 0, t_fac = 0, t_pc = 0, t_mv = 0;

    int nrounds = 0;
    // ---------------- 0. reuse: are all stored tree edges still in the support? ----------------
    bool rebuilt = true;
    if (A.reuse) {
        if (tid == 0) s_flag = 1;
        __syncthreads();
        const int ne = A.ctr[2];
        for (int t = tid; t < ne; t += kTT) {
            const int i = A.tei[t], j = A.tej[t];
            long long lo = A.rowptr[i], hi = A.rowptr[i + 1] - 1;
            double wv = -1.0;
            while (lo <= hi) {                     // columns ascending inside a CSR row
                const long long mid = (lo + hi) >> 1;
                const int cj = A.colidx[mid];
                if (cj == j) { wv = A.val[mid]; break; }
                if (cj < j) lo = mid + 1; else hi = mid - 1;
            }
            if (wv < 0.0) s_flag = 0;
            A.tval[t] = wv;
        }
        __syncthreads();
        if (s_flag) {
            nrounds = A.ctr[1];
            for (int k = tid; k <= nrounds; k += kTT) rs[k] = A.rstart[k];
            __syncthreads();
            rebuilt = false;
        }
    }
    if (rebuilt) {
    // ---------------- 1. maximum spanning forest (Boruvka), state in smem ----------------
    int *comp = reinterpret_cast<int *>(dyn);                 // N
    unsigned *bw = reinterpret_cast<unsigned *>(dyn) + N;     // N: best weight bits, then hook
    for (int i = tid; i < m; i += kTT)
        for (long long e = A.rowptr[i]; e < A.rowptr[i + 1]; ++e) A.erow[e] = i;
    for (int v = tid; v < N; v += kTT) comp[v] = v;
    for (long long e = tid; e < nnz; e += kTT) A.tmark[e] = 0;
    __syncthreads();
    for (int round = 0; round < 64; ++round) {
        for (int v = tid; v < N; v += kTT) {
            bw[v] = 0u;
            A.hook[v] = -1;                                   // best edge id
        }
        if (tid == 0) s_flag = 0;
        __syncthreads();
        for (long long e = tid; e < nnz; e += kTT) {
            const int cu = comp[A.erow[e]], cv = comp[m + A.colidx[e]];
            if (cu == cv) continue;
            const unsigned wb = __float_as_uint((float)A.val[e]);
            atomicMax(bw + cu, wb);
            atomicMax(bw + cv, wb);
        }
        __syncthreads();
        for (long long e = tid; e < nnz; e += kTT) {          // heaviest edge, ties -> largest id
            const int cu = comp[A.erow[e]], cv = comp[m + A.colidx[e]];
            if (cu == cv) continue;
            const unsigned wb = __float_as_uint((float)A.val[e]);
            if (wb == bw[cu]) atomicMax(A.hook + cu, (int)e);
            if (wb == bw[cv]) atomicMax(A.hook + cv, (int)e);
        }
        __syncthreads();
        for (int c = tid; c < N; c += kTT) {
            int h = c;
            const int e = A.hook[c];
            if (comp[c] == c && e >= 0) {
                const int cu = comp[A.erow[e]], cv = comp[m + A.colidx[e]];
                const int other = cu == c ? cv : cu;
                if (!(A.hook[other] == e && c < other)) h = other;   // mutual: smaller id stays
                A.tmark[e] = 1;
                s_flag = 1;
            }
            bw[c] = (unsigned)h;                              // bw reused as the hook target
        }
        __syncthreads();
        if (!s_flag) break;
        for (int v = tid; v < N; v += kTT) comp[v] = (int)bw[comp[v]];
        __syncthreads();
        for (int it = 0; it < 40; ++it) {                     // pointer jumping
            if (tid == 0) s_cnt = 0;
            __syncthreads();
            for (int v = tid; v < N; v += kTT) {
                const int c = comp[v], cc = comp[c];
                if (c != cc) { comp[v] = cc; s_cnt = 1; }
            }
            __syncthreads();
            if (!s_cnt) break;
        }
    }
    t_mst = clock64() - t_start;

    // ---------------- 2. tree adjacency (CSR of the forest) ----------------
    for (int v = tid; v <= N; v += kTT) A.tptr[v] = 0;
    __syncthreads();
    for (long long e = tid; e < nnz; e += kTT)
        if (A.tmark[e]) {
            atomicAdd(A.tptr + A.erow[e] + 1, 1);
            atomicAdd(A.tptr + m + A.colidx[e] + 1, 1);
        }
    __syncthreads();
    {
        __shared__ int carry;
        if (tid == 0) carry = 0;
        __syncthreads();
        for (int base = 1; base <= N; base += kTT) {
            const int idx = base + tid;
            const int v = idx <= N ? A.tptr[idx] : 0;
            int tot;
            const int off = block_excl_scan(v, wsc, &tot);
            if (idx <= N) A.tptr[idx] = carry + off + v;
            __syncthreads();
            if (tid == 0) carry += tot;
            __syncthreads();
        }
    }
    int *deg = reinterpret_cast<int *>(dyn);                                  // N ints
    unsigned char *alive = dyn + 4 * (size_t)N;                               // N
    unsigned char *sel = dyn + 5 * (size_t)N;                                 // N
    for (int v = tid; v < N; v += kTT) deg[v] = 0;                            // fill cursor
    if (tid == 0) A.ctr[2] = 0;
    __syncthreads();
    for (long long e = tid; e < nnz; e += kTT)
        if (A.tmark[e]) {
            const int u = A.erow[e], v = m + A.colidx[e];
            const double w = A.val[e];
            const int t = atomicAdd(A.ctr + 2, 1);
            A.tei[t] = u;
            A.tej[t] = v - m;
            A.tval[t] = w;
            const int pu = A.tptr[u] + atomicAdd(deg + u, 1);
            const int pv = A.tptr[v] + atomicAdd(deg + v, 1);
            A.tnbr[pu] = v;
            A.tw[pu] = w;
            A.tsrc[pu] = t;
            A.tnbr[pv] = u;
            A.tw[pv] = w;
            A.tsrc[pv] = t;
        }
    __syncthreads();
    // adjacency lists in neighbour order (the atomic fill order is arbitrary): the
    // contraction's choice of v1 / v2, hence every rounding downstream, is then fixed
    for (int v = tid; v < N; v += kTT) {
        const int b = A.tptr[v], e = A.tptr[v + 1];
        for (int k = b + 1; k < e; ++k) {
            const int nb = A.tnbr[k], sr = A.tsrc[k];
            const double wk = A.tw[k];
            int j = k - 1;
            while (j >= b && A.tnbr[j] > nb) {
                A.tnbr[j + 1] = A.tnbr[j];
                A.tw[j + 1] = A.tw[j];
                A.tsrc[j + 1] = A.tsrc[j];
                --j;
            }
            A.tnbr[j + 1] = nb;
            A.tw[j + 1] = wk;
            A.tsrc[j + 1] = sr;
        }
    }
    for (int v = tid; v < N; v += kTT) {
        alive[v] = 1;
        A.dcur[v] = (v < m ? A.dr[v] : A.dc[v - m]) + mu;
        A.hook[v] = v;                                                        // active list
    }
    if (tid == 0) {
        A.ctr[0] = 0;
        A.rstart[0] = 0;
    }
    __syncthreads();

    // ---------------- 3. tree contraction = exact LDL^T of M_T ----------------
    // active list ping-pong: A.hook (current) <-> A.comp (next)
    int *act = A.hook, *nxt = A.comp;
    int nact = N;
    for (int round = 0; round < kTreeMaxRounds && nact > 0; ++round) {
        for (int q = tid; q < nact; q += kTT) {
            const int u = act[q];
            unsigned char s0 = 0;
            if (deg[u] <= 2) {
                const unsigned pu = hash_prio(u, round);
                s0 = 1;
                for (int k = A.tptr[u]; k < A.tptr[u + 1]; ++k) {
                    const int v = A.tnbr[k];
                    if (v < 0 || !alive[v] || deg[v] > 2) continue;
                    const unsigned pv = hash_prio(v, round);
                    if (pv < pu || (pv == pu && v < u)) { s0 = 0; break; }
                }
            }
            sel[u] = s0;
        }
        __syncthreads();
        for (int q = tid; q < nact; q += kTT) {
            const int u = act[q];
            if (!sel[u]) continue;
            int v1 = -1, v2 = -1, s1 = 0, s2 = 0;
            double w1 = 0.0, w2 = 0.0;
            for (int k = A.tptr[u]; k < A.tptr[u + 1]; ++k) {
                const int v = A.tnbr[k];
                if (v < 0) continue;
                if (v1 < 0) { v1 = v; w1 = A.tw[k]; s1 = A.tsrc[k]; }
                else { v2 = v; w2 = A.tw[k]; s2 = A.tsrc[k]; }
            }
            const double inv = 1.0 / A.dcur[u];
            const int pos = atomicAdd(A.ctr + 0, 1);
            A.fu[pos] = u;
            A.fv1[pos] = v1;
            A.fv2[pos] = v2;
            A.fs1[pos] = s1;
            A.fs2[pos] = s2;
            A.fw1[pos] = w1;
            A.fw2[pos] = w2;
            A.fc1[pos] = w1 * inv;
            A.fc2[pos] = w2 * inv;
            A.finv[pos] = inv;
            alive[u] = 0;
            if (v1 >= 0) atomicAdd(A.dcur + v1, -w1 * w1 * inv);
            if (v2 >= 0) atomicAdd(A.dcur + v2, -w2 * w2 * inv);
            if (v2 < 0 && v1 >= 0) {          // rake: drop u from v1's list
                for (int k = A.tptr[v1]; k < A.tptr[v1 + 1]; ++k)
                    if (A.tnbr[k] == u) { A.tnbr[k] = -1; break; }
                atomicSub(deg + v1, 1);
            } else if (v2 >= 0) {             // compress: v1 -- v2 with the fill weight
                const double wf = -w1 * w2 * inv;
                for (int k = A.tptr[v1]; k < A.tptr[v1 + 1]; ++k)
                    if (A.tnbr[k] == u) { A.tnbr[k] = v2; A.tw[k] = wf; A.tsrc[k] = -(pos + 1); break; }
                for (int k = A.tptr[v2]; k < A.tptr[v2 + 1]; ++k)
                    if (A.tnbr[k] == u) { A.tnbr[k] = v1; A.tw[k] = wf; A.tsrc[k] = -(pos + 1); break; }
            }
        }
        __syncthreads();
        // compact the active list (order-preserving): thread t owns act[q0, q0 + per)
        const int per = (nact + kTT - 1) / kTT;
        const int q0 = tid * per;
        int nk = 0;
        for (int j = 0; j < per; ++j) {
            const int qq = q0 + j;
            nk += (qq < nact && alive[act[qq]]) ? 1 : 0;
        }
        int tot;
        int o = block_excl_scan(nk, wsc, &tot);
        for (int j = 0; j < per; ++j) {
            const int qq = q0 + j;
            if (qq < nact && alive[act[qq]]) nxt[o++] = act[qq];
        }
        __syncthreads();
        if (tid == 0) A.rstart[round + 1] = A.ctr[0];
        int *t = act; act = nxt; nxt = t;
        nact = tot;
        nrounds = round + 1;
        __syncthreads();
    }
    if (tid == 0) A.ctr[1] = nrounds;
    for (int k = tid; k <= nrounds; k += kTT) rs[k] = A.rstart[k];
    __syncthreads();
    // ---- child lists of the schedule (pull form): record q gathers from the records
    // eliminated next to it; sorted by node id, so the order is independent of the
    // (atomic) record numbering inside a round
    {
        const int nrec = rs[nrounds];
        for (int q = tid; q < nrec; q += kTT) {
            A.rpos[A.fu[q]] = q;
            A.cur[q] = 0;
        }
        __syncthreads();
        for (int p = tid; p < nrec; p += kTT) {
            if (A.fv1[p] >= 0) atomicAdd(A.cur + A.rpos[A.fv1[p]], 1);
            if (A.fv2[p] >= 0) atomicAdd(A.cur + A.rpos[A.fv2[p]], 1);
        }
        __syncthreads();
        __shared__ int carry2;
        if (tid == 0) { carry2 = 0; A.cptr[0] = 0; }
        __syncthreads();
        for (int base = 0; base < nrec; base += kTT) {
            const int q = base + tid;
            const int v = q < nrec ? A.cur[q] : 0;
            int tot;
            const int off = block_excl_scan(v, wsc, &tot);
            if (q < nrec) A.cptr[q + 1] = carry2 + off + v;
            __syncthreads();
            if (tid == 0) carry2 += tot;
            __syncthreads();
        }
        for (int q = tid; q < nrec; q += kTT) A.cur[q] = 0;
        __syncthreads();
        for (int p = tid; p < nrec; p += kTT)
            for (int sl = 0; sl < 2; ++sl) {
                const int v = sl ? A.fv2[p] : A.fv1[p];
                if (v < 0) continue;
                const int q = A.rpos[v];
                A.cent[A.cptr[q] + atomicAdd(A.cur + q, 1)] = 2 * p + sl;
            }
        __syncthreads();
        for (int q = tid; q < nrec; q += kTT) {
            const int b = A.cptr[q], e = A.cptr[q + 1];
            for (int k = b + 1; k < e; ++k) {           // insertion sort by child node
                const int ck = A.cent[k], key = A.fu[ck >> 1];
                int j = k - 1;
                while (j >= b && A.fu[A.cent[j] >> 1] > key) { A.cent[j + 1] = A.cent[j]; --j; }
                A.cent[j + 1] = ck;
            }
            for (int k = b; k < e; ++k) {
                A.ppos[A.cent[k]] = k;
                A.pe[k].node = A.fu[A.cent[k] >> 1];
                A.pe[k].pad = 0;
            }
            A.pk[q] = make_int4(A.fu[q], b, e - b, 0);
        }
        __syncthreads();
    }
    }   // rebuild
    // ---- numeric factor in pull form, round by round (deterministic, no atomics):
    // d_u = diag_u - sum over children p of w_p^2 / d_p; slot weights from the tree
    // edges (tval) or the fill edge of an earlier record (-w1 w2 / d)
    for (int v = tid; v < N; v += kTT) A.dcur[v] = (v < m ? A.dr[v] : A.dc[v - m]) + mu;
    __syncthreads();
    for (int rr = 0; rr < nrounds; ++rr) {
        const int q1 = rs[rr + 1];
        for (int q = rs[rr] + tid; q < q1; q += kTT) {
            const int u = A.fu[q];
            double d = A.dcur[u];
            for (int k = A.cptr[q]; k < A.cptr[q + 1]; ++k) {
                const int ce = A.cent[k], p = ce >> 1;
                const double w = (ce & 1) ? A.fw2[p] : A.fw1[p];
                d -= w * w * A.finv[p];
            }
            const int s1 = A.fs1[q], s2 = A.fs2[q];
            double w1 = 0.0, w2 = 0.0;
            if (A.fv1[q] >= 0) {
                if (s1 >= 0) w1 = A.tval[s1];
                else { const int p0 = -s1 - 1; w1 = -A.fw1[p0] * A.fw2[p0] * A.finv[p0]; }
            }
            if (A.fv2[q] >= 0) {
                if (s2 >= 0) w2 = A.tval[s2];
                else { const int p0 = -s2 - 1; w2 = -A.fw1[p0] * A.fw2[p0] * A.finv[p0]; }
            }
            const double inv = 1.0 / d;
            A.fw1[q] = w1;
            A.fw2[q] = w2;
            A.fc1[q] = w1 * inv;
            A.fc2[q] = w2 * inv;
            A.finv[q] = inv;
            if (A.fv1[q] >= 0) A.pe[A.ppos[2 * q]].coef = w1 * inv;
            if (A.fv2[q] >= 0) A.pe[A.ppos[2 * q + 1]].coef = w2 * inv;
        }
        __syncthreads();
    }
    t_fac = clock64() - t_start - t_mst;

    // ---------------- 4. PCG on M with z = M_T^-1 r ----------------
    double *vs = reinterpret_cast<double *>(dyn);                             // N doubles
    // factor records packed (one 40-byte load per eliminated node); the late
    // (small) rounds are latency-bound, so their records also go to shared memory
    Rec *frec = reinterpret_cast<Rec *>(A.frec);
    const int nrec = A.rstart[nrounds];
    for (int qq = tid; qq < nrec; qq += kTT) {
        Rec rc;
        rc.u = A.fu[qq]; rc.v1 = A.fv1[qq]; rc.v2 = A.fv2[qq]; rc.pad = 0;
        rc.c1 = A.fc1[qq]; rc.c2 = A.fc2[qq]; rc.inv = A.finv[qq];
        frec[qq] = rc;
    }
    if (A.setup_only) {
        __syncthreads();
        if (tid == 0) {
            A.st[4] = (double)nrounds;
            A.st[5] = (double)A.ctr[2];
            A.st[6] = (double)t_mst;
            A.st[7] = (double)t_fac;
            A.st[11] = rebuilt ? 1.0 : 0.0;
        }
        return;
    }
    Rec *tail = reinterpret_cast<Rec *>(dyn + 8 * (size_t)N);
    const int tail_cap = A.tail_cap;
    int R0 = nrounds;
    while (R0 > 0 && nrec - A.rstart[R0 - 1] <= tail_cap) --R0;
    const int tbase = A.rstart[R0];
    __syncthreads();
    for (int qq = tbase + tid; qq < nrec; qq += kTT) tail[qq - tbase] = frec[qq];
    __syncthreads();
    // the suffix of rounds with <= 32 records each is run by warp 0 alone, with
    // __syncwarp between rounds instead of a CTA barrier
    // round boundaries in shared memory (read every round of every preconditioner apply)
    for (int k = tid; k <= nrounds; k += kTT) rs[k] = A.rstart[k];
    __syncthreads();
    int RW = nrounds;
    while (RW > R0 && rs[RW] - rs[RW - 1] <= 32) --RW;
    const int warp_id = tid >> 5, lane_id = tid & 31;
    // in place on vs: forward elimination then back substitution (vs: r -> z)
    long long tpf = 0, tpw = 0, tpb = 0;
    // forward elimination, pull form: record q's node gathers its children's final values
    auto pull_row = [&](int q) {
        const int4 h = A.pk[q];
        double acc = vs[h.x];
        for (int k = h.y; k < h.y + h.z; ++k) {
            const PullE e = A.pe[k];
            acc = fma(-e.coef, vs[e.node], acc);
        }
        vs[h.x] = acc;
    };
    auto precond_inplace = [&]() {
        const long long c0 = clock64();
        for (int rr = 0; rr < RW; ++rr) {
            const int q0r = rs[rr], q1 = rs[rr + 1];
            if (rr < R0) {                        // read-only path: loads may run ahead
#pragma unroll 2
                for (int q = q0r + tid; q < q1; q += kTT) {
                    pull_row(q);
                }
            } else {
                const Rec *src = tail - tbase;
                for (int q = q0r + tid; q < q1; q += kTT) {
                    pull_row(q);
                }
            }
            __syncthreads();
        }
        const long long c1 = clock64();
        if (warp_id == 0) {
            const Rec *src = tail - tbase;
            for (int rr = RW; rr < nrounds; ++rr) {
                const int q = rs[rr] + lane_id;
                if (q < rs[rr + 1]) {
                    pull_row(q);
                }
                __syncwarp();
            }
            for (int rr = nrounds - 1; rr >= RW; --rr) {
                const int q = rs[rr] + lane_id;
                if (q < rs[rr + 1]) {
                    const Rec rc = src[q];
                    double xu = vs[rc.u] * rc.inv;
                    if (rc.v1 >= 0) xu = fma(-rc.c1, vs[rc.v1], xu);
                    if (rc.v2 >= 0) xu = fma(-rc.c2, vs[rc.v2], xu);
                    vs[rc.u] = xu;
                }
                __syncwarp();
            }
        }
        __syncthreads();
        const long long c2 = clock64();
        for (int rr = RW - 1; rr >= 0; --rr) {
            const int q0r = rs[rr], q1 = rs[rr + 1];
            if (rr < R0) {
#pragma unroll 2
                for (int q = q0r + tid; q < q1; q += kTT) {
                    const Rec rc = ldg_rec(frec + q);
                    double xu = vs[rc.u] * rc.inv;
                    if (rc.v1 >= 0) xu = fma(-rc.c1, vs[rc.v1], xu);
                    if (rc.v2 >= 0) xu = fma(-rc.c2, vs[rc.v2], xu);
                    vs[rc.u] = xu;
                }
            } else {
                const Rec *src = tail - tbase;
                for (int q = q0r + tid; q < q1; q += kTT) {
                    const Rec rc = src[q];
                    double xu = vs[rc.u] * rc.inv;
                    if (rc.v1 >= 0) xu = fma(-rc.c1, vs[rc.v1], xu);
                    if (rc.v2 >= 0) xu = fma(-rc.c2, vs[rc.v2], xu);
                    vs[rc.u] = xu;
                }
            }
            __syncthreads();
        }
        const long long c3 = clock64();
        tpf += c1 - c0;
        tpw += c2 - c1;
        tpb += c3 - c2;
    };
    const long long *rp = A.rowptr, *cp = A.colptr;
    double *x = A.x, *r = A.r, *p = A.p, *q = A.q;
    // init: x = 0, r = b; z = M_T^-1 r (in vs); p = z (global and in vs)
    double l_bb = 0.0;
    for (int k = tid; k < N; k += kTT) {
        const double bk = A.rhs[k];
        x[k] = 0.0;
        r[k] = bk;
        vs[k] = bk;
        l_bb = fma(bk, bk, l_bb);
    }
    const double bb = tree_block_sum(l_bb, red);     // (synchronises)
    double rr2 = bb;
    int it = 0;
    double relres = bb > 0.0 ? 1.0 : 0.0;
    double rz = 0.0;
    if (bb > 0.0) {
        const long long tp0 = clock64();
        precond_inplace();
        t_pc += clock64() - tp0;
        double l = 0.0;
        for (int k = tid; k < N; k += kTT) {
            const double zk = vs[k];
            p[k] = zk;
            l = fma(r[k], zk, l);
        }
        rz = tree_block_sum(l, red);
    }
    while (bb > 0.0) {
        relres = sqrt(rr2 / bb);
        if (relres <= A.rtol || it >= A.maxit) break;
        // q = M p (p in vs), fused <p, q>
        const long long tm0 = clock64();
        double l = 0.0;
        for (int k0 = tid; k0 < N; k0 += 4 * kTT) {
            long long b_[4], e_[4];
            double s_[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int k = k0 + j * kTT;
                b_[j] = e_[j] = 0;
                s_[j] = 0.0;
                if (k < m) { b_[j] = rp[k]; e_[j] = rp[k + 1]; s_[j] = (A.dr[k] + mu) * vs[k]; }
                else if (k < N) { b_[j] = cp[k - m]; e_[j] = cp[k - m + 1]; s_[j] = (A.dc[k - m] + mu) * vs[k]; }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int k = k0 + j * kTT;
                if (k >= N) continue;
                double sv = s_[j];
                if (k < m)
                    for (long long e = b_[j]; e < e_[j]; ++e) sv = fma(A.val[e], vs[m + A.colidx[e]], sv);
                else
                    for (long long e = b_[j]; e < e_[j]; ++e) sv = fma(A.valT[e], vs[A.rowidx[e]], sv);
                q[k] = sv;
                l = fma(vs[k], sv, l);
            }
        }
        const double pq = tree_block_sum(l, red);
        t_mv += clock64() - tm0;
        if (!(pq > 0.0)) break;
        const double alpha = rz / pq;
        // x += alpha p, r -= alpha q, ||r||^2; stage r into vs for the preconditioner
        double l2 = 0.0;
        for (int k = tid; k < N; k += kTT) {
            x[k] = fma(alpha, vs[k], x[k]);
            const double rv = fma(-alpha, q[k], r[k]);
            r[k] = rv;
            vs[k] = rv;
            l2 = fma(rv, rv, l2);
        }
        rr2 = tree_block_sum(l2, red);
        ++it;
        if (sqrt(rr2 / bb) <= A.rtol || it >= A.maxit) { relres = sqrt(rr2 / bb); break; }
        const long long tp0 = clock64();
        precond_inplace();
        t_pc += clock64() - tp0;
        double l3 = 0.0;
        for (int k = tid; k < N; k += kTT) l3 = fma(r[k], vs[k], l3);
        const double rz2 = tree_block_sum(l3, red);
        const double beta = rz2 / rz;
        rz = rz2;
        for (int k = tid; k < N; k += kTT) {           // p = z + beta p, kept in vs too
            const double pk = fma(beta, p[k], vs[k]);
            p[k] = pk;
            vs[k] = pk;
        }
        __syncthreads();
    }
    __syncthreads();
    double l_s = 0.0, l_a = 0.0;
    if (A.gradf) {
        for (int k = tid; k < N; k += kTT) {
            const double xv = x[k];
            if (k < m) {
                l_s = fma(A.gradf[k], xv, l_s);
                l_a = fma(A.a[k], xv, l_a);
            } else {
                l_s = fma(A.gradg[k - m], xv, l_s);
                l_a = fma(A.b[k - m], xv, l_a);
            }
        }
    }
    const double S = tree_block_sum(l_s, red);
    const double AD = tree_block_sum(l_a, red);
    if (tid == 0) {
        A.st[0] = (double)it;
        A.st[1] = relres;
        A.st[2] = S;
        A.st[3] = AD;
        A.st[4] = (double)nrounds;
        A.st[5] = (double)(A.tptr[N] / 2);
        A.st[6] = (double)t_mst;
        A.st[7] = (double)t_fac;
        A.st[8] = (double)t_pc;
        A.st[9] = (double)t_mv;
        A.st[10] = (double)(clock64() - t_start);
        A.st[11] = rebuilt ? 1.0 : 0.0;
        A.st[12] = (double)tpf;
        A.st[13] = (double)tpw;
        A.st[14] = (double)tpb;
        A.st[15] = (double)(R0 * 1000 + RW);
    }
}

}  // namespace pins
