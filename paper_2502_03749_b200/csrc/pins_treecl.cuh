// pins_treecl.cuh -- spanning-tree preconditioned CG on one thread-block cluster.
//
// The factor of M_T (pins_tree.cuh: maximum spanning forest + exact tree
// contraction) is built by tree_pcg_kernel in setup-only mode; this kernel then
// runs the PCG of Alg. 2 line 12 (reading R5) on the full system
//     M = [[Dr, X],[X^T, Dc]]
// with the work split by role inside one 8-CTA cluster:
//  * CTAs 1..7 ("workers") own contiguous slices of the m + n unknowns; x, r,
//    p, q/z live in their shared memory, the sparse products gather p from the
//    owning worker's shared memory (DSMEM); hub rows go warp-per-row;
//  * CTA 0 ("solver") holds the whole preconditioner vector in its shared
//    memory: workers store r into it (DSMEM), CTA 0 applies M_T^-1 in place
//    (forward elimination / back substitution, round by round, the small late
//    rounds by one warp), workers read z back.
// Five cluster barriers per iteration plus the tree solve; no grid-wide
// synchronisation.  Same stopping rule as the oracle (||r||_2 <= rtol ||b||_2).
#pragma once
#include "pins_cg.cuh"
#include "pins_tree.cuh"

namespace pins {

constexpr int kTCW = 7;                  // worker CTAs (CTA 0 is the tree solver)
constexpr int kTCHeavy = 16;

struct TreeCLArgs {
    int m, n;
    const long long *rowptr;
    const int *colidx;
    const double *val;
    const long long *colptr;
    const int *rowidx;
    const double *valT;
    const double *dr, *dc;
    double mu;
    const double *rhs;
    double *x;
    double rtol;
    int maxit;
    const double *gradf, *gradg, *a, *b;
    double *st;                          // [0] iterations [1] relres [2] slope [3] <(a,b),d>
    const double *frec;                  // packed factor records (Rec, 40 B each)
    const int *rstart;                   // round boundaries
    const int *ctr;                      // [1] rounds
    const int *cptr;                     // pull form of the forward elimination (pins_tree.cuh)
    const int4 *pk;
    const PullE *pe;
    int R;                               // unknowns per worker
    int tail_cap;                        // factor records cached in CTA 0's shared memory
    int use_x0;                          // 1: start from alpha x (x = the previous system's solution),
                                         //    alpha = <x,b>/<x,Mx> (the A-norm-optimal multiple)
};

// y = M p for one worker's slice (p gathered from the owners through DSMEM).
// f(k, s) receives the row sum for local node k.
template <class F>
__device__ __forceinline__ void treecl_spmv(cgc::cluster_group &cl, const TreeCLArgs &A, int k0, int nloc,
                                            const double *p_loc, F f) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int m = A.m, R = A.R;
    auto gather = [&](int node) -> double {
        const int own = node / R;
        return cl.map_shared_rank(p_loc, 1 + own)[node - own * R];
    };
    // light nodes: one thread each
    for (int k = tid; k < nloc; k += kCGT) {
        const int node = k0 + k;
        long long b, e;
        if (node < m) { b = A.rowptr[node]; e = A.rowptr[node + 1]; }
        else { b = A.colptr[node - m]; e = A.colptr[node - m + 1]; }
        if (e - b > kTCHeavy) continue;
        double s = 0.0;
        if (node < m)
            for (long long q = b; q < e; ++q) s = fma(A.val[q], gather(m + A.colidx[q]), s);
        else
            for (long long q = b; q < e; ++q) s = fma(A.valT[q], gather(A.rowidx[q]), s);
        f(k, s);
    }
    // heavy nodes: one warp each (found by a ballot over each warp's chunk)
    for (int base = warp * 32; base < nloc; base += kCGT) {
        const int k = base + lane;
        bool heavy = false;
        if (k < nloc) {
            const int node = k0 + k;
            const long long d = node < m ? A.rowptr[node + 1] - A.rowptr[node]
                                         : A.colptr[node - m + 1] - A.colptr[node - m];
            heavy = d > kTCHeavy;
        }
        unsigned msk = __ballot_sync(0xffffffffu, heavy);
        while (msk) {
            const int l = __ffs(msk) - 1;
            msk &= msk - 1u;
            const int kk = base + l, node = k0 + kk;
            double s = 0.0;
            if (node < m) {
                for (long long q = A.rowptr[node] + lane; q < A.rowptr[node + 1]; q += 32)
                    s = fma(A.val[q], gather(m + A.colidx[q]), s);
            } else {
                for (long long q = A.colptr[node - m] + lane; q < A.colptr[node - m + 1]; q += 32)
                    s = fma(A.valT[q], gather(A.rowidx[q]), s);
            }
            s = warp_sum(s);
            if (lane == 0) f(kk, s);
        }
    }
}

__global__ void __cluster_dims__(kCGC, 1, 1) __launch_bounds__(kCGT, 1) cg_tree_cluster_kernel(TreeCLArgs A) {
    extern __shared__ __align__(16) unsigned char dyn[];
    __shared__ double wsum[32][4];
    __shared__ double redA[4], redB[4], bc[4];
    __shared__ int rs[kTreeMaxRounds + 1];
    cgc::cluster_group cl = cgc::this_cluster();
    const int rank = (int)cl.block_rank();
    const int tid = threadIdx.x;
    const int m = A.m, N = A.m + A.n, R = A.R;
    const double mu = A.mu;
    const bool worker = rank > 0;
    const int k0 = worker ? (rank - 1) * R : 0;
    const int nloc = worker ? max(0, min(R, N - k0)) : 0;
    // worker slices: x, r, p, q (q also holds z); diagonal
    double *xs = reinterpret_cast<double *>(dyn);
    double *rsl = xs + R, *ps = rsl + R, *qs = ps + R, *dg = qs + R;
    // solver: the preconditioner vector and the cached factor tail
    double *vs = reinterpret_cast<double *>(dyn);
    double *vs0 = cl.map_shared_rank(vs, 0);          // CTA 0's vector, seen from any CTA
    const int nrounds = A.ctr[1];
    for (int k = tid; k <= nrounds; k += kCGT) rs[k] = A.rstart[k];
    const Rec *frec = reinterpret_cast<const Rec *>(A.frec);
    Rec *tail = reinterpret_cast<Rec *>(dyn + 8 * (size_t)N);
    // the tail's forward (pull) lists: record headers and entries
    int4 *tl_h = reinterpret_cast<int4 *>(
        (reinterpret_cast<uintptr_t>(tail + A.tail_cap) + 15) & ~uintptr_t(15));
    PullE *tl_e = reinterpret_cast<PullE *>(tl_h + A.tail_cap);
    __syncthreads();
    const int nrec = rs[nrounds];
    int R0 = nrounds;
    while (R0 > 0 && nrec - rs[R0 - 1] <= A.tail_cap && A.cptr[nrec] - A.cptr[rs[R0 - 1]] <= 2 * A.tail_cap) --R0;
    const int tbase = rs[R0];
    const int kbase = A.cptr[tbase];
    int RW = nrounds;
    while (RW > R0 && rs[RW] - rs[RW - 1] <= 32) --RW;
    if (!worker) {
        for (int q = tbase + tid; q < nrec; q += kCGT) {
            tail[q - tbase] = frec[q];
            int4 h = A.pk[q];
            h.y -= kbase;
            tl_h[q - tbase] = h;
        }
        for (int k = kbase + tid; k < A.cptr[nrec]; k += kCGT) tl_e[k - kbase] = A.pe[k];
    }
    const int lane = tid & 31, warp = tid >> 5;
    // forward elimination, pull form: record q's node gathers its children's final values
    // (lists of the early rounds from global memory, of the cached tail from shared memory)
    auto pull_row = [&](int q) {
        const bool t = q >= tbase;
        const int4 h = t ? tl_h[q - tbase] : A.pk[q];
        const PullE *E = t ? tl_e : A.pe;
        double acc = vs[h.x];
        for (int k = h.y; k < h.y + h.z; ++k) {
            const PullE e = E[k];
            acc = fma(-e.coef, vs[e.node], acc);
        }
        vs[h.x] = acc;
    };
    // M_T^-1 in place on vs (CTA 0 only)
    long long t_fwd = 0, t_warp = 0, t_bwd = 0;
    const long long t_start = clock64();
    auto tree_apply = [&]() {
        const long long c0 = clock64();
        for (int rr = 0; rr < RW; ++rr) {
            const int q0r = rs[rr], q1 = rs[rr + 1];
            if (rr < R0) {
                for (int q = q0r + tid; q < q1; q += kCGT) {
                    pull_row(q);
                }
            } else {
                for (int q = q0r + tid; q < q1; q += kCGT) {
                    pull_row(q);
                }
            }
            __syncthreads();
        }
        const long long c1 = clock64();
        if (warp == 0) {
            for (int rr = RW; rr < nrounds; ++rr) {
                const int q = rs[rr] + lane;
                if (q < rs[rr + 1]) {
                    pull_row(q);
                }
                __syncwarp();
            }
            for (int rr = nrounds - 1; rr >= RW; --rr) {
                const int q = rs[rr] + lane;
                if (q < rs[rr + 1]) {
                    const Rec rc = tail[q - tbase];
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
                for (int q = q0r + tid; q < q1; q += kCGT) {
                    const Rec rc = ldg_rec(frec + q);
                    double xu = vs[rc.u] * rc.inv;
                    if (rc.v1 >= 0) xu = fma(-rc.c1, vs[rc.v1], xu);
                    if (rc.v2 >= 0) xu = fma(-rc.c2, vs[rc.v2], xu);
                    vs[rc.u] = xu;
                }
            } else {
                for (int q = q0r + tid; q < q1; q += kCGT) {
                    const Rec rc = tail[q - tbase];
                    double xu = vs[rc.u] * rc.inv;
                    if (rc.v1 >= 0) xu = fma(-rc.c1, vs[rc.v1], xu);
                    if (rc.v2 >= 0) xu = fma(-rc.c2, vs[rc.v2], xu);
                    vs[rc.u] = xu;
                }
            }
            __syncthreads();
        }
        t_fwd += c1 - c0;
        t_warp += c2 - c1;
        t_bwd += clock64() - c2;
    };

    // ---- init: x = x0, r = b - M x0, z = M_T^-1 r, p = z ----
    double o1[1];
    double bb, rr0;
    if (A.use_x0) {
        // x0 = alpha xp, xp = the previous Newton system's solution (still in A.x)
        for (int k = tid; k < nloc; k += kCGT) {
            const int node = k0 + k;
            dg[k] = (node < m ? A.dr[node] : A.dc[node - m]) + mu;
            ps[k] = A.x[node];
        }
        cl.sync();                                           // xp slices complete everywhere
        if (worker)
            treecl_spmv(cl, A, k0, nloc, ps, [&](int k, double s) { qs[k] = fma(dg[k], ps[k], s); });
        __syncthreads();
        double l_pq = 0.0, l_pb = 0.0;
        for (int k = tid; k < nloc; k += kCGT) {
            l_pq = fma(ps[k], qs[k], l_pq);
            l_pb = fma(ps[k], A.rhs[k0 + k], l_pb);
        }
        double o2i[2];
        {
            const double in2[2] = {l_pq, l_pb};
            cluster_sums<2>(cl, in2, wsum, redB, bc, o2i);
        }
        const double alpha0 = o2i[0] > 0.0 ? o2i[1] / o2i[0] : 0.0;
        double l_bb = 0.0, l_rr = 0.0;
        for (int k = tid; k < nloc; k += kCGT) {
            const int node = k0 + k;
            const double bk = A.rhs[node];
            xs[k] = alpha0 * ps[k];
            const double rv = fma(-alpha0, qs[k], bk);
            rsl[k] = rv;
            vs0[node] = rv;
            l_bb = fma(bk, bk, l_bb);
            l_rr = fma(rv, rv, l_rr);
        }
        double o2r[2];
        {
            const double in2[2] = {l_bb, l_rr};
            cluster_sums<2>(cl, in2, wsum, redA, bc, o2r);  // also: vs0 complete
        }
        bb = o2r[0];
        rr0 = o2r[1];
    } else {
        double l_bb = 0.0;
        for (int k = tid; k < nloc; k += kCGT) {
            const int node = k0 + k;
            const double bk = A.rhs[node];
            xs[k] = 0.0;
            rsl[k] = bk;
            dg[k] = (node < m ? A.dr[node] : A.dc[node - m]) + mu;
            vs0[node] = bk;
            l_bb = fma(bk, bk, l_bb);
        }
        {
            const double in1[1] = {l_bb};
            cluster_sums<1>(cl, in1, wsum, redA, bc, o1);      // also: vs0 complete
        }
        bb = o1[0];
        rr0 = bb;
    }
    if (!worker && bb > 0.0) tree_apply();
    cl.sync();
    double l_rz = 0.0;
    for (int k = tid; k < nloc; k += kCGT) {
        const double z = vs0[k0 + k];
        ps[k] = z;
        l_rz = fma(rsl[k], z, l_rz);
    }
    {
        const double in1[1] = {l_rz};
        cluster_sums<1>(cl, in1, wsum, redB, bc, o1);
    }
    double rz = o1[0];
    double rr2 = rr0, relres = bb > 0.0 ? sqrt(rr0 / bb) : 0.0;
    int it = 0;
    while (bb > 0.0 && relres > A.rtol && it < A.maxit) {
        cl.sync();                                           // p complete everywhere
        double l_pq = 0.0;
        if (worker)
            treecl_spmv(cl, A, k0, nloc, ps, [&](int k, double s) { qs[k] = fma(dg[k], ps[k], s); });
        __syncthreads();
        for (int k = tid; k < nloc; k += kCGT) l_pq = fma(ps[k], qs[k], l_pq);
        {
            const double in1[1] = {l_pq};
            cluster_sums<1>(cl, in1, wsum, redA, bc, o1);
        }
        const double pq = o1[0];
        if (!(pq > 0.0)) break;
        const double alpha = rz / pq;
        double l_rr = 0.0;
        for (int k = tid; k < nloc; k += kCGT) {
            xs[k] = fma(alpha, ps[k], xs[k]);
            const double rv = fma(-alpha, qs[k], rsl[k]);
            rsl[k] = rv;
            vs0[k0 + k] = rv;
            l_rr = fma(rv, rv, l_rr);
        }
        {
            const double in1[1] = {l_rr};
            cluster_sums<1>(cl, in1, wsum, redB, bc, o1);  // also: vs0 complete
        }
        rr2 = o1[0];
        ++it;
        relres = sqrt(rr2 / bb);
        if (relres <= A.rtol || it >= A.maxit) break;
        if (!worker) tree_apply();
        cl.sync();                                           // z ready in CTA 0
        double l_rz2 = 0.0;
        for (int k = tid; k < nloc; k += kCGT) {
            const double z = vs0[k0 + k];
            qs[k] = z;                                       // q is free: keep z
            l_rz2 = fma(rsl[k], z, l_rz2);
        }
        {
            const double in1[1] = {l_rz2};
            cluster_sums<1>(cl, in1, wsum, redA, bc, o1);
        }
        const double beta = o1[0] / rz;
        rz = o1[0];
        for (int k = tid; k < nloc; k += kCGT) ps[k] = fma(beta, ps[k], qs[k]);
    }
    // ---- output ----
    cl.sync();      // every CTA is past the last reduction before its slots are reused
    double l_s = 0.0, l_a = 0.0;
    for (int k = tid; k < nloc; k += kCGT) {
        const int node = k0 + k;
        const double xv = xs[k];
        A.x[node] = xv;
        if (A.gradf) {
            if (node < m) {
                l_s = fma(A.gradf[node], xv, l_s);
                l_a = fma(A.a[node], xv, l_a);
            } else {
                l_s = fma(A.gradg[node - m], xv, l_s);
                l_a = fma(A.b[node - m], xv, l_a);
            }
        }
    }
    double o2[2];
    {
        const double in2[2] = {l_s, l_a};
        cluster_sums<2>(cl, in2, wsum, redB, bc, o2);
    }
    if (rank == 0 && tid == 0) {
        A.st[0] = (double)it;
        A.st[1] = relres;
        A.st[2] = o2[0];
        A.st[3] = o2[1];
        // dev instrumentation (PINS_TREE_STATS): rounds, CTA 0's cycles in the tree solve
        A.st[4] = (double)nrounds;
        A.st[8] = (double)(t_fwd + t_warp + t_bwd);
        A.st[10] = (double)(clock64() - t_start);
        A.st[12] = (double)t_fwd;
        A.st[13] = (double)t_warp;
        A.st[14] = (double)t_bwd;
        A.st[15] = (double)(R0 * 1000 + RW);
    }
    cl.sync();   // keep shared memory alive until every remote access is done
}

}  // namespace pins
