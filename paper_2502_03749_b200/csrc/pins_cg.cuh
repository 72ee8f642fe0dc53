// pins_cg.cuh -- conjugate gradients on the sparsified Newton system, v2.
//
// Newton system of Alg. 2 line 12 (Eq. (9); reading R5):
//     [[Dr, X],[X^T, Dc]] (df, dg) = (rf, rg),   Dr = diag(X~ e) + mu,
//     Dc = diag(X~^T e) + mu,  X = the sparsified plan block (CSR + CSC).
// The diagonal block of the eliminated side is inverted exactly (block
// Gauss elimination) and Jacobi-preconditioned CG runs on the Schur
// complement of the kept side:
//     S df = rf - X Dc^-1 rg,   S = Dr - X Dc^-1 X^T,   dg = Dc^-1 (rg - X^T df).
// Same linear system (the full residual equals the Schur residual because dg
// is recovered exactly), half the unknowns, and about half the iterations of
// CG on the full system, whose Jacobi-scaled spectrum is symmetric about 1
// (DESIGN.md §6).
//
// cg_schur_cluster_kernel: ONE thread-block cluster of kCGC CTAs.  CTA c owns
// a contiguous slice of the kept and of the eliminated unknowns; all vectors
// live in its shared memory, and so does its slice of the CSR / CSC when it
// fits.  The two sparse products gather their operands from the owning CTA's
// shared memory (DSMEM).  Rows of degree > kHeavy are done warp-per-row (one
// thread per row would serialise a hub row).  The iteration is the
// single-reduction form of PCG (Chronopoulos & Gear): per iteration one
// product S u and ONE fused cluster reduction of (r,u), (S u,u), (r,r) --
// three cluster barriers instead of six, and no grid-wide synchronisation.
#pragma once
#include <cooperative_groups.h>

#include "pins_device.cuh"

namespace pins {
namespace cgc = cooperative_groups;

constexpr int kCGC = 8;        // CTAs per cluster
constexpr int kCGT = 1024;     // threads per CTA
constexpr int kHeavy = 16;     // rows with more entries go warp-per-row

struct CGSArgs {
    long long m, n;                        // kept / eliminated sizes
    // X (m x n, kept side = rows): CSR (rowptr, colidx, val) and CSC (colptr, rowidx, valT)
    const long long *rowptr;
    const int *colidx;
    const double *val;
    const long long *colptr;
    const int *rowidx;
    const double *valT;
    const double *dr, *dc;                 // diagonals without mu
    double mu;
    const double *rhs_r, *rhs_c;           // right-hand side parts
    double *x_r, *x_c;                     // solution parts
    double rtol;
    int maxit;
    const double *grad_r, *grad_c, *a_r, *a_c;   // optional slope / <(a,b), d> terms
    double *st;                            // [0] iterations [1] rel. residual [2] slope [3] <(a,b),d>
    int R, Cc;                             // slice sizes (kept / eliminated) per CTA
    int smem;                              // dynamic shared memory bytes
};

// cluster-wide sums of NV values; identical (fixed-order) result in every CTA
template <int NV>
__device__ __forceinline__ void cluster_sums(cgc::cluster_group &cl, const double (&v)[NV], double (*wsum)[4],
                                             double *red, double *bc, double (&o)[NV]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        const double t = warp_sum(v[q]);
        if (lane == 0) wsum[warp][q] = t;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const double t = warp_sum(wsum[lane][q]);
            if (lane == 0) red[q] = t;
        }
    }
    cl.sync();
    if (warp == 0) {
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            double t = 0.0;
            if (lane < kCGC) t = cl.map_shared_rank(red, lane)[q];
            t = warp_sum(t);
            if (lane == 0) bc[q] = t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NV; ++q) o[q] = bc[q];
}

// local slice of a compressed sparse matrix: pointers (int offsets) in smem,
// index / value arrays in smem when they fit, else in global memory
struct LocalCS {
    const int *ptr;        // [n + 1] offsets from the slice's first entry
    const int *idx;
    const double *val;
    const int *heavy;      // local ids of rows with degree > kHeavy
    int nheavy;
};

// y_k = sum_e val_e * src(idx_e), src owned by CTA idx / chunk in DSMEM.
// Light rows: thread per row; heavy rows: warp per row.  Calls f(k, sum).
template <class F>
__device__ __forceinline__ void cs_apply(cgc::cluster_group &cl, const LocalCS &L, int nloc, const double *src,
                                         int chunk, F f) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int k = tid; k < nloc; k += kCGT) {
        const int b = L.ptr[k], e = L.ptr[k + 1];
        if (e - b > kHeavy) continue;
        double s = 0.0;
        for (int q = b; q < e; ++q) {
            const int j = L.idx[q];
            const int own = j / chunk;
            s = fma(L.val[q], cl.map_shared_rank(src, own)[j - own * chunk], s);
        }
        f(k, s);
    }
    for (int h = warp; h < L.nheavy; h += kCGT / 32) {
        const int k = L.heavy[h];
        const int b = L.ptr[k], e = L.ptr[k + 1];
        double s = 0.0;
        for (int q = b + lane; q < e; q += 32) {
            const int j = L.idx[q];
            const int own = j / chunk;
            s = fma(L.val[q], cl.map_shared_rank(src, own)[j - own * chunk], s);
        }
        s = warp_sum(s);
        if (lane == 0) f(k, s);
    }
}

__global__ void __cluster_dims__(kCGC, 1, 1) __launch_bounds__(kCGT, 1) cg_schur_cluster_kernel(CGSArgs A) {
    extern __shared__ __align__(16) unsigned char smraw[];
    __shared__ double wsum[32][4];
    __shared__ double redA[4], redB[4], bc[4];
    __shared__ int nh_r, nh_c;
    cgc::cluster_group cl = cgc::this_cluster();
    const int rank = (int)cl.block_rank();
    const int tid = threadIdx.x;
    const int R = A.R, Cc = A.Cc;
    const long long r0 = (long long)rank * R, r1 = min((long long)(rank + 1) * R, A.m);
    const long long c0 = (long long)rank * Cc, c1 = min((long long)(rank + 1) * Cc, A.n);
    const int nr = (int)max(0LL, r1 - r0), nc = (int)max(0LL, c1 - c0);
    const double mu = A.mu;

    // ---- shared-memory layout ----
    double *p = reinterpret_cast<double *>(smraw);
    double *r = p + R, *u = r + R, *s = u + R, *w = s + R, *x = w + R, *idS = x + R, *drp = idS + R;
    double *t = drp + R, *idc = t + Cc;
    int *iptr_r = reinterpret_cast<int *>(idc + Cc);
    int *iptr_c = iptr_r + (R + 1);
    int *heavy_r = iptr_c + (Cc + 1);
    int *heavy_c = heavy_r + R;
    unsigned char *free0 = reinterpret_cast<unsigned char *>(heavy_c + Cc);
    size_t used = (size_t)(free0 - smraw);
    used = (used + 15) & ~(size_t)15;
    size_t room = A.smem > (int)used ? (size_t)A.smem - used : 0;
    unsigned char *cache = smraw + used;

    // ---- local matrix slices (cached in smem when they fit) ----
    const long long rb = nr ? A.rowptr[r0] : 0, re = nr ? A.rowptr[r1] : 0;
    const long long cb = nc ? A.colptr[c0] : 0, ce = nc ? A.colptr[c1] : 0;
    const long long nzr = re - rb, nzc = ce - cb;
    LocalCS Lr, Lc;
    Lr.ptr = iptr_r;
    Lc.ptr = iptr_c;
    Lr.heavy = heavy_r;
    Lc.heavy = heavy_c;
    if (tid == 0) { nh_r = 0; nh_c = 0; }
    __syncthreads();
    for (int k = tid; k <= nr; k += kCGT) iptr_r[k] = (int)(A.rowptr[r0 + k] - rb);
    for (int k = tid; k <= nc; k += kCGT) iptr_c[k] = (int)(A.colptr[c0 + k] - cb);
    // heavy lists in index order (deterministic work assignment): ordered compaction by
    // warp ballots and a prefix over the warps of each block-sized batch
    {
        __shared__ int wcnt[kCGT / 32];
        const int lane = tid & 31, warp = tid >> 5;
        for (int side = 0; side < 2; ++side) {
            const int len = side == 0 ? nr : nc;
            const long long *pp = side == 0 ? A.rowptr + r0 : A.colptr + c0;
            int *out = side == 0 ? heavy_r : heavy_c;
            int base = 0;
            for (int k0 = 0; k0 < len; k0 += kCGT) {
                const int k = k0 + tid;
                const bool h = k < len && pp[k + 1] - pp[k] > kHeavy;
                const unsigned bal = __ballot_sync(0xffffffffu, h);
                if (lane == 0) wcnt[warp] = __popc(bal);
                __syncthreads();
                int off = base, tot = 0;
                for (int w2 = 0; w2 < kCGT / 32; ++w2) {
                    if (w2 < warp) off += wcnt[w2];
                    tot += wcnt[w2];
                }
                if (h) out[off + __popc(bal & ((1u << lane) - 1u))] = k;
                base += tot;
                __syncthreads();
            }
            if (tid == 0) (side == 0 ? nh_r : nh_c) = base;
        }
    }
    const size_t need_r = (size_t)nzr * 12, need_c = (size_t)nzc * 12;
    const bool cache_r = need_r <= room;
    const bool cache_c = need_c + (cache_r ? need_r : 0) <= room;
    double *vr_s = reinterpret_cast<double *>(cache);
    double *vc_s = vr_s + (cache_r ? nzr : 0);
    int *ir_s = reinterpret_cast<int *>(vc_s + (cache_c ? nzc : 0));
    int *ic_s = ir_s + (cache_r ? nzr : 0);
    if (cache_r) {
        for (long long q = tid; q < nzr; q += kCGT) {
            vr_s[q] = A.val[rb + q];
            ir_s[q] = A.colidx[rb + q];
        }
        Lr.val = vr_s;
        Lr.idx = ir_s;
    } else {
        Lr.val = A.val + rb;
        Lr.idx = A.colidx + rb;
    }
    if (cache_c) {
        for (long long q = tid; q < nzc; q += kCGT) {
            vc_s[q] = A.valT[cb + q];
            ic_s[q] = A.rowidx[cb + q];
        }
        Lc.val = vc_s;
        Lc.idx = ic_s;
    } else {
        Lc.val = A.valT + cb;
        Lc.idx = A.rowidx + cb;
    }

    // ---- setup: Dc^-1, Schur diagonal, Schur right-hand side ----
    for (int k = tid; k < nc; k += kCGT) idc[k] = 1.0 / (A.dc[c0 + k] + mu);
    double l_bb = 0.0;
    for (int k = tid; k < nr; k += kCGT) {
        const long long i = r0 + k;
        const double d = A.dr[i] + mu;
        double sd = d, bs = A.rhs_r[i];
        for (long long e = A.rowptr[i]; e < A.rowptr[i + 1]; ++e) {
            const int j = A.colidx[e];
            const double v = A.val[e];
            const double ic = 1.0 / (A.dc[j] + mu);
            sd -= v * v * ic;
            bs -= v * ic * A.rhs_c[j];
        }
        drp[k] = d;
        idS[k] = 1.0 / fmax(sd, mu);
        r[k] = bs;
        x[k] = 0.0;
        u[k] = bs * idS[k];
        l_bb = fma(A.rhs_r[i], A.rhs_r[i], l_bb);
    }
    for (int k = tid; k < nc; k += kCGT) l_bb = fma(A.rhs_c[c0 + k], A.rhs_c[c0 + k], l_bb);
    __syncthreads();
    Lr.nheavy = nh_r;
    Lc.nheavy = nh_c;

    // w = S u = Dr u - X (Dc^-1 (X^T u)); needs u complete cluster-wide
    auto apply_S = [&]() {
        cl.sync();                                   // u complete everywhere
        cs_apply(cl, Lc, nc, u, R, [&](int k, double v) { t[k] = v * idc[k]; });
        cl.sync();                                   // t complete everywhere
        cs_apply(cl, Lr, nr, t, Cc, [&](int k, double v) { w[k] = fma(drp[k], u[k], -v); });
        __syncthreads();                             // heavy-row results visible
    };

    apply_S();
    double gam, del, rr, bb;
    {
        double l_g = 0.0, l_d = 0.0, l_r = 0.0;
        for (int k = tid; k < nr; k += kCGT) {
            l_g = fma(r[k], u[k], l_g);
            l_d = fma(w[k], u[k], l_d);
            l_r = fma(r[k], r[k], l_r);
        }
        const double in4[4] = {l_g, l_d, l_r, l_bb};
        double o4[4];
        cluster_sums<4>(cl, in4, wsum, redA, bc, o4);
        gam = o4[0]; del = o4[1]; rr = o4[2]; bb = o4[3];
    }
    for (int k = tid; k < nr; k += kCGT) {
        p[k] = u[k];
        s[k] = w[k];
    }
    double alpha = del > 0.0 ? gam / del : 0.0;
    int it = 0;
    double relres = bb > 0.0 ? sqrt(rr / bb) : 0.0;
    int parity = 0;
    while (bb > 0.0 && relres > A.rtol && it < A.maxit && del > 0.0) {
        for (int k = tid; k < nr; k += kCGT) {
            x[k] = fma(alpha, p[k], x[k]);
            const double rv = fma(-alpha, s[k], r[k]);
            r[k] = rv;
            u[k] = rv * idS[k];
        }
        apply_S();
        double l_g = 0.0, l_d = 0.0, l_r = 0.0;
        for (int k = tid; k < nr; k += kCGT) {
            l_g = fma(r[k], u[k], l_g);
            l_d = fma(w[k], u[k], l_d);
            l_r = fma(r[k], r[k], l_r);
        }
        const double in3[3] = {l_g, l_d, l_r};
        double o3[3];
        cluster_sums<3>(cl, in3, wsum, parity ? redB : redA, bc, o3);
        parity ^= 1;
        ++it;
        rr = o3[2];
        relres = sqrt(rr / bb);
        const double gnew = o3[0];
        const double beta = gnew / gam;
        const double den = o3[1] - beta * gnew / alpha;
        gam = gnew;
        if (!(den > 0.0)) break;
        alpha = gnew / den;
        for (int k = tid; k < nr; k += kCGT) {
            p[k] = fma(beta, p[k], u[k]);
            s[k] = fma(beta, s[k], w[k]);
        }
    }
    // ---- back-substitution dg = Dc^-1 (rc - X^T df); write the solution ----
    cl.sync();
    double l_s = 0.0, l_a = 0.0;
    for (int k = tid; k < nr; k += kCGT) {
        const long long i = r0 + k;
        A.x_r[i] = x[k];
        if (A.grad_r) {
            l_s = fma(A.grad_r[i], x[k], l_s);
            l_a = fma(A.a_r[i], x[k], l_a);
        }
    }
    cs_apply(cl, Lc, nc, x, R, [&](int k, double v) { t[k] = v; });
    __syncthreads();
    for (int k = tid; k < nc; k += kCGT) {
        const long long j = c0 + k;
        const double dg = (A.rhs_c[j] - t[k]) * idc[k];
        A.x_c[j] = dg;
        if (A.grad_c) {
            l_s = fma(A.grad_c[j], dg, l_s);
            l_a = fma(A.a_c[j], dg, l_a);
        }
    }
    const double in2[2] = {l_s, l_a};
    double o2[2];
    cluster_sums<2>(cl, in2, wsum, parity ? redB : redA, bc, o2);
    if (rank == 0 && tid == 0) {
        A.st[0] = (double)it;
        A.st[1] = relres;
        A.st[2] = o2[0];
        A.st[3] = o2[1];
    }
    cl.sync();   // keep every CTA's shared memory alive until all remote reads are done
}

}  // namespace pins
