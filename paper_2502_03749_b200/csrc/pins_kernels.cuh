// pins_kernels.cuh -- the PINS dense passes, sparsification, CSR/CSC builders
// and the cooperative CG kernel.  Included once by pins_api.cu.
#pragma once
#include <cooperative_groups.h>

#include "pins_device.cuh"

namespace pins {
namespace cgx = cooperative_groups;

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

// =========================================================================
// Sparsification of a caller-given dense plan block P (pins_sparsify_dense;
// PAPER.md:255-256, Alg. 2 line 11, reading R3): keep P_ij >= tau, compact
// into a row-major CSR with columns ascending.  One warp per row: each lane
// tests one column of a 32-column chunk, __ballot_sync gives the chunk's keep
// mask, popc of the lanes below gives the lane's slot (warp-ballot
// compaction); the row starts come from a block prefix scan of the counts
// (scan_counts_kernel).  Exact: a comparison per entry, values copied bitwise.
// =========================================================================
__global__ void sparsify_count_kernel(long long m, long long n, const double *__restrict__ P, long long ldp,
                                      double tau, int *cnt) {
    const int lane = threadIdx.x & 31;
    const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = gw; i < m; i += nw) {
        const double *row = P + i * ldp;
        int c = 0;
        for (long long j0 = 0; j0 < n; j0 += 32) {
            const long long j = j0 + lane;
            const bool keep = j < n && __ldg(row + j) >= tau;
            c += __popc(__ballot_sync(0xffffffffu, keep));
        }
        if (lane == 0) cnt[i] = c;
    }
}

__global__ void sparsify_fill_kernel(long long m, long long n, const double *__restrict__ P, long long ldp,
                                     double tau, const long long *rowptr, int *colidx, double *val) {
    const int lane = threadIdx.x & 31;
    const unsigned below = (1u << lane) - 1u;
    const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = gw; i < m; i += nw) {
        const double *row = P + i * ldp;
        long long dst = rowptr[i];
        for (long long j0 = 0; j0 < n; j0 += 32) {
            const long long j = j0 + lane;
            const double p = j < n ? __ldg(row + j) : 0.0;
            const bool keep = j < n && p >= tau;
            const unsigned mask = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const long long q = dst + __popc(mask & below);
                colidx[q] = (int)j;
                val[q] = p;
            }
            dst += __popc(mask);
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

}  // namespace pins
