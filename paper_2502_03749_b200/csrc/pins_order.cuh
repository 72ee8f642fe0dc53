// pins_order.cuh -- locality ordering of point clouds for the dense passes.
//
// pins_solve permutes the rows (source points) and the columns (target
// points) of a point-cost problem into Morton (Z-curve) order of their
// coordinates before solving, and scatters the potentials back at the end.
// Nearby points then share a warp (rows) and a staged chunk (columns), so the
// negligible-entry skip of pins_pass.cuh happens for whole warps instead of
// single lanes.  The permutation changes nothing but summation order: PINS
// is equivariant under relabelling of the points (Eq. (1)).
#pragma once
#include <cub/device/device_radix_sort.cuh>

#include "pins_device.cuh"

namespace pins {

// per-dimension bounding box of x (m x d) and y (n x d): one block of 1024
__global__ void __launch_bounds__(1024) bbox_kernel(long long m, long long n, int d, const double *x,
                                                    const double *y, double *lohi) {
    __shared__ double slo[32][16], shi[32][16];
    double lo[16], hi[16];
    for (int k = 0; k < 16; ++k) { lo[k] = INFINITY; hi[k] = -INFINITY; }
    for (long long p = threadIdx.x; p < m + n; p += 1024) {
        const double *v = p < m ? x + p * d : y + (p - m) * d;
        for (int k = 0; k < d; ++k) { lo[k] = fmin(lo[k], v[k]); hi[k] = fmax(hi[k], v[k]); }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int k = 0; k < d; ++k) {
        double a = lo[k], b = hi[k];
        for (int o = 16; o > 0; o >>= 1) {
            a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
            b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
        }
        if (lane == 0) { slo[warp][k] = a; shi[warp][k] = b; }
    }
    __syncthreads();
    if (threadIdx.x < d) {
        double a = INFINITY, b = -INFINITY;
        for (int w = 0; w < 32; ++w) { a = fmin(a, slo[w][threadIdx.x]); b = fmax(b, shi[w][threadIdx.x]); }
        lohi[threadIdx.x] = a;
        lohi[16 + threadIdx.x] = b;
    }
}

// Morton key: B = min(21, 64 / d) bits per dimension, interleaved from the
// most significant level down; also writes the identity permutation.
__global__ void morton_kernel(long long np, int d, const double *x, const double *lohi,
                              unsigned long long *key, int *idx) {
    const int B = min(21, 64 / d);
    const double levels = (double)((1ull << B) - 1);
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < np;
         p += (long long)gridDim.x * blockDim.x) {
        unsigned q[16];
        for (int k = 0; k < d; ++k) {
            const double lo = lohi[k], span = lohi[16 + k] - lo;
            const double t = span > 0.0 ? (x[p * d + k] - lo) / span : 0.0;
            q[k] = (unsigned)fmin(levels, fmax(0.0, rint(t * levels)));
        }
        unsigned long long kk = 0;
        for (int l = B - 1; l >= 0; --l)
            for (int k = 0; k < d; ++k) kk = (kk << 1) | ((q[k] >> l) & 1u);
        key[p] = kk;
        idx[p] = (int)p;
    }
}

// xp[k] = x[perm[k]] (rows of width d), ap[k] = a[perm[k]]
__global__ void gather_points_kernel(long long np, int d, const int *perm, const double *x, const double *a,
                                     double *xp, double *ap) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < np;
         k += (long long)gridDim.x * blockDim.x) {
        const long long src = perm[k];
        for (int t = 0; t < d; ++t) xp[k * d + t] = x[src * d + t];
        ap[k] = a[src];
    }
}

// out[perm[k]] = in[k]
__global__ void scatter_kernel(long long np, const int *perm, const double *in, double *out) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < np;
         k += (long long)gridDim.x * blockDim.x)
        out[perm[k]] = in[k];
}

}  // namespace pins
