// pins_device.cuh -- device building blocks of the PINS hot path (sm_100a).
//
//  * pexp():   full-precision fp64 exp, table-driven (2^(j/64) hi/lo table in
//              shared memory, degree-6 polynomial on |r| <= ln2/128).  ~10
//              fp64 pipe ops instead of ~20 for the libdevice routine.
//  * CostDesc: the cost source (dense C or point coordinates).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pins {

constexpr int kThreads = 256;          // 8 warps per CTA (CG, vector kernels)
constexpr int kWarps = kThreads / 32;

struct ExpTable {
    double hi[64];
    double lo[64];
};

// exp(z) for any z: 0 below -745.2 (with graceful denormals), +inf above 709.78,
// NaN passthrough.  Max error ~1 ulp.
__device__ __forceinline__ double pexp(double z, const double *__restrict__ thi,
                                       const double *__restrict__ tlo) {
    if (!(z > -745.2)) return (z != z) ? z : 0.0;
    if (z > 709.78) return __longlong_as_double(0x7ff0000000000000LL);
    const double kL2E64 = 92.332482616893657;                  // 64 / ln 2
    const double kLn2Hi = 6.93147180369123816490e-01 * 0.015625;  // ln2_hi / 64 (21 trailing zero bits)
    const double kLn2Lo = 1.90821492927058770002e-10 * 0.015625;  // ln2_lo / 64
    const double kShift = 6755399441055744.0;                    // 1.5 * 2^52
    double t = fma(z, kL2E64, kShift);
    double kd = t - kShift;
    int k = __double2loint(t);
    double r = fma(-kd, kLn2Hi, z);
    r = fma(-kd, kLn2Lo, r);
    double p = fma(r, 1.0 / 720.0, 1.0 / 120.0);
    p = fma(p, r, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = p * r;                                                    // expm1(r)
    int j = k & 63;
    int e = k >> 6;
    double th = thi[j];
    double res = th + fma(th, p, tlo[j]);
    if (e >= -1021) return res * __hiloint2double((e + 1023) << 20, 0);
    return res * __hiloint2double((e + 1623) << 20, 0) * 0x1p-600;
}

// exp(z) for z in [-745, 709] without range branches (callers clamp): the same
// table and polynomial as pexp, so results agree with pexp bit for bit there.
__device__ __forceinline__ double pexp_lean(double z, const double *__restrict__ thi,
                                            const double *__restrict__ tlo) {
    const double kL2E64 = 92.332482616893657;
    const double kLn2Hi = 6.93147180369123816490e-01 * 0.015625;
    const double kLn2Lo = 1.90821492927058770002e-10 * 0.015625;
    const double kShift = 6755399441055744.0;
    double t = fma(z, kL2E64, kShift);
    double kd = t - kShift;
    int k = __double2loint(t);
    double r = fma(-kd, kLn2Hi, z);
    r = fma(-kd, kLn2Lo, r);
    double p = fma(r, 1.0 / 720.0, 1.0 / 120.0);
    p = fma(p, r, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = p * r;
    int j = k & 63;
    int e = k >> 6;
    double th = thi[j];
    double res = th + fma(th, p, tlo[j]);
    // 2^e in two factors (e in [-1075, 1023]): exact, no denormal branch
    const int e1 = e >> 1, e2 = e - e1;
    return res * __hiloint2double((e1 + 1023) << 20, 0) * __hiloint2double((e2 + 1023) << 20, 0);
}

__device__ __forceinline__ void load_exp_table(const ExpTable *__restrict__ g, double *shi,
                                               double *slo) {
    for (int t = threadIdx.x; t < 64; t += blockDim.x) {
        shi[t] = g->hi[t];
        slo[t] = g->lo[t];
    }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ----------------------------------------------------------------- cost
// Cost source shared by all dense passes.  D_ij is the unscaled distance;
// callers fold cost_scale into their exponent weight.
struct CostDesc {
    int kind;          // 0 dense, 1 sqeuclid, 2 L1
    int d;
    const double *C;
    long long ldc;
    const double *x;   // m x d
    const double *y;   // n x d
};

}  // namespace pins
