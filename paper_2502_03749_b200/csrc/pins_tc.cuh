// pins_tc.cuh -- 5th-generation tensor-core primitives (tcgen05, sm_100a) for
// the cost cross term x.y of the squared-Euclidean point cost.
//
// D_ij = |x_i|^2 + |y_j|^2 - 2 x_i.y_j is the one dense contraction of the
// path (north star); for integer coordinates |x| <= 2048 the fp16 operands
// are exact, every product (< 2^22) and every partial sum (< 2^24, checked
// on the host) is exact in the fp32 accumulator, so the tensor-core D is
// bit-identical to the SIMT fp32 path.
//
// Layout: A = the CTA's 128 pass rows x K=16 fp16, B = a chunk of N pass
// columns x K=16 fp16, both K-major without swizzle in the canonical UMMA
// "interleave" layout: core matrices of 8 rows x 16 B, the two K halves of
// a row group 128 B apart (LBO), row groups 256 B apart (SBO).  One
// tcgen05.mma (M=128, N, K=16, fp32 accumulate) per chunk writes the N dot
// products of every row into TMEM lane = row; each thread then reads its own
// row with tcgen05.ld.32x32b.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

namespace pins {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// byte offset of element (row, k) (k < 16) in the interleaved K-major tile
__device__ __forceinline__ int kmajor_off(int row, int k) {
    return (row >> 3) * 256 + (k >> 3) * 128 + (row & 7) * 16 + (k & 7) * 2;
}

// shared-memory matrix descriptor: no swizzle, K-major, LBO = 128 B, SBO = 256 B
__device__ __forceinline__ uint64_t make_desc(const void *smem_tile) {
    const uint64_t addr = smem_u32(smem_tile);
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;                 // start address  [0,14)
    d |= (uint64_t)(128 >> 4) << 16;              // leading byte offset [16,30)
    d |= (uint64_t)(256 >> 4) << 32;              // stride byte offset  [32,46)
    d |= (uint64_t)1 << 46;                       // descriptor version (sm_100)
    return d;                                     // base offset 0, lbo mode 0, SWIZZLE_NONE
}

// instruction descriptor: kind::f16, A/B fp16, D fp32, K-major A and B, M = 128
__host__ __device__ constexpr uint32_t make_idesc(int N) {
    return (1u << 4)                              // D format F32
           | (0u << 7) | (0u << 10)               // A, B format F16
           | ((uint32_t)(N >> 3) << 17)           // N >> 3
           | ((uint32_t)(128 >> 4) << 24);        // M >> 4
}

__device__ __forceinline__ void tmem_alloc(uint32_t *smem_dst, int ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(smem_dst)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}
__device__ __forceinline__ void tmem_free(uint32_t taddr, int ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols));
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
// generic-proxy smem writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// D[tmem] = A[smem] * B[smem]^T  (single K=16 step, no accumulation)
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(0));
}

__device__ __forceinline__ void commit(uint64_t *mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     smem_u32(mbar))
                 : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *mbar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t *mbar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(mbar)),
        "r"(phase)
        : "memory");
}

// 32 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = __uint_as_float(r[k]);
}

}  // namespace tc
}  // namespace pins
