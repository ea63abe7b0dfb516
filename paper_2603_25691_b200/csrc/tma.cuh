// tma.cuh — sm_100a bulk-copy (TMA) and mbarrier primitives shared by the streaming kernels.
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace cphifi {
namespace tma {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy, completion counted in bytes on `bar` (16-byte aligned, bytes % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// 2-D tensor-map copy of the box at (c0 = innermost, c1) into shared memory (128-byte aligned)
__device__ __forceinline__ void tensor_g2s_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
// 3-D tensor-map copy of the box at (c0 innermost, c1, c2)
__device__ __forceinline__ void tensor_g2s_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
// L2 prefetch of a 2-D tensor-map box (no shared memory, no completion)
__device__ __forceinline__ void tensor_prefetch_l2_2d(const CUtensorMap* map, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

}  // namespace tma

// host: encode a 2-D fp64 tensor map (column-major matrix rows x cols, leading dimension ld
// elements, box box0 x box1; out-of-bounds elements read as zero).  Returns false when the
// layout violates the TMA constraints (16-byte aligned base and stride).
// swizzle128: CU_TENSOR_MAP_SWIZZLE_128B (box0 * 8 <= 128 bytes; the shared-memory box 1024-byte
// aligned: 16-byte chunk c of box row y lands at chunk c ^ (y mod 8))
bool encode_tmap_2d_f64(CUtensorMap* map, const double* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box0,
                        uint32_t box1, bool swizzle128 = false);
// 3-D fp64 tensor map over a column-major n0 x n1 x n2 array (strides n0, n0 n1), box b0 x b1 x b2
bool encode_tmap_3d_f64(CUtensorMap* map, const double* base, uint64_t n0, uint64_t n1, uint64_t n2, uint32_t b0,
                        uint32_t b1, uint32_t b2);

}  // namespace cphifi
