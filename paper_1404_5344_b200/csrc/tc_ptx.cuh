// tc_ptx.cuh -- thin inline-PTX wrappers for the sm_100a 5th-generation tensor cores
// (tcgen05: TMEM allocation, TMEM <-> register moves, TF32 MMA with A in TMEM and B in
// shared memory, commit to an mbarrier) used by the tensor-core FoE stencil (K8).
//
// Encodings (instruction descriptor, shared-memory matrix descriptor) follow the sm_100
// UMMA formats: idesc bits [4,6) D format (1 = F32), [7,10) A format, [10,13) B format
// (2 = TF32), [15] / [16] A / B major (0 = K-major), [17,23) N >> 3, [24,29) M >> 4.
// Smem descriptor: [0,14) start address >> 4, [16,30) leading-dimension byte offset >> 4,
// [32,46) stride-dimension byte offset >> 4, [46,48) version = 1, [61,64) layout (0 = no
// swizzle).  K-major, no swizzle: 8-row x 16-byte core matrices (128 contiguous bytes);
// LBO = byte distance between the two 16-byte K halves of one MMA (K = 8 tf32), SBO =
// byte distance between 8-row groups along M/N.
#pragma once

#include <cuda_runtime.h>

// 1: round the low part of each 3xTF32 split to tf32 (unbiased); 0: let the tensor core drop its
// low bits (3 fewer FP32x2 operations per value pair)
// 1: the 3xTF32 split of the thread-built operands with integer rounding (hi = (bits + 2^12) &
// ~(2^13 - 1) on the ALU pipe, lo = x - hi): the same round-to-nearest hi as the Veltkamp split
// below, a shorter dependency chain and the FMA pipe left to the arithmetic (K8 1.212 -> 1.185 ms,
// K8 vs K1 unchanged at 2.95e-6); 0: the paired-FP32 Veltkamp split
#ifndef FOE_TF32_SPLIT_INT
#define FOE_TF32_SPLIT_INT 1
#endif
#ifndef FOE_TF32_LO_ROUND
#define FOE_TF32_LO_ROUND 0
#endif
#include <stdint.h>

namespace foe {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- TMEM allocation (one warp; ncols a power of 2 >= 32) -------------------------------
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(dst_smem)),
                 "n"(NCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
}
template <int NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "n"(NCOLS));
}

__device__ __forceinline__ void fence_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// ---- TMEM <-> registers: warp w moves lanes [32w, 32w+32), thread t = lane 32w+t --------
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t* r = reinterpret_cast<uint32_t*>(v);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
    uint32_t* r = reinterpret_cast<uint32_t*>(v);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
    const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

// ---- descriptors -------------------------------------------------------------------------
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4)            // D = F32
           | (2u << 7)          // A = TF32
           | (2u << 10)         // B = TF32
           | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// kind::f16 with fp16 A and B (formats 0), fp32 D
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4)            // D = F32
           | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ uint64_t sdesc_kmajor(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version (sm_100)
    return d;                // base offset 0, layout 0 = no swizzle
}

// ---- MMA: D[tmem] (+)= A[tmem] . B[smem], kind::tf32, one thread issues -------------------
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// D[tmem] (+)= A[smem] . B[smem]
__device__ __forceinline__ void mma_tf32_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// Warp-collective forms: every lane of the warp executes the call with warp-uniform operands
// (so the compiler keeps descriptors in uniform registers) and one elected lane issues.
__device__ __forceinline__ void mma_tf32_ts_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                                 uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// D[tmem] (+)= A[tmem] . B[smem], kind::f16 (fp16 operands packed two per 32-bit TMEM column)
__device__ __forceinline__ void mma_f16_ts_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                                uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit_warp(uint64_t* mbar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(mbar))
        : "memory");
}

// arrive on `mbar` when all previously issued MMAs of this thread have completed
__device__ __forceinline__ void mma_commit(uint64_t* mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(mbar))
                 : "memory");
}

// ---- mbarrier ------------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(mbar)),
        "r"(parity)
        : "memory");
}

// arrive (count 1) on an mbarrier from a thread (release at CTA scope)
// TMA bulk copy (1-D, no tensor map): bytes (multiple of 16, 16-B aligned ends) from global to
// this CTA's shared memory, completing on mbar; the issuing thread first arms mbar with the
// byte count (arrive + expect_tx)
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* mbar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(smem_dst)),
                 "l"(gmem_src), "r"(bytes), "r"(smem_u32(mbar))
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* mbar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(smem_u32(mbar))
                 : "memory");
}
// named barrier among `nthreads` threads of the CTA (id 1..15; 0 is __syncthreads)
__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
// TMEM load of 16 / 32-bit columns without waiting (the caller issues tcgen05.wait::ld once)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t* r = reinterpret_cast<uint32_t*>(v);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_st2u(uint32_t taddr, uint32_t a, uint32_t b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};\n" ::"r"(taddr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void tmem_st4u(uint32_t taddr, const uint32_t (&v)[4]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
                 "r"(v[2]), "r"(v[3])
                 : "memory");
}
__device__ __forceinline__ void tmem_st1(uint32_t taddr, float v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};\n" ::"r"(taddr), "r"(__float_as_uint(v)) : "memory");
}
__device__ __forceinline__ void tmem_ld2(uint32_t taddr, float& a, float& b) {
    uint32_t x, y;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n" : "=r"(x), "=r"(y) : "r"(taddr));
    a = __uint_as_float(x);
    b = __uint_as_float(y);
}

// x rounded to the nearest tf32 (ties away from zero; finite x) with two integer ops.  For the
// 3xTF32 split hi = tf32_hi(x), lo = tf32_hi(x - hi): x - hi is exact in fp32, |x - hi| <=
// 2^-11 |x|, and rounding lo (instead of letting the tensor core drop its low bits) keeps the
// residual error unbiased, <= 2^-22 |x|.
__device__ __forceinline__ float tf32_hi(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// Paired 3xTF32 split of two values (Veltkamp-Dekker with s = 2^13 + 1 on FP32x2 pipes, no
// contraction): hi = x rounded to 11 significant bits (tf32), lo = x - hi rounded likewise.
// 7 paired ops per 2 values instead of 5 integer/fp ops per value.
// the rounded paired product x*s as an FFMA2 with a zero addend: ptxas fuses a separate
// multiply into the following subtraction (FMUL2 + FADD2 -> FFMA2, even for the .rn forms),
// which would break Veltkamp's split; an FMA result is not re-fused
__device__ __forceinline__ float2 fmul2_nocontract(float2 a, float2 b) {
    return __ffma2_rn(a, b, make_float2(0.0f, 0.0f));
}

__device__ __forceinline__ void tf32_split2(float2 x, float2& hi, float2& lo) {
#if FOE_TF32_SPLIT_INT
    // hi = x rounded to tf32 by integer ops (ALU pipe), lo = x - hi exact (left to the TC)
    hi = make_float2(__uint_as_float((__float_as_uint(x.x) + 0x1000u) & 0xFFFFE000u),
                     __uint_as_float((__float_as_uint(x.y) + 0x1000u) & 0xFFFFE000u));
    lo = __fadd2_rn(x, make_float2(-hi.x, -hi.y));
    return;
#endif
    const float2 s = make_float2(8193.0f, 8193.0f);
    const float2 c = fmul2_nocontract(x, s);
    const float2 t = __fadd2_rn(c, make_float2(-x.x, -x.y));
    hi = __fadd2_rn(c, make_float2(-t.x, -t.y));
    const float2 r = __fadd2_rn(x, make_float2(-hi.x, -hi.y));        // exact
#if FOE_TF32_LO_ROUND
    const float2 c2 = fmul2_nocontract(r, s);
    const float2 t2 = __fadd2_rn(c2, make_float2(-r.x, -r.y));
    lo = __fadd2_rn(c2, make_float2(-t2.x, -t2.y));
#else
    lo = r;   // the tensor core keeps lo's top 11 bits: error <= 2^-11 |lo| <= 2^-22 |x|
#endif
}

// fp32 -> tf32 (round to nearest, ties away), kept in a 32-bit container
__device__ __forceinline__ float to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

}  // namespace tc
}  // namespace foe
