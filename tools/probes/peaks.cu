// Peak microbenchmarks for the roofline denominators bench.py reports (the
// measured peaks file has no FP32 figure; the TF32 tensor figure is otherwise derived from bf16):
//   * FP32 FMA: independent FFMA2 chains (paired fp32 FMA, sm_100), 148 x 4 x 8 warps;
//   * TF32 tensor: back-to-back tcgen05.mma.kind::tf32, M = 128, N = 256, K = 8, A and B in
//     shared memory (SS), one elected thread per CTA, one CTA per SM, accumulators in TMEM.
// Prints one JSON line: {"fp32_tflops": ..., "tf32_tflops": ..., "sm_count": ...}.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1404_5344_b200/csrc/tc_ptx.cuh"
using namespace foe::tc;

__global__ void __launch_bounds__(256) ffma_peak(float* out, int iters) {
    float2 a[8], b = make_float2(1.0001f, 0.9999f), c = make_float2(1e-7f, -1e-7f);
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 1e-3f + i, blockIdx.x * 1e-3f - i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], b, c);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
    if (s == 12345.678f) out[0] = s;   // keep the chains alive
}

constexpr int N = 256, KT = 64;   // B: N x KT tf32 (64 KB), A: 128 x KT (32 KB)
__global__ void __launch_bounds__(128, 1) tf32_peak(int iters, float* out) {
    extern __shared__ __align__(1024) float sm[];
    float* as = sm;                  // [KT/4][128][4]
    float* bs = sm + 128 * KT;       // [KT/4][N][4]
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t mbar;
    const int t = threadIdx.x, warp = t >> 5;
    for (int i = t; i < 128 * KT + N * KT; i += 128) sm[i] = 1e-3f * (i % 17);
    if (warp == 0) tmem_alloc<256>(&tbase);
    if (t == 0) { mbar_init(&mbar, 1); mbar_fence_init(); }
    fence_proxy_async_smem();
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t id = idesc_tf32(128, N);
    if (warp == 0) {
        const uint32_t ab = smem_u32(as), bb = smem_u32(bs);
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < KT / 8; ++k) {
                const uint64_t ad = sdesc_kmajor(ab + k * 2 * 128 * 16, 128 * 16, 128);
                const uint64_t bd = sdesc_kmajor(bb + k * 2 * N * 16, N * 16, 128);
                // D[tmem] += A[smem] . B[smem]  (elected lane)
                asm volatile(
                    "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tbase),
                    "l"(ad), "l"(bd), "r"(id), "r"((uint32_t)(it | k)));
            }
        }
        mma_commit_warp(&mbar);
    }
    mbar_wait(&mbar, 0);
    fence_after_sync();
    float v[8];
    tmem_ld8(tbase + ((uint32_t)(warp * 32) << 16), v);
    wait_ld();
    if (v[0] == 12345.678f) out[0] = v[1];
    fence_before_sync();
    __syncthreads();
    if (warp == 0) tmem_dealloc<256>(tbase);
}

int main() {
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    float* out;
    cudaMalloc(&out, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    // FP32: grid = 8 CTAs/SM x 256 threads
    const int fit = 20000;
    ffma_peak<<<nsm * 8, 256>>>(out, 100);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        ffma_peak<<<nsm * 8, 256>>>(out, fit);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double fflop = (double)nsm * 8 * 256 * fit * 16 * 8 * 2 * 2;   // 2 lanes x 2 flop per FFMA2
    const double fp32 = fflop / (best * 1e-3) / 1e12;
    // TF32 tensor
    const int smem = (128 * KT + N * KT) * 4;
    cudaFuncSetAttribute(tf32_peak, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int tit = 4000;
    tf32_peak<<<nsm, 128, smem>>>(10, out);
    cudaError_t err = cudaDeviceSynchronize();
    double tf32 = -1;
    if (err == cudaSuccess) {
        best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            tf32_peak<<<nsm, 128, smem>>>(tit, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        const double tflop = (double)nsm * tit * (KT / 8) * 2.0 * 128 * N * 8;
        tf32 = tflop / (best * 1e-3) / 1e12;
    }
    printf("{\"fp32_tflops\": %.2f, \"tf32_tflops\": %.2f, \"sm_count\": %d, \"error\": \"%s\"}\n", fp32, tf32, nsm,
           cudaGetErrorString(err));
    return 0;
}
