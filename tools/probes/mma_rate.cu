// Tensor-pipe rate of K8's MMA shapes (tcgen05.mma.kind::tf32, M = 128, K = 8 per instruction):
// chains of NMMA dependent MMAs into one TMEM accumulator, A from TMEM (as K8) or shared memory,
// N = 48 (K8's filters / taps) vs 256, with and without a commit + mbarrier wait after every chain
// (K8 waits once per response row and chain).  CTAS CTAs per SM share the tensor pipe.
// Prints one line per variant: achieved TFLOP/s and cycles per chain.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1404_5344_b200/csrc/tc_ptx.cuh"
using namespace foe::tc;

template <int N, bool TS, bool WAIT, int NMMA>
__global__ void __launch_bounds__(128, 2) mma_chain(int iters, float* out, long long* cyc) {
    extern __shared__ __align__(1024) float sm[];
    float* as = sm;                 // [KT/4][128][4], KT = 8
    float* bs = sm + 128 * 8;       // [KT/4][N][4]
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t mbar;
    const int t = threadIdx.x, warp = t >> 5;
    for (int i = t; i < 128 * 8 + N * 8; i += 128) sm[i] = 1e-3f * (i % 17);
    if (warp == 0) tmem_alloc<256>(&tbase);
    if (t == 0) { mbar_init(&mbar, 1); mbar_fence_init(); }
    fence_proxy_async_smem();
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tb = tbase;
    const uint32_t id = idesc_tf32(128, N);
    const uint32_t ab = smem_u32(as), bb = smem_u32(bs);
    const uint64_t ad = sdesc_kmajor(ab, 128 * 16, 128);
    const uint64_t bd = sdesc_kmajor(bb, N * 16, 128);
    const long long c0 = clock64();
    if (warp == 0) {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < NMMA; ++k) {
                if (TS) mma_tf32_ts_warp(tb, tb + 128 + (k & 7) * 8, bd, id, (uint32_t)(it | k));
                else {
                    asm volatile(
                        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tb),
                        "l"(ad), "l"(bd), "r"(id), "r"((uint32_t)(it | k)));
                }
            }
            if (WAIT) {
                mma_commit_warp(&mbar);
                mbar_wait(&mbar, (uint32_t)(it & 1));
            }
        }
        if (!WAIT) {
            mma_commit_warp(&mbar);
            mbar_wait(&mbar, 0);
        }
    }
    __syncthreads();
    const long long c1 = clock64();
    if (t == 0 && blockIdx.x == 0) *cyc = c1 - c0;
    fence_after_sync();
    float v[8];
    tmem_ld8(tb + ((uint32_t)(warp * 32) << 16), v);
    wait_ld();
    if (v[0] == 12345.678f) out[0] = v[1];
    fence_before_sync();
    __syncthreads();
    if (warp == 0) tmem_dealloc<256>(tb);
}

template <int N, bool TS, bool WAIT, int NMMA>
void run(const char* name, int nsm, int ctas_per_sm, float* out, long long* dcyc) {
    const int smem = (128 * 8 + N * 8) * 4;
    cudaFuncSetAttribute(mma_chain<N, TS, WAIT, NMMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    mma_chain<N, TS, WAIT, NMMA><<<nsm * ctas_per_sm, 128, smem>>>(10, out, dcyc);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(err)); return; }
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        mma_chain<N, TS, WAIT, NMMA><<<nsm * ctas_per_sm, 128, smem>>>(iters, out, dcyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    long long cyc = 0;
    cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
    const double flop = (double)nsm * ctas_per_sm * iters * NMMA * 2.0 * 128 * N * 8;
    printf("%-34s CTAs/SM %d: %7.1f TFLOP/s, %6.0f cycles per chain of %d MMAs (CTA 0)\n", name, ctas_per_sm,
           flop / (best * 1e-3) / 1e12, (double)cyc / iters, NMMA);
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    long long* cyc;
    cudaMalloc(&out, 64);
    cudaMalloc(&cyc, 8);
    run<256, false, false, 8>("SS N=256 continuous", nsm, 1, out, cyc);
    run<48, false, false, 21>("SS N=48 continuous", nsm, 1, out, cyc);
    run<48, true, false, 21>("TS N=48 continuous", nsm, 1, out, cyc);
    run<48, true, true, 21>("TS N=48 chain 21 + wait", nsm, 1, out, cyc);
    run<48, true, true, 21>("TS N=48 chain 21 + wait", nsm, 2, out, cyc);
    run<48, true, true, 18>("TS N=48 chain 18 + wait", nsm, 2, out, cyc);
    run<96, true, true, 21>("TS N=96 chain 21 + wait", nsm, 2, out, cyc);
    run<96, true, false, 21>("TS N=96 continuous", nsm, 1, out, cyc);
    run<128, true, false, 21>("TS N=128 continuous", nsm, 1, out, cyc);
    run<256, true, false, 8>("TS N=256 continuous", nsm, 1, out, cyc);
    return 0;
}
