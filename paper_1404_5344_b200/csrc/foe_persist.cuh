// foe_persist.cuh -- the persistent small-image solver of SURVEY.md 8(f) f4: the whole iPiano
// trial loop (PAPER.md:157-166 with the backtracking test of SPEC.md:287) in ONE cooperative
// kernel launch, for problems too small to fill the GPU (configs c1-c3: one 128^2 .. 512^2
// image), where the graph path's per-trial cost is three dependent launches (K2 -> K1 -> K3)
// and their gaps rather than arithmetic.
//
// Per trial round, every CTA of a co-resident grid:
//   phase A  K2 (inertial point + prox + test partials) over the (pixel block, image) items,
//   barrier
//   phase B  K1 (fused prior energy+gradient, paired FFMA) over the (tile x group, image) items,
//   barrier
//   phase C  K3 (decision) of every active image, computed REDUNDANTLY by each CTA on its own
//            copy of the control block: the partials and the fixed-order reductions are the
//            same for all CTAs, so every copy takes the same (bitwise) decision, and the third
//            grid barrier a shared decision would need is not needed.
// The test partials of K2 are double-buffered by round parity: a CTA that has finished phase
// C may start the next round's phase A while a slower CTA still reads this round's partials.
// The K1 energy partials need no second buffer (they are rewritten only after the next
// round's first barrier, which every CTA reaches after its phase C).  Copy 0 of the control
// blocks is the state's ctl (read by the host after the launch); CTA 0 alone writes the trace.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "foe_kernels.cuh"

namespace foe {

struct PersistArgs {
    K1Args a1;           // ctl = copy 0 (replaced per CTA)
    K2Args a2;           // ppart = buffer 0 (buffer 1 at + ppart_stride)
    K3Args a3;
    ImgCtl* ctl;         // [grid][B] per-CTA control copies; copy 0 = the state's
    unsigned int* bar;   // grid barrier counter, zero at launch
    size_t ppart_stride; // doubles between the two test-partial buffers
    int B, max_rounds;
    int k1_items;        // ntiles * groups (per image)
    int k2_items;        // K2 pixel blocks (per image)
    int* rounds_out;     // rounds run (written by CTA 0)
    // diagnostics (nullable): CTA 0's %globaltimer at the phase boundaries of the first
    // kPhaseRounds rounds, [round][4] = {start, after K2 + barrier, after K1 + barrier, after K3}
    unsigned long long* phase_ns;
};
constexpr int kPhaseRounds = 256;

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Sense-free grid barrier on a monotone arrival counter (all CTAs co-resident: cooperative
// launch).  The CTA barrier orders the CTA's writes before thread 0's arrival, a release-ordered
// atomic add at GPU scope publishes them (cumulatively); thread 0 spins with acquire loads, and
// the closing CTA barrier orders every thread's later reads after that acquire.
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int nblocks, unsigned int& gen) {
    __syncthreads();
    gen += 1;
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        // modular target and a wrap-safe comparison: the counter may wrap past 2^32 on long solves
        const unsigned int target = gen * nblocks;
        unsigned int v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        } while ((int)(v - target) < 0);
    }
    __syncthreads();
}

template <int M, int NCP, int SF, int PXT>
__global__ void __launch_bounds__(kThreads, 2)
k_ipiano_persistent(const PersistArgs pa, const __grid_constant__ TapParams2 tp) {
    const unsigned int G = gridDim.x;
    const int cta = blockIdx.x, B = pa.B;
    ImgCtl* my = pa.ctl + (size_t)cta * B;
    if (cta != 0) {   // this CTA's copy of the control blocks (copy 0 is only written after 2 barriers)
        const int words = (int)(sizeof(ImgCtl) / sizeof(long long)) * B;
        const long long* src = reinterpret_cast<const long long*>(pa.ctl);
        long long* dst = reinterpret_cast<long long*>(my);
        for (int i = threadIdx.x; i < words; i += kThreads) dst[i] = src[i];
    }
#if FOE_K2_ETAB && !FOE_K2_ETAB_G
    k2_etab_init();   // the prox's exponential table (phase A)
#endif
    __syncthreads();
    unsigned int gen = 0;
    int round = 0;
    for (; round < pa.max_rounds; ++round) {
        int any = 0;
        for (int b = 0; b < B; ++b) any |= my[b].active;
        __syncthreads();   // every thread has read the flags before phase C rewrites them
        if (!any) break;
        const bool stamp = pa.phase_ns != nullptr && cta == 0 && threadIdx.x == 0 && round < kPhaseRounds;
        if (stamp) pa.phase_ns[4 * round + 0] = global_ns();
        const size_t poff = (size_t)(round & 1) * pa.ppart_stride;
        // phase A: K2
        K2Args a2 = pa.a2;
        a2.ctl = my;
        a2.ppart += poff;
        const int n2 = pa.k2_items * B;
        for (int it = cta; it < n2; it += G) {
            const int b = it / pa.k2_items;
            inertial_prox_blk<PXT>(a2, it - b * pa.k2_items, b);
            __syncthreads();
        }
        grid_barrier(pa.bar, G, gen);
        if (stamp) pa.phase_ns[4 * round + 1] = global_ns();
        // phase B: K1 at the candidate
        K1Args a1 = pa.a1;
        a1.ctl = my;
        const int n1 = pa.k1_items * B;
        for (int it = cta; it < n1; it += G) {
            const int b = it / pa.k1_items;
            prior_grad2_item<M, NCP, SF>(a1, tp, it - b * pa.k1_items, b);
            __syncthreads();
        }
        grid_barrier(pa.bar, G, gen);
        if (stamp) pa.phase_ns[4 * round + 2] = global_ns();
        // phase C: K3, redundantly per CTA
        K3Args a3 = pa.a3;
        a3.ctl = my;
        a3.ppart += poff;
        if (cta != 0) a3.trace = nullptr;
        for (int b = 0; b < B; ++b) {
            decide_img(a3, b);
            __syncthreads();
        }
        if (stamp) pa.phase_ns[4 * round + 3] = global_ns();
    }
    if (cta == 0 && threadIdx.x == 0 && pa.rounds_out != nullptr) *pa.rounds_out = round;
}

}  // namespace foe
