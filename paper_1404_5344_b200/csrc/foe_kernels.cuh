// foe_kernels.cuh -- sm_100a kernels of the FoE/iPiano despeckling hot path.
//
//   K1  k_prior_grad   fused FoE prior energy + gradient stencil (Eq.(2),
//                      :176-183 grad_w F = W sum_i theta_i K_i^T rho'(K_i e^w)).  FP32 FFMA
//                      register-blocked correlations out of shared memory; taps are
//                      kernel parameters read through the uniform datapath (LDCU + FFMA
//                      with a UR operand).
//   K1h k_prior_hvp    the same stencil for the Hessian-vector product (R-10).
//   K2  k_inertial_prox  w_hat = w - a g + b (w - w_prev) and the
//                      Newton prox of Eq.(10) in fp64, plus the
//                      fixed-order block partials of the backtracking test.
//   K3  k_decide       per-image decision of the descent-lemma test, state rotation,
//                      Lipschitz update and trace (device-side control: no host sync per trial).
//
// Numerics: the iterate w is fp64 in HBM; the stencil computes in
// fp32 on u - c (c = e^w at the tile centre; K(u - c) + c sum(k) = K u exactly), the
// energy accumulates per response in fp32 and per thread/block in fp64, and every
// reduction has a fixed order (no atomics), so results are bitwise reproducible.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace foe {

constexpr int kMaxFilters = 64;
constexpr int kMaxTaps = 3136;
constexpr int kThreads = 256;
#ifndef FOE_K2_UNROLL
#define FOE_K2_UNROLL 2   // K2 pixels in flight per thread
#endif
#ifndef FOE_K2_ETAB
#define FOE_K2_ETAB 1     // K2 fast path: table-driven fp64 exponential (k2_etab in shared memory)
#endif
#ifndef FOE_K2_RCP1
#define FOE_K2_RCP1 1     // K2 fast path: the fp64 Newton step's 1/phi' with one refinement step
#endif
#ifndef FOE_K2_ETAB_G
#define FOE_K2_ETAB_G 1   // ... read from global memory through L1 (no per-CTA shared-memory copy)
#endif
#ifndef FOE_K2_PAIRS
#define FOE_K2_PAIRS 1    // K2 by pixel pairs (inertial_prox_pairs) when HW % 4 == 0
#endif
#ifndef FOE_K2_LOCKSTEP
#define FOE_K2_LOCKSTEP 0 // K2 pairs: both fast-path proxes as one block (k2_pair; measured 153 vs 152 us: off)
#endif
#ifndef FOE_K2_CTAS
#define FOE_K2_CTAS 3     // K2 CTAs per SM (80 registers; pairs: 223 us at 4 CTAs (spills) vs 163 at 3)
#endif
constexpr int kK2Unroll = FOE_K2_UNROLL;
constexpr int kTile = 64;  // output tile side of K1
constexpr int kNumPart = 8;  // K2 block partials
constexpr int kHalo = 6;     // ghost rows per side of a row slab (2C for m <= 7)
constexpr int kBandRows = 64; // rows per band of the slab-invariant partial reduction (= kTile)

// Filter taps, resident in the kernel-parameter constant bank.
struct TapParams {
    float fwd[kMaxTaps];           // flipped taps: K_i u is a correlation with k_i[m-1-a][m-1-b]
    float bwd[kMaxTaps];           // 2 theta_i k_i[a][b]: K_i^T is a correlation with k_i (x2 of rho')
    float sumk[kMaxFilters];       // sum_ab k_i[a][b] (fp64-summed), restores the DC shift
    double theta_ln2[kMaxFilters]; // theta_i * ln 2 (energy accumulates log2)
};

// Per-image iPiano control block (device resident; written only by K3 / host setup).
struct ImgCtl {
    double L;        // current Lipschitz estimate L_n
    double F;        // F(w^n)
    double lam1, lam2;
    int n;           // accepted iterations
    int trials;      // failed trials so far in the current iteration
    int total_trials;
    int status;      // foe_status of this image
    int cur, prev, cand;  // w slots
    int gcur, gcand;      // gradient slots
    int active;      // take part in the next trial round
    int done;        // stopped by rel_change_tol
    int target;      // iterations to reach
    int pad;
};

struct SolverParams {
    double beta, safety, eta, shrink, newton_tol, rel_tol, w_guard;
    int max_backtracks, newton_cap, record_trace, max_iters;
};

struct K1Args {
    const double* w;        // [slots][B][H][W] (or one image set when ctl == nullptr)
    size_t w_slot_stride;
    float* g;               // [slots][groups][B][H][W]
    size_t g_slot_stride;
    size_t g_group_stride;
    double* epart;          // [B][tiles*groups] energy partials
    const ImgCtl* ctl;      // nullable
    int which_cur;          // 1: evaluate at ctl.cur -> ctl.gcur; 0: ctl.cand -> ctl.gcand
    int H, W, tiles_x, ntiles, groups, nf, nchunks;
    // Row slab: rows y < 0 come from halo row kHalo + y, rows y >= H from
    // halo row kHalo + (y - H) ([2][kHalo][W] fp64, filled by the halo exchange); nullptr =
    // periodic wrap inside the image (single-GPU scene).
    const double* halo;
    // Data model of the iterate: 0 = w-domain (models (8)/(10): u = e^w, grad_w F = u (.) s),
    // 1 = u-domain (model (6): the iterate is u, grad_u F = s)
    int udom;
    // K8 column packing (0 = none): each 64-row band has tiles_x full tiles of 128 - 2C output
    // columns; the last tc_rem columns of tc_spt consecutive bands share one tile (strips of
    // tc_rem + 4C lanes), instead of one mostly idle tile per band
    int tc_rem, tc_spt;
    int tc_rows;            // K8: output rows per tile (64 / 32 / 16 / 8)
    // K8 launch over a tile range (row slabs: interior bands before the ghost-row exchange, the
    // two boundary bands after it): tile = tile_off + blockIdx.x; energy partials by tile index
    int tile_off;
    int ncp;                // K1 v2: filter pairs per shared-memory chunk (1 or 2; 0 = 2)
    // K8 without row halos (foe_th.cuh, NH): a tile computes the responses of its own R rows only;
    // an output row within C of a band start takes contributions from two bands -- the band below
    // writes its share into g, the band above its share into gedge [slots][B][nb][2C][W] (boundary
    // t = the lower band, row k = y + C - t R) -- and the second of the two tiles to finish adds
    // them (a per-boundary arrival counter in tcnt [B][nb][tiles_x + 1], left at 0)
    float* gedge;
    size_t gedge_slot_stride;
    unsigned int* tcnt;
    // ... and without column halos either (W % 128 == 0, 128-column tiles): the pieces of the
    // rows near band edges x the columns near tile edges -- gright [slots][B][ns][H][2C] (column
    // boundary s = the right tile), gcorner [slots][B][nb][ns][2C][2C]; counters [3][B][nb][ns + 1]
    float* gright;
    float* gcorner;
    size_t gright_slot_stride, gcorner_slot_stride;
    // HVP only
    float* sbuf;            // [B][NP][H][W] S_i = rho''(K_i u)/2 (k_hvp_th writes it when set, k_hvp_s reads)
    const double* v;        // [B][H][W]
    const float* gw;        // [B][H][W] gradient at w
};

// raw MUFU approximations (argument d = 1 + r^2 >= 1: no denormal/range guards needed)
__device__ __forceinline__ float lg2_approx(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Programmatic dependent launch (graph trial rounds K2 -> K8 -> K3): a kernel launched with the
// programmatic-serialization attribute may start while its predecessor drains; pdl_wait() blocks
// until the predecessor grid has completed and its memory is visible (a no-op for a normal launch),
// pdl_trigger() lets the successor be scheduled once every CTA has triggered or exited.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ int wrap_idx(int i, int n) {
    int r = i % n;
    return r < 0 ? r + n : r;
}

// ---------------------------------------------------------------------------------
// Geometry of K1 for an m x m bank.
// ---------------------------------------------------------------------------------
template <int M, int NC, int SF>
struct K1Geom {
    static constexpr int C = (M - 1) / 2;
    static constexpr int CW = 4;                                  // columns per thread item
    static constexpr int RX = ((kTile + 2 * C + 3) / 4) * 4;      // response cols computed
    static constexpr int NSTRIP_F = RX / CW;
    static constexpr int RY = ((kTile + 2 * C + SF - 1) / SF) * SF;  // response rows computed
    static constexpr int NSEG_F = RY / SF;
    static constexpr int ITEMS_F = NSTRIP_F * NSEG_F;             // forward items per filter
    static constexpr int NV = (CW + M - 1 + 3) / 4;               // float4 per row read
    static constexpr int UY = RY + M - 1;                         // staged rows
    static constexpr int UX = RX + M - 1;                         // staged cols used
    static constexpr int UP0 = ((RX - CW + 4 * NV) > UX ? (RX - CW + 4 * NV) : UX);
    static constexpr int UP1 = ((UP0 + 3) / 4) * 4;
    static constexpr int UP = ((UP1 * SF) % 32 == 0) ? UP1 + 4 : UP1;  // staged pitch
    static constexpr int SB = 4;                                  // backward rows per item
    static constexpr int PP0 = ((kTile - CW + 4 * NV) > RX ? (kTile - CW + 4 * NV) : RX);
    static constexpr int PP = ((PP0 + 3) / 4) * 4;                // rho' pitch
    static constexpr int WPF = (kThreads / 32) / NC;              // warps per filter (forward)
    static_assert(WPF * NC == kThreads / 32, "NC must divide the warp count");
    static constexpr int SMEM_FLOATS = UY * UP + NC * RY * PP;
    static constexpr int SMEM_FLOATS_HVP = 2 * UY * UP + NC * RY * PP;
};

// out[o][x] += sum_{a,b} taps[a*M+b] * in[(o+a)*pitch + x + b],  o < S, x < 4.
// `in` is 16-byte aligned; taps are warp-uniform (constant bank, UR operand).
template <int M, int S, int NV>
__device__ __forceinline__ void corr_block(const float* __restrict__ in, int pitch,
                                           const float* __restrict__ taps, float (&acc)[S][4]) {
#pragma unroll
    for (int i = 0; i < S + M - 1; ++i) {
        float row[4 * NV];
        const float4* rp = reinterpret_cast<const float4*>(in + i * pitch);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const float4 t = rp[v];
            row[4 * v + 0] = t.x; row[4 * v + 1] = t.y; row[4 * v + 2] = t.z; row[4 * v + 3] = t.w;
        }
#pragma unroll
        for (int a = 0; a < M; ++a) {
            const int o = i - a;
            if (o >= 0 && o < S) {
#pragma unroll
                for (int b = 0; b < M; ++b) {
                    const float t = taps[a * M + b];
#pragma unroll
                    for (int x = 0; x < 4; ++x) acc[o][x] = fmaf(t, row[x + b], acc[o][x]);
                }
            }
        }
    }
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Fixed-order block sum (all threads get the result).  `red` holds >= 32 doubles.
__device__ __forceinline__ double block_sum_d(double v, double* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum_d(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < nw; ++i) t += red[i];
    return t;
}
__device__ __forceinline__ double block_max_d(double v, double* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_max_d(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double t = red[0];
    for (int i = 1; i < nw; ++i) t = fmax(t, red[i]);
    return t;
}

// ---------------------------------------------------------------------------------
// K1: fused prior energy + gradient.  One CTA = one 64x64 output tile x one filter group.
// ---------------------------------------------------------------------------------
template <int M, int NC, int SF, bool HVP>
__global__ void __launch_bounds__(kThreads, 2)
k_prior_grad(const K1Args args, const __grid_constant__ TapParams tp) {
    using G = K1Geom<M, NC, SF>;
    constexpr int C = G::C;
    extern __shared__ float4 smem4[];
    float* us = reinterpret_cast<float*>(smem4);           // [UY][UP]  u - c
    float* uvs = us + G::UY * G::UP;                        // [UY][UP]  u * v (HVP only)
    float* ps = us + (HVP ? 2 : 1) * G::UY * G::UP;         // [NC][RY][PP] rho' (or rho'' t)
    __shared__ double red[32];

    const int b = blockIdx.y, bx = blockIdx.x;
    int wslot = 0, gslot = 0;
    if (args.ctl != nullptr) {
        const ImgCtl& c = args.ctl[b];
        if (!c.active) return;
        wslot = args.which_cur ? c.cur : c.cand;
        gslot = args.which_cur ? c.gcur : c.gcand;
    }
    const int H = args.H, W = args.W;
    const size_t HW = (size_t)H * W;
    const int tile = bx / args.groups, grp = bx - tile * args.groups;
    const int ty = tile / args.tiles_x, tx = tile - ty * args.tiles_x;
    const int y0 = ty * kTile, x0 = tx * kTile;
    const double* w = args.w + (size_t)wslot * args.w_slot_stride + (size_t)b * HW;
    const double* vv = HVP ? args.v + (size_t)b * HW : nullptr;
    const int ck0 = (grp * args.nchunks) / args.groups;
    const int ck1 = ((grp + 1) * args.nchunks) / args.groups;

    // (a2) stage u - c on the tile + 2C halo, with c = e^w at the tile centre (fp64 exp).
    const int yc = wrap_idx(y0 + kTile / 2, H), xc = wrap_idx(x0 + kTile / 2, W);
    const bool udom = args.udom != 0;
    const float cst = (float)(udom ? w[(size_t)yc * W + xc] : exp(w[(size_t)yc * W + xc]));
    const double cstd = (double)cst;
    for (int idx = threadIdx.x; idx < G::UY * G::UX; idx += kThreads) {
        const int uy = idx / G::UX, ux = idx - uy * G::UX;
        const int gy = wrap_idx(y0 - 2 * C + uy, H), gx = wrap_idx(x0 - 2 * C + ux, W);
        const size_t gi = (size_t)gy * W + gx;
        const double u = udom ? w[gi] : exp(w[gi]);
        us[uy * G::UP + ux] = (float)(u - cstd);
        // HVP in w: u (.) v is the direction of u; in u the direction is v itself
        if (HVP) uvs[uy * G::UP + ux] = (float)(udom ? vv[gi] : u * vv[gi]);
    }
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fj = warp / G::WPF;                               // filter slot of this warp
    const int flane = (warp - fj * G::WPF) * 32 + lane;        // lane within the filter group
    const int bstrip = threadIdx.x & 15, bseg = threadIdx.x >> 4;
    float acc[G::SB][4];
#pragma unroll
    for (int o = 0; o < G::SB; ++o)
#pragma unroll
        for (int x = 0; x < 4; ++x) acc[o][x] = 0.f;
    double e_acc = 0.0;

    for (int ck = ck0; ck < ck1; ++ck) {
        const int fbase = ck * NC;
        const int nc = min(NC, args.nf - fbase);
        // (a3, a4, a7) forward responses, rho, rho' of this warp's filter
        const int j = __shfl_sync(0xffffffffu, fj, 0);
        if (j < nc) {
            const int fi = fbase + j;
            const float* tf = &tp.fwd[fi * M * M];
            const float cs = cst * tp.sumk[fi];
            float el = 0.f;
            for (int it = flane; it < G::ITEMS_F; it += 32 * G::WPF) {
                const int seg = it / G::NSTRIP_F, strip = it - seg * G::NSTRIP_F;
                float r[SF][4];
#pragma unroll
                for (int o = 0; o < SF; ++o)
#pragma unroll
                    for (int x = 0; x < 4; ++x) r[o][x] = 0.f;
                corr_block<M, SF, G::NV>(us + seg * SF * G::UP + strip * 4, G::UP, tf, r);
                float* pdst = ps + j * G::RY * G::PP + seg * SF * G::PP + strip * 4;
                if (!HVP) {
                    // owned responses: tile rows/cols [0,64) inside the image (energy only)
                    bool colok[4];
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        const int tcx = strip * 4 + x - C;
                        colok[x] = tcx >= 0 && tcx < kTile && x0 + tcx < W;
                    }
#pragma unroll
                    for (int o = 0; o < SF; ++o) {
                        const int tcy = seg * SF + o - C;
                        const bool rowok = tcy >= 0 && tcy < kTile && y0 + tcy < H;
                        float4 q;
                        float* qp = reinterpret_cast<float*>(&q);
#pragma unroll
                        for (int x = 0; x < 4; ++x) {
                            const float rv = r[o][x] + cs;
                            const float d = fmaf(rv, rv, 1.f);
                            const float lg = __log2f(d);
                            el += (rowok && colok[x]) ? lg : 0.f;
                            qp[x] = __fdividef(rv, d);        // rho'(r)/2; the 2 is in bwd taps
                        }
                        *reinterpret_cast<float4*>(pdst + o * G::PP) = q;
                    }
                } else {
                    float t[SF][4];
#pragma unroll
                    for (int o = 0; o < SF; ++o)
#pragma unroll
                        for (int x = 0; x < 4; ++x) t[o][x] = 0.f;
                    corr_block<M, SF, G::NV>(uvs + seg * SF * G::UP + strip * 4, G::UP, tf, t);
#pragma unroll
                    for (int o = 0; o < SF; ++o) {
                        float4 q;
                        float* qp = reinterpret_cast<float*>(&q);
#pragma unroll
                        for (int x = 0; x < 4; ++x) {
                            const float rv = r[o][x] + cs;
                            const float r2 = rv * rv;
                            const float d = 1.f + r2;
                            qp[x] = __fdividef((1.f - r2) * t[o][x], d * d);  // rho''(r) t / 2
                        }
                        *reinterpret_cast<float4*>(pdst + o * G::PP) = q;
                    }
                }
            }
            if (!HVP) e_acc += tp.theta_ln2[fi] * (double)el;
        }
        __syncthreads();
        // (a5) transposed correlations, summed over the chunk's filters
        for (int jj = 0; jj < nc; ++jj) {
            corr_block<M, G::SB, G::NV>(ps + jj * G::RY * G::PP + bseg * G::SB * G::PP + bstrip * 4,
                                        G::PP, &tp.bwd[(fbase + jj) * M * M], acc);
        }
        __syncthreads();
    }

    // (a6) chain rule g = u (.) s and store (owned pixels only)
    float* gout = args.g + (size_t)gslot * args.g_slot_stride + (size_t)grp * args.g_group_stride +
                  (size_t)b * HW;
#pragma unroll
    for (int o = 0; o < G::SB; ++o) {
        const int oy = bseg * G::SB + o;
        const int gy = y0 + oy;
        if (gy >= H) continue;
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            const int ox = bstrip * 4 + x;
            const int gx = x0 + ox;
            if (gx >= W) continue;
            const float u = us[(oy + 2 * C) * G::UP + ox + 2 * C] + cst;
            float val;
            if (!HVP) {
                val = udom ? acc[o][x] : u * acc[o][x];
            } else if (udom) {
                val = acc[o][x];                  // Hess F(u) v = sum theta K^T [rho'' (.) K v]
            } else {
                const size_t gi = (size_t)gy * W + gx;
                val = (float)(vv[gi] * (double)args.gw[(size_t)b * HW + gi] + (double)(u * acc[o][x]));
            }
            gout[(size_t)gy * W + gx] = val;
        }
    }
    if (!HVP) {
        const double e = block_sum_d(e_acc, red);
        if (threadIdx.x == 0) args.epart[(size_t)b * args.ntiles * args.groups + blockIdx.x] = e;
    }
}

// ---------------------------------------------------------------------------------
// K1 v2: the same fused stencil with filters processed in PAIRS so that every FMA
// instruction is a paired fp32 FMA (FFMA2, sm_100): forward  r_(A,B) += u * (kA, kB)
// (the input pixel is broadcast to both lanes of the pair), backward
// s_(A,B) += (rho'_A, rho'_B) * (2 theta_A kA, 2 theta_B kB) with rho' of the pair stored
// interleaved (float2) in shared memory.  This halves the FMA issue slots of v1, which
// ncu showed issue-bound (82% issue active, FMA pipe 68%).
// ---------------------------------------------------------------------------------
constexpr int kMaxPairs = kMaxFilters / 2;

struct TapParams2 {
    float2 fwd[kMaxPairs * 49];    // (kA, kB) flipped taps of pair p (m <= 7)
    float2 bwd[kMaxPairs * 49];    // (2 theta_A kA, 2 theta_B kB)
    float sumk[kMaxFilters];       // sum_ab k_i (restores the DC shift), pair order (A,B) = (2p, 2p+1)
    double theta_ln2[kMaxFilters];
};

// smallest pitch >= lo (multiple of 4 floats) with pitch*sf = 8 (mod 32): the two row
// segments a forward quarter-warp may straddle then hit disjoint banks
__host__ __device__ constexpr int pick_pitch_safe(int lo, int sf) {
    int p = lo;
    for (int k = 0; k < 8; ++k, p += 4)
        if ((p * sf) % 32 == 8) return p;
    return lo;
}

template <int M, int NCP, int SF>
struct G2 {
    static constexpr int C = (M - 1) / 2;
    static constexpr int RX = ((kTile + 2 * C + 3) / 4) * 4;          // response cols
    static constexpr int NSTRIP = RX / 4;
    static constexpr int RY = ((kTile + 2 * C + SF - 1) / SF) * SF;   // response rows
    static constexpr int NSEG = RY / SF;
    static constexpr int ITEMS = NSTRIP * NSEG;                        // forward items per pair
    static constexpr int NVF = (4 + M - 1 + 3) / 4;                    // float4 per forward row
    static constexpr int UY = RY + M - 1;
    static constexpr int UX = RX + M - 1;
    static constexpr int UPMIN0 = (RX - 4 + 4 * NVF) > UX ? (RX - 4 + 4 * NVF) : UX;
    static constexpr int UPMIN = ((UPMIN0 + 3) / 4) * 4;
    static constexpr int UP = pick_pitch_safe(UPMIN, SF);
    static constexpr int SB = 8, CWB = 2;                               // backward thread tile 8x2
    static constexpr int NBSTRIP = kTile / CWB, NBSEG = kTile / SB;
    static_assert(NBSTRIP * NBSEG == kThreads, "backward tiling must use every thread once");
    static constexpr int NVB = (CWB + M - 1 + 1) / 2;                  // float4 (= 2 float2) per bwd row
    static constexpr int PP0 = (kTile - CWB + 2 * NVB) > RX ? (kTile - CWB + 2 * NVB) : RX;
    static constexpr int PP = PP0;                                     // rho' pitch in float2
    static constexpr int SMEM_BYTES = UY * UP * 4 + NCP * RY * PP * 8;
};

// acc[o][x] += (u[(o+a)][x+b] - sub) * (kA, kB)[a][b]   (FFMA2 with a broadcast scalar; `sub`
// is the item's own DC shift, restored by the caller as sub * sum k)
template <int M, int S, int NV>
__device__ __forceinline__ void corr_fwd2(const float* __restrict__ in, int pitch, float sub,
                                          const float2* __restrict__ taps, float2 (&acc)[S][4]) {
#pragma unroll
    for (int i = 0; i < S + M - 1; ++i) {
        float row[4 * NV];
        const float4* rp = reinterpret_cast<const float4*>(in + i * pitch);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const float4 t = rp[v];
            const float2 lo = __fadd2_rn(make_float2(t.x, t.y), make_float2(-sub, -sub));
            const float2 hi = __fadd2_rn(make_float2(t.z, t.w), make_float2(-sub, -sub));
            row[4 * v + 0] = lo.x; row[4 * v + 1] = lo.y; row[4 * v + 2] = hi.x; row[4 * v + 3] = hi.y;
        }
#pragma unroll
        for (int a = 0; a < M; ++a) {
            const int o = i - a;
            if (o >= 0 && o < S) {
#pragma unroll
                for (int b = 0; b < M; ++b) {
                    const float2 t = taps[a * M + b];
#pragma unroll
                    for (int x = 0; x < 4; ++x)
                        acc[o][x] = __ffma2_rn(make_float2(row[x + b], row[x + b]), t, acc[o][x]);
                }
            }
        }
    }
}

// acc[o][x] += (pA, pB)[(o+a)][x+b] * (tA, tB)[a][b]   (FFMA2 on interleaved pairs)
template <int M, int S, int NV>
__device__ __forceinline__ void corr_bwd2(const float2* __restrict__ in, int pitch2,
                                          const float2* __restrict__ taps, float2 (&acc)[S][2]) {
#pragma unroll
    for (int i = 0; i < S + M - 1; ++i) {
        float2 row[2 * NV];
        const float4* rp = reinterpret_cast<const float4*>(in + i * pitch2);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const float4 t = rp[v];
            row[2 * v + 0] = make_float2(t.x, t.y);
            row[2 * v + 1] = make_float2(t.z, t.w);
        }
#pragma unroll
        for (int a = 0; a < M; ++a) {
            const int o = i - a;
            if (o >= 0 && o < S) {
#pragma unroll
                for (int b = 0; b < M; ++b) {
                    const float2 t = taps[a * M + b];
#pragma unroll
                    for (int x = 0; x < 2; ++x) acc[o][x] = __ffma2_rn(row[x + b], t, acc[o][x]);
                }
            }
        }
    }
}

// one (tile x filter group, image) work item: bx = tile * groups + group, b = image (the
// persistent solver runs several per CTA; the caller syncs the CTA between items)
template <int M, int NCP, int SF>
__device__ __forceinline__ void prior_grad2_item(const K1Args& args, const TapParams2& tp, const int bx, const int b) {
    using G = G2<M, NCP, SF>;
    constexpr int C = G::C;
    extern __shared__ float4 smem4[];
    float* us = reinterpret_cast<float*>(smem4);                          // [UY][UP]  u - c
    float2* ps = reinterpret_cast<float2*>(us + G::UY * G::UP);          // [NCP][RY][PP] (rho'_A, rho'_B)/2
    __shared__ double red[32];

    int wslot = 0, gslot = 0;
    if (args.ctl != nullptr) {
        const ImgCtl& c = args.ctl[b];
        if (!c.active) return;
        wslot = args.which_cur ? c.cur : c.cand;
        gslot = args.which_cur ? c.gcur : c.gcand;
    }
    const int H = args.H, W = args.W;
    const size_t HW = (size_t)H * W;
    const int tile = bx / args.groups, grp = bx - tile * args.groups;
    const int ty = tile / args.tiles_x, tx = tile - ty * args.tiles_x;
    const int y0 = ty * kTile, x0 = tx * kTile;
    const double* w = args.w + (size_t)wslot * args.w_slot_stride + (size_t)b * HW;
    const int npairs = (args.nf + 1) / 2;
    const int ck0 = (grp * args.nchunks) / args.groups;
    const int ck1 = ((grp + 1) * args.nchunks) / args.groups;

    // (a2) stage u - c on the tile + 2C halo (fp64 exp, one rounding to fp32); c = e^w at a
    // pixel inside the tile (so a row slab and the whole scene use the same c)
    const int yc = min(y0 + kTile / 2, H - 1), xc = min(x0 + kTile / 2, W - 1);
    const bool udom = args.udom != 0;
    const float cst = (float)(udom ? w[(size_t)yc * W + xc] : exp(w[(size_t)yc * W + xc]));
    const double cstd = (double)cst;
    const double* halo = args.halo;
    // batches of SB independent loads per thread before their exponentials, so that a CTA
    // alone on its SM (small images, the persistent driver) does not wait one memory latency
    // per staged pixel
    constexpr int NST = G::UY * G::UX, SBAT = 8;
    for (int i0 = threadIdx.x; i0 < NST; i0 += SBAT * kThreads) {
        double v[SBAT];
#pragma unroll
        for (int j = 0; j < SBAT; ++j) {
            const int idx = i0 + j * kThreads;
            if (idx < NST) {
                const int uy = idx / G::UX, ux = idx - uy * G::UX;
                const int y = y0 - 2 * C + uy, gx = wrap_idx(x0 - 2 * C + ux, W);
                const double* src;
                if (halo == nullptr) src = w + (size_t)wrap_idx(y, H) * W;
                else if (y < 0) src = halo + (size_t)(kHalo + y) * W;
                else if (y >= H) src = halo + (size_t)(kHalo + y - H) * W;
                else src = w + (size_t)y * W;
                v[j] = src[gx];
            }
        }
#pragma unroll
        for (int j = 0; j < SBAT; ++j) {
            const int idx = i0 + j * kThreads;
            if (idx < NST) {
                const int uy = idx / G::UX, ux = idx - uy * G::UX;
                us[uy * G::UP + ux] = (float)((udom ? v[j] : exp(v[j])) - cstd);
            }
        }
    }
    __syncthreads();

    // fixed forward item of this thread (one per filter pair) and its energy weights
    const int tid = threadIdx.x;
    const bool fwd_on = tid < G::ITEMS;
    const int fseg = tid / G::NSTRIP, fstrip = tid - fseg * G::NSTRIP;
    static_assert(SF * 4 <= 32, "ownership mask is 32 bits");
    unsigned own = 0u;   // bit o*4+x: response (o,x) of this item is owned by the tile (energy)
#pragma unroll
    for (int o = 0; o < SF; ++o) {
        const int tcy = fseg * SF + o - C;
        const bool rok = tcy >= 0 && tcy < kTile && y0 + tcy < H;
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            const int tcx = fstrip * 4 + x - C;
            if (rok && tcx >= 0 && tcx < kTile && x0 + tcx < W) own |= 1u << (o * 4 + x);
        }
    }
    // the item's own DC shift: u at the centre of its response block (second-level shift on
    // top of the tile's c; local differences keep the FFMA accumulation accurate on rough images)
    const float isub = fwd_on ? us[(fseg * SF + SF / 2 + C) * G::UP + fstrip * 4 + 2 + C] : 0.f;
    const float icst = cst + isub;
    const int bstrip = tid % G::NBSTRIP, bseg = tid / G::NBSTRIP;
    float2 bacc[G::SB][G::CWB];
#pragma unroll
    for (int o = 0; o < G::SB; ++o)
#pragma unroll
        for (int x = 0; x < G::CWB; ++x) bacc[o][x] = make_float2(0.f, 0.f);
    double e_acc = 0.0;

    for (int ck = ck0; ck < ck1; ++ck) {
        const int pbase = ck * NCP;
        const int ncp = min(NCP, npairs - pbase);
        // (a3, a4, a7) forward responses of each pair, rho for the energy, rho' to smem
        for (int p = 0; p < ncp; ++p) {
            const int pi = pbase + p;
            if (fwd_on) {
                // r = (c + isub) sum(k) + K(u - c - isub): the DC restore is the accumulator's
                // initial value
                const float2 cs = make_float2(icst * tp.sumk[2 * pi], icst * tp.sumk[2 * pi + 1]);
                float2 r[SF][4];
#pragma unroll
                for (int o = 0; o < SF; ++o)
#pragma unroll
                    for (int x = 0; x < 4; ++x) r[o][x] = cs;
                corr_fwd2<M, SF, G::NVF>(us + fseg * SF * G::UP + fstrip * 4, G::UP, isub, &tp.fwd[pi * M * M], r);
                float2 el = make_float2(0.f, 0.f);
                float2* pdst = ps + (size_t)p * G::RY * G::PP + (size_t)(fseg * SF) * G::PP + fstrip * 4;
#pragma unroll
                for (int o = 0; o < SF; ++o) {
                    float2 q[4];
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        const float2 rv = r[o][x];
                        const float2 d = __ffma2_rn(rv, rv, make_float2(1.f, 1.f));
                        const float2 lg = make_float2(lg2_approx(d.x), lg2_approx(d.y));
                        if (own & (1u << (o * 4 + x))) el = __fadd2_rn(el, lg);   // owned responses only
                        q[x] = __fmul2_rn(rv, make_float2(rcp_approx(d.x), rcp_approx(d.y)));
                    }
                    float4* dst = reinterpret_cast<float4*>(pdst + o * G::PP);
                    dst[0] = make_float4(q[0].x, q[0].y, q[1].x, q[1].y);
                    dst[1] = make_float4(q[2].x, q[2].y, q[3].x, q[3].y);
                }
                e_acc += tp.theta_ln2[2 * pi] * (double)el.x + tp.theta_ln2[2 * pi + 1] * (double)el.y;
            }
        }
        __syncthreads();
        // (a5) transposed correlations of the chunk's pairs, summed in registers
        for (int p = 0; p < ncp; ++p) {
            corr_bwd2<M, G::SB, G::NVB>(ps + (size_t)p * G::RY * G::PP + (size_t)(bseg * G::SB) * G::PP + bstrip * G::CWB,
                                        G::PP, &tp.bwd[(pbase + p) * M * M], bacc);
        }
        __syncthreads();
    }

    // (a6) g = u (.) (s_A + s_B) on owned pixels
    float* gout = args.g + (size_t)gslot * args.g_slot_stride + (size_t)grp * args.g_group_stride +
                  (size_t)b * HW;
#pragma unroll
    for (int o = 0; o < G::SB; ++o) {
        const int oy = bseg * G::SB + o;
        const int gy = y0 + oy;
        if (gy >= H) continue;
#pragma unroll
        for (int x = 0; x < G::CWB; ++x) {
            const int ox = bstrip * G::CWB + x;
            const int gx = x0 + ox;
            if (gx >= W) continue;
            const float u = udom ? 1.0f : us[(oy + 2 * C) * G::UP + ox + 2 * C] + cst;   // W = diag(e^w)
            gout[(size_t)gy * W + gx] = u * (bacc[o][x].x + bacc[o][x].y);
        }
    }
    const double e = block_sum_d(e_acc, red);
    if (threadIdx.x == 0) args.epart[(size_t)b * args.ntiles * args.groups + bx] = e;
}

template <int M, int NCP, int SF>
__global__ void __launch_bounds__(kThreads, 2)
k_prior_grad2(const K1Args args, const __grid_constant__ TapParams2 tp) {
    prior_grad2_item<M, NCP, SF>(args, tp, blockIdx.x, blockIdx.y);
}

// ---------------------------------------------------------------------------------
// K2: inertial forward point + Newton prox of Eq.(10) + block partials of the test.
// ---------------------------------------------------------------------------------

// e^x for |x| <= 1/16: Taylor polynomial of degree 10 (remainder < 1e-20 relative)
__device__ __forceinline__ double exp_small(double x) {
    double p = 2.7557319223985893e-07;            // 1/10!
    p = fma(p, x, 2.7557319223985888e-06);        // 1/9!
    p = fma(p, x, 2.4801587301587302e-05);        // 1/8!
    p = fma(p, x, 1.9841269841269841e-04);        // 1/7!
    p = fma(p, x, 1.3888888888888889e-03);        // 1/6!
    p = fma(p, x, 8.3333333333333332e-03);        // 1/5!
    p = fma(p, x, 4.1666666666666664e-02);        // 1/4!
    p = fma(p, x, 1.6666666666666666e-01);        // 1/3!
    p = fma(p, x, 0.5);
    p = fma(p, x, 1.0);
    return fma(p, x, 1.0);
}
__device__ __forceinline__ double exp_near0(double x) { return fabs(x) <= 0.0625 ? exp_small(x) : exp(x); }

// Taylor coefficients 1/k! of the cosh / sinh parts, in the constant bank (fp64 FMAs take them
// as c[] operands; as immediates every use cost two uniform moves)
__constant__ double kCoshC[9] = {4.7794773323873853e-14, 1.1470745597729725e-11, 2.0876756987868100e-09,
                                 2.7557319223985891e-07, 2.4801587301587302e-05, 1.3888888888888889e-03,
                                 4.1666666666666664e-02, 0.5, 1.0};   // 1/16!, 1/14!, ..., 1/2!, 1
__constant__ double kSinhC[8] = {7.6471637318198164e-13, 1.6059043836821613e-10, 2.5052108385441720e-08,
                                 2.7557319223985893e-06, 1.9841269841269841e-04, 8.3333333333333332e-03,
                                 1.6666666666666666e-01, 1.0};        // 1/15!, 1/13!, ..., 1/3!, 1

// e^{x} and e^{-x} together for |x| <= 1/16: even and odd Taylor parts C = cosh x, S = sinh x
// (terms to x^10, remainder < 1e-20 relative), e^{+-x} = C +- S -- half the work of two exp_small
__device__ __forceinline__ void exp_pm_small(double x, double& ep, double& em) {
    const double x2 = x * x;
    double c = kCoshC[3];                          // 1/10!
#pragma unroll
    for (int i = 4; i < 9; ++i) c = fma(c, x2, kCoshC[i]);
    double sh = kSinhC[3];                         // 1/9!
#pragma unroll
    for (int i = 4; i < 8; ++i) sh = fma(sh, x2, kSinhC[i]);
    sh *= x;
    ep = c + sh;
    em = c - sh;
}

// e^{2a} and e^{-2a} from one range reduction (|2a| <= 700): 2a = n ln2 + r, |r| <= ln2/2;
// cosh/sinh Taylor parts of r to r^16 (remainder < 1e-19 relative), scaled by 2^{+-n}
__device__ __forceinline__ void exp2a_pm(double a, double& ep, double& em) {
    const double x = 2.0 * a;
    const double n = rint(x * 1.4426950408889634);                   // x / ln 2
    const double r = fma(-n, 2.3190468138462996e-17, fma(-n, 6.9314718055994529e-01, x));   // x - n ln2
    const double r2 = r * r;
    double c = kCoshC[0];                          // 1/16!
#pragma unroll
    for (int i = 1; i < 9; ++i) c = fma(c, r2, kCoshC[i]);
    double sh = kSinhC[0];                         // 1/15!
#pragma unroll
    for (int i = 1; i < 8; ++i) sh = fma(sh, r2, kSinhC[i]);
    sh *= r;
    const int ni = (int)n;
    ep = (c + sh) * __hiloint2double((ni + 1023) << 20, 0);
    em = (c - sh) * __hiloint2double((1023 - ni) << 20, 0);
}

// Table-driven e^{2a} and e^{-2a} for the prox's fast path (|2a| <= 160): 2a = (64 m + j) ln2/64 + r,
// |r| <= ln2/128; e^{+-2a} = 2^{+-m} 2^{+-j/64} e^{+-r}, the cosh/sinh parts of r to r^6 / r^5
// (remainder < 4e-17 relative).  tab = k2_etab(): [0, 64) = 2^{j/64}, [64, 128) = 2^{-j/64}, in
// shared memory (filled by k2_etab_init); 2 table reads instead of ten more fp64 FMAs.
__device__ __forceinline__ double* k2_etab() {
    __shared__ double t[128];
    return t;
}
// 2^{j/64} (j = 0..63), then 2^{-j/64}: correctly rounded (60-digit decimal evaluation)
__device__ const double kK2Etab[128] = {
    1.0, 1.0108892860517005, 1.0218971486541166, 1.0330248790212284,
    1.0442737824274138, 1.0556451783605572, 1.0671404006768237, 1.0787607977571199,
    1.0905077326652577, 1.102382583307841, 1.1143867425958924, 1.1265216186082418,
    1.1387886347566916, 1.1511892299529827, 1.1637248587775775, 1.1763969916502812,
    1.189207115002721, 1.202156731452703, 1.215247359980469, 1.22848053610687,
    1.241857812073484, 1.255380757024691, 1.2690509571917332, 1.2828700160787783,
    1.2968395546510096, 1.3109612115247644, 1.3252366431597413, 1.339667524053303,
    1.3542555469368927, 1.3690024229745905, 1.383909881963832, 1.3989796725383112,
    1.4142135623730951, 1.42961333839197, 1.4451808069770467, 1.460917794180647,
    1.4768261459394993, 1.4929077282912648, 1.5091644275934228, 1.5255981507445384,
    1.5422108254079407, 1.559004400237837, 1.5759808451078865, 1.593142151342267,
    1.6104903319492543, 1.6280274218573478, 1.645755478153965, 1.6636765803267364,
    1.681792830507429, 1.7001063537185235, 1.718619298122478, 1.7373338352737062,
    1.7562521603732995, 1.7753764925265212, 1.7947090750031072, 1.8142521755003989,
    1.8340080864093424, 1.8539791250833855, 1.8741676341103, 1.8945759815869656,
    1.9152065613971474, 1.9360617934922943, 1.9571441241754002, 1.978456026387951,
    1.0, 0.9892280131939755, 0.9785720620877001, 0.9680308967461472,
    0.9576032806985737, 0.9472879907934828, 0.93708381705515, 0.9269895625416927,
    0.9170040432046712, 0.9071260877501994, 0.8973545375015536, 0.8876882462632606,
    0.8781260801866497, 0.8686669176368531, 0.859309649061239, 0.8500531768592617,
    0.8408964152537145, 0.8318382901633682, 0.8228777390769825, 0.8140137109286739,
    0.8052451659746271, 0.7965710756711335, 0.7879904225539432, 0.7795022001189185,
    0.7711054127039704, 0.7627990753722692, 0.7545822137967114, 0.7464538641456324,
    0.7384130729697497, 0.7304588970903235, 0.7225904034885233, 0.714806669195985,
    0.7071067811865476, 0.6994898362691556, 0.691954940981916, 0.6845012114872953,
    0.6771277734684463, 0.6698337620266515, 0.6626183215798707, 0.6554806057623822,
    0.6484197773255048, 0.6414350080393891, 0.6345254785958666, 0.6276903785123455,
    0.620928906036742, 0.614240268053435, 0.6076236799902345, 0.6010783657263515,
    0.5946035575013605, 0.5881984958251406, 0.5818624293887887, 0.5755946149764913,
    0.5693943173783458, 0.5632608093041209, 0.5571933712979462, 0.5511912916539204,
    0.5452538663326288, 0.5393803988785599, 0.5335702003384118, 0.5278225891802786,
    0.5221368912137069, 0.5165124395106142, 0.5109485743270583, 0.5054446430258502,
};
__device__ __forceinline__ void k2_etab_init() {
    double* t = k2_etab();
    for (int i = threadIdx.x; i < 128; i += blockDim.x) t[i] = kK2Etab[i];
}
__device__ __forceinline__ void exp2a_pm_tab(double a, double& ep, double& em) {
    const double x = 2.0 * a;
    const double kd = rint(x * 92.33248261689366);                                 // x 64 / ln 2
    const double r = fma(-kd, 3.623510646634843e-19, fma(-kd, 1.0830424696249145e-02, x));   // x - kd ln2/64
    const int k = (int)kd, j = k & 63, m = k >> 6;
    const double r2 = r * r;
#if FOE_K2_ETAB_G
    // |r| <= ln2/128: the r^6/720 term of the even part is below 4e-17 (half an ulp of c ~ 1)
    const double c = fma(r2, fma(r2, 1.0 / 24.0, 0.5), 1.0);
    const double tp = __ldg(kK2Etab + j), tm = __ldg(kK2Etab + 64 + j);
#else
    const double c = fma(r2, fma(r2, fma(r2, 1.0 / 720.0, 1.0 / 24.0), 0.5), 1.0);
    const double* t = k2_etab();
    const double tp = t[j], tm = t[64 + j];
#endif
    const double s = r * fma(r2, fma(r2, 1.0 / 120.0, 1.0 / 6.0), 1.0);
    // 2^{+-m} by the exponent field (|m| <= 127)
    ep = (c + s) * __hiloint2double(__double2hiint(tp) + (m << 20), __double2loint(tp));
    em = (c - s) * __hiloint2double(__double2hiint(tm) - (m << 20), __double2loint(tm));
}

// 1/b to full fp64 precision: MUFU reciprocal seed + two Newton steps (b finite, nonzero)
__device__ __forceinline__ double rcp_f64(double b) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(b));
    y = fma(y, fma(-b, y, 1.0), y);
    y = fma(y, fma(-b, y, 1.0), y);
    return y;
}

// fp32 Newton steps of the prox after the first (exponential-free) one, before the fp64 step
#ifndef FOE_K2_F32_STEPS
#define FOE_K2_F32_STEPS 1
#endif
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Root of phi(z) = z - what + tau [l1 (1 - f^2 e^{-2z}) + l2 (e^{2z} - f^2)],
// solved for the increment d = z - what:
//   phi(d) = d + tau(l1 - l2 f^2) - A e^{-2d} + Bc e^{2d},  A = tau l1 f^2 e^{-2 what},
//   Bc = tau l2 e^{2 what},  phi'(d) = 1 + 2 A e^{-2d} + 2 Bc e^{2d} > 0,
//   |phi''(d)| <= 4 (A e^{-2d} + Bc e^{2d}) = 2 (phi'(d) - 1).
// Newton's method from d = 0: the first step needs no exponential; at d1 one fp64
// evaluation gives the second step st, and the Newton error bound |phi(d1 - st)| <~
// |phi''|/2 st^2 <= (phi' - 1) st^2 accepts d2 = d1 - st when that bound is <= tol/4.  Otherwise
// (large steps, overflow) the safeguarded fp64 Newton/bisection iteration on the bracket
// [min(0, log f - what) - 1, max(0, log f - what) + 1] runs to |phi| <= tol
// (SPEC.md:251).  Returns the Newton updates, or -1 past the cap; em_out = e^{-2z}, ep_out = e^{2z}.
// fp32 copies of the per-image prox constants tau l1, tau l2 (hoisted out of the pixel loop: an
// fp64 <-> fp32 conversion is a slow instruction on sm_100, and K2 was stalled on them)
struct ProxF {
    float tl1, tl2;
};
// The fast path: one fp32 Newton step from d = 0 and FOE_K2_F32_STEPS more (MUFU exponentials,
// ~1e-7 relative), then ONE fp64 Newton step from there -- quadratic convergence takes the fp32
// error to ~1e-14, accepted by the error bound above; one fp64 exponential pair (at
// z0 = what + d32) instead of two.  Branch-free (|what| > 40 is computed at what = 0 and
// rejected), so that the two pixels of a pair interleave.  Returns true when accepted.
__device__ __forceinline__ bool prox_fast(double what, double f2, float ff, const ProxF& pf, double tau, double l1,
                                          double l2, double tol, double& z_out, double& em_out, double& ep_out) {
    const bool inr = fabs(what) <= 40.0;
    const double wc = inr ? what : 0.0;
    const float f2f = ff * ff, tl1f2 = pf.tl1 * f2f, tl2 = pf.tl2, c0f = fmaf(-pf.tl2, f2f, pf.tl1);
    const float wf = (float)wc;
    const float Af = tl1f2 * ex2_approx(-2.8853900817779268f * wf), Bf = tl2 * ex2_approx(2.8853900817779268f * wf);
    float d = -(c0f - Af + Bf) * rcp_approx(1.0f + 2.0f * (Af + Bf));
#pragma unroll
    for (int k = 0; k < FOE_K2_F32_STEPS; ++k) {
        const float p = ex2_approx(2.8853900817779268f * d), q = rcp_approx(p);
        const float am = Af * q, bp = Bf * p;
        d -= (d + c0f - am + bp) * rcp_approx(1.0f + 2.0f * (am + bp));
    }
    const double z0 = wc + (double)d;
    double Ep0, Em0;
#if FOE_K2_ETAB
    exp2a_pm_tab(z0, Ep0, Em0);                // e^{2 z0}, e^{-2 z0}
#else
    exp2a_pm(z0, Ep0, Em0);
#endif
    const double am = tau * l1 * f2 * Em0, bp = tau * l2 * Ep0;
    const double phi = (double)d + tau * (l1 - l2 * f2) - am + bp;
    const double dphi = 1.0 + 2.0 * (am + bp);
#if FOE_K2_RCP1
    // one Newton step on the MUFU seed (2^-22 -> ~2^-44 relative): st is accepted only when
    // |st| <= 1e-6, so its relative error contributes < 1e-19 to z
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(dphi));
    const double st = phi * fma(y, fma(-dphi, y, 1.0), y);
#else
    const double st = phi * rcp_f64(dphi);
#endif
    const double e = -2.0 * st;                                  // e^{+-e}, |e| <= 2e-6 when accepted
    z_out = z0 - st;
    ep_out = Ep0 * fma(0.5 * e, e, 1.0 + e);
    em_out = Em0 * fma(0.5 * e, e, 1.0 - e);
    // (|z0| <= 80 keeps 2 z0 inside the table exponential's range, |2a| <= 160)
    return inr & (fabs(z0) <= 80.0) & isfinite(st) & ((dphi - 1.0) * st * st <= 0.25 * tol) & (fabs(st) <= 1e-6);
}

// The safeguarded part of the prox (when the fast path rejects)
__device__ __forceinline__ int prox_slow(double what, double ft, double f2, double tau, double l1, double l2,
                                         double tol, int cap, double& z_out, double& em_out, double& ep_out) {
    double Em, Ep;
    if (fabs(what) <= 340.0) {
        exp2a_pm(what, Ep, Em);                    // e^{2 what}, e^{-2 what}
    } else {
        Em = exp(-2.0 * what);
        Ep = 1.0 / Em;
    }
    const double A = tau * l1 * f2 * Em, Bc = tau * l2 * Ep, c0 = tau * (l1 - l2 * f2);
    if (isfinite(A) && isfinite(Bc)) {
        const double phi0 = c0 - A + Bc;
        if (fabs(phi0) <= tol) { z_out = what; em_out = Em; ep_out = Ep; return 0; }
        const double d1 = -phi0 * rcp_f64(1.0 + 2.0 * (A + Bc));
        if (fabs(d1) <= 0.03125) {
            double ep2, em2;
            exp_pm_small(2.0 * d1, ep2, em2);
            const double phi = d1 + c0 - A * em2 + Bc * ep2;
            if (fabs(phi) <= tol) { z_out = what + d1; em_out = Em * em2; ep_out = Ep * ep2; return 1; }
            const double dphi = 1.0 + 2.0 * (A * em2 + Bc * ep2);
            const double st = phi * rcp_f64(dphi);
            if ((dphi - 1.0) * st * st <= 0.25 * tol && fabs(st) <= 1e-6) {
                const double e = -2.0 * st;                              // e^{+-e}, |e| <= 2e-6
                z_out = what + (d1 - st);
                ep_out = Ep * ep2 * fma(0.5 * e, e, 1.0 + e);
                em_out = Em * em2 * fma(0.5 * e, e, 1.0 - e);
                return 2;
            }
        }
    }
    const double lfw = (double)__logf((float)ft) - what;
    double lo = fmin(0.0, lfw) - 1.0, hi = fmax(0.0, lfw) + 1.0;
    double d = 0.0;
    for (int it = 0; it <= cap; ++it) {
        const double x = 2.0 * d;
        const double ep2 = exp_near0(x), em2 = exp_near0(-x);
        const double phi = d + c0 - A * em2 + Bc * ep2;
        if (fabs(phi) <= tol) { z_out = what + d; em_out = Em * em2; ep_out = Ep * ep2; return it; }
        if (phi > 0.0) hi = d; else lo = d;
        const double dphi = 1.0 + 2.0 * (A * em2 + Bc * ep2);
        double dn = d - phi / dphi;
        if (!(dn > lo && dn < hi)) dn = 0.5 * (lo + hi);
        if (dn == d) { z_out = what + d; em_out = Em * em2; ep_out = Ep * ep2; return it; }
        d = dn;
    }
    z_out = what + d; em_out = exp(-2.0 * z_out); ep_out = exp(2.0 * z_out);
    return -1;
}

__device__ __forceinline__ int prox_newton(double what, double ft, float ff, const ProxF& pf, double tau, double l1,
                                           double l2, double tol, int cap, double& z_out,
                                           double& em_out, double& ep_out) {
    const double f2 = ft * ft;
    if (prox_fast(what, f2, ff, pf, tau, l1, l2, tol, z_out, em_out, ep_out)) return 4;
    return prox_slow(what, ft, f2, tau, l1, l2, tol, cap, z_out, em_out, ep_out);
}

struct K2Args {
    double* w;            // [3][B][HW]
    size_t w_slot_stride;
    const float* g;       // [2][groups][B][HW]
    size_t g_slot_stride, g_group_stride;
    const float* ft;      // [B][HW]  f~ = max(f,1)
    double* ppart;        // [B][nblk][kNumPart]
    const ImgCtl* ctl;
    SolverParams sp;
    int groups, nblk;
    size_t HW;
    // Row slab: w+ of the first kHalo rows is also stored at halo_up (the slab above's bottom
    // ghost rows), of the last kHalo rows at halo_dn (the slab below's top ghost rows) -- a
    // neighbour's buffer written directly (same GPU, or a peer GPU over NVLink through a CUDA IPC
    // mapping), or this slab's send buffer for NCCL; nullptr = no slab.
    double* halo_up;
    double* halo_dn;
    int halo_sys_fence;    // peer-GPU destination: make the stores visible system-wide
    int pairs;             // HW % 4 == 0: pixel pairs by 16-/8-byte vector loads (inertial_prox_pairs)
    size_t halo_px;        // kHalo * W
    int idiv;              // model (6) in u: closed-form prox of (lam/2)(u^2 - 2 f^2 log u), lam = lam1
};

// Test partials of one trial (a10): <g, D>, ||D||^2, G(w+), ||w||^2, max |w+| (or the domain
// flag of model (6)), max Newton iterations, prox failures.
struct K2Acc {
    double gd = 0, dd = 0, Gp = 0, ww = 0;
    unsigned long long wbits = 0;   // max |w+| as the bits of a non-negative double (NaN > inf)
    int nit = 0, fail = 0;
};

// a pixel's contribution to the test partials (a10)
// (G(w+) of Eq. (10): (l1/2)(2z + f^2 e^{-2z}) + (l2/2)(e^{2z} - 2 f^2 z) = l1 z + (l1/2) f^2 e^{-2z}
//  + (l2/2) e^{2z} - l2 f^2 z; max |w+| by the bits of |z|, NaN above inf)
__device__ __forceinline__ void k2_acc(K2Acc& acc, double wv, double gv, double f2, double z, double em, double ep,
                                       int it, double l1, double l2, int idiv) {
    const double d = z - wv;
    acc.gd += gv * d;
    acc.dd += d * d;
    if (idiv) {
        acc.Gp += 0.5 * l1 * (z * z - 2.0 * f2 * log(z));                 // Eq.(5)
        const unsigned long long b = z > 0.0 ? 0ull : 0x7ff0000000000000ull;   // the iterate must stay > 0
        acc.wbits = max(acc.wbits, b);
    } else {
        double g = fma(0.5 * l1, f2 * em, acc.Gp);
        g = fma(0.5 * l2, ep, g);
        g = fma(l1, z, g);
        acc.Gp = fma(-l2, f2 * z, g);
        acc.wbits = max(acc.wbits, (unsigned long long)__double_as_longlong(z) & 0x7fffffffffffffffull);
    }
    acc.ww += wv * wv;
    if (it < 0) ++acc.fail; else acc.nit = max(acc.nit, it);
}

// One pixel of K2 (a8-a10): inertial point, prox, and its contribution to the test partials.
// Shared by k_inertial_prox and the persistent driver's phase A; the inertial point is written
// with explicit roundings so that both compile to the same arithmetic (bitwise-equal w+).
__device__ __forceinline__ double k2_pixel(double wv, double wpv, double gv, double f, float ff, double alpha,
                                           double beta, double l1, double l2, const ProxF& pf,
                                           const SolverParams& sp, int idiv, K2Acc& acc) {
    const double what = __fma_rn(beta, __dsub_rn(wv, wpv), __fma_rn(-alpha, gv, wv));
    double z, em, ep;
    int it;
    if (idiv) {
        // u = (u^ + sqrt(u^2 + 4 (1 + tau lam) tau lam f^2)) / (2 (1 + tau lam))
        const double tl = alpha * l1;
        z = (what + sqrt(fma(what, what, 4.0 * (1.0 + tl) * tl * f * f))) / (2.0 * (1.0 + tl));
        em = 0.0; ep = 0.0; it = 0;
    } else {
        it = prox_newton(what, f, ff, pf, alpha, l1, l2, sp.newton_tol, sp.newton_cap, z, em, ep);
    }
    k2_acc(acc, wv, gv, f * f, z, em, ep, it, l1, l2, idiv);
    return z;
}

// Lock-step pair of pixels of model (10)/(8) (inertial_prox_pairs): both inertial points, both
// fast-path proxes as one straight-line block (the scheduler interleaves the two dependency
// chains), the safeguarded prox only for a rejected pixel, then the partials in pixel order --
// per pixel the same arithmetic as k2_pixel.
__device__ __forceinline__ double2 k2_pair(const double2 wv, const double2 wpv, const float2 gs, const float2 fv,
                                           double alpha, double beta, double l1, double l2, const ProxF& pf,
                                           const SolverParams& sp, K2Acc& acc) {
    const double gx = (double)gs.x, gy = (double)gs.y, fx = (double)fv.x, fy = (double)fv.y;
    const double wx = __fma_rn(beta, __dsub_rn(wv.x, wpv.x), __fma_rn(-alpha, gx, wv.x));
    const double wy = __fma_rn(beta, __dsub_rn(wv.y, wpv.y), __fma_rn(-alpha, gy, wv.y));
    const double f2x = fx * fx, f2y = fy * fy;
    double zx, emx, epx, zy, emy, epy;
    const bool okx = prox_fast(wx, f2x, fv.x, pf, alpha, l1, l2, sp.newton_tol, zx, emx, epx);
    const bool oky = prox_fast(wy, f2y, fv.y, pf, alpha, l1, l2, sp.newton_tol, zy, emy, epy);
    int itx = 4, ity = 4;
    if (!okx) itx = prox_slow(wx, fx, f2x, alpha, l1, l2, sp.newton_tol, sp.newton_cap, zx, emx, epx);
    if (!oky) ity = prox_slow(wy, fy, f2y, alpha, l1, l2, sp.newton_tol, sp.newton_cap, zy, emy, epy);
    k2_acc(acc, wv.x, gx, f2x, zx, emx, epx, itx, l1, l2, 0);
    k2_acc(acc, wv.y, gy, f2y, zy, emy, epy, ity, l1, l2, 0);
    return make_double2(zx, zy);
}

// fixed-order CTA reduction of the 7 test partials (sums; slots 4 and 5 max) -> out[0..7]
// (out[7] = 0); every thread of the CTA calls it
__device__ __forceinline__ void k2_block_partials(const K2Acc& acc, double* out) {
    const double wmax = acc.wbits > 0x7ff0000000000000ull ? INFINITY : __longlong_as_double((long long)acc.wbits);
    double v[7] = {acc.gd, acc.dd, acc.Gp, acc.ww, wmax, (double)acc.nit, (double)acc.fail};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int k = 0; k < 7; ++k) {
            const double t = __shfl_xor_sync(0xffffffffu, v[k], o);
            v[k] = (k == 4 || k == 5) ? fmax(v[k], t) : v[k] + t;
        }
    __shared__ double wred[32][8];
    const int nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int k = 0; k < 7; ++k) wred[threadIdx.x >> 5][k] = v[k];
    __syncthreads();
    if (threadIdx.x < 7) {
        const int k = threadIdx.x;
        double t = wred[0][k];
        for (int i = 1; i < nw; ++i) t = (k == 4 || k == 5) ? fmax(t, wred[i][k]) : t + wred[i][k];
        out[k] = t;
        if (k == 0) out[7] = 0.0;
    }
}

// pixel block bx of image b (kThreads * PXT pixels); the caller syncs the CTA between blocks
template <int PXT>
__device__ __forceinline__ void inertial_prox_blk(const K2Args& a, const int bx, const int b) {
    const ImgCtl& c = a.ctl[b];
    if (!c.active) return;
    const double alpha = a.sp.safety * 2.0 * (1.0 - a.sp.beta) / c.L;
    const double beta = a.sp.beta, l1 = c.lam1, l2 = c.lam2;
    const ProxF pf{(float)(alpha * l1), (float)(alpha * l2)};
    const double* w = a.w + (size_t)c.cur * a.w_slot_stride + (size_t)b * a.HW;
    const double* wp = a.w + (size_t)c.prev * a.w_slot_stride + (size_t)b * a.HW;
    double* wn = a.w + (size_t)c.cand * a.w_slot_stride + (size_t)b * a.HW;
    const float* g = a.g + (size_t)c.gcur * a.g_slot_stride + (size_t)b * a.HW;
    const float* ft = a.ft + (size_t)b * a.HW;
    K2Acc acc;
    const size_t base = (size_t)bx * (kThreads * PXT);
#pragma unroll kK2Unroll
    for (int k = 0; k < PXT; ++k) {
        const size_t p = base + (size_t)k * kThreads + threadIdx.x;
        if (p >= a.HW) break;
        float gs = g[p];
        for (int q = 1; q < a.groups; ++q) gs += g[(size_t)q * a.g_group_stride + p];
        const float fv = ft[p];
        const double z = k2_pixel(w[p], wp[p], (double)gs, (double)fv, fv, alpha, beta, l1, l2, pf, a.sp, a.idiv, acc);
        wn[p] = z;
        if (a.halo_up != nullptr) {
            if (p < a.halo_px) a.halo_up[p] = z;
            else if (p >= a.HW - a.halo_px) a.halo_dn[p - (a.HW - a.halo_px)] = z;
        }
    }
    if (a.halo_sys_fence) __threadfence_system();
    k2_block_partials(acc, a.ppart + ((size_t)b * a.nblk + bx) * kNumPart);
}

// Pixel block bx of image b by pixel PAIRS (HW % 4 == 0, so every pair is 16-/8-byte aligned): one
// vector load per array per pair, 32-bit pair indices, the next pair's loads issued before the
// current pair's arithmetic; the per-image constants come from shared memory (im).  Same per-pixel
// arithmetic as inertial_prox_blk (k2_pixel), so w+ is bitwise the same.
struct K2Img {
    double alpha, beta, l1, l2;
    ProxF pf;
};
template <int PXT>
__device__ __forceinline__ void inertial_prox_pairs(const K2Args& a, const K2Img& im, const int bx, const int b) {
    const ImgCtl& c = a.ctl[b];
    const size_t base = (size_t)bx * (kThreads * PXT), o = (size_t)b * a.HW + base;
    const double2* w2 = reinterpret_cast<const double2*>(a.w + (size_t)c.cur * a.w_slot_stride + o);
    const double2* wp2 = reinterpret_cast<const double2*>(a.w + (size_t)c.prev * a.w_slot_stride + o);
    double2* wn2 = reinterpret_cast<double2*>(a.w + (size_t)c.cand * a.w_slot_stride + o);
    const float2* g2 = reinterpret_cast<const float2*>(a.g + (size_t)c.gcur * a.g_slot_stride + o);
    const float2* f2p = reinterpret_cast<const float2*>(a.ft + o);
    const int n2 = (int)(min((size_t)(kThreads * PXT), a.HW - base) >> 1);
    const int gq = (int)(a.g_group_stride >> 1);
    K2Acc acc;
    int q = threadIdx.x;
    if (q < n2) {
        double2 wv = w2[q], wpv = wp2[q];
        float2 gs = g2[q], fv = f2p[q];
        for (int k = 1; k < a.groups; ++k) { const float2 t = g2[k * gq + q]; gs.x += t.x; gs.y += t.y; }
#pragma unroll 1
        for (int k = 0; k < PXT / 2; ++k) {
            const int qn = q + kThreads;
            const bool more = k + 1 < PXT / 2 && qn < n2;
            double2 wv1 = make_double2(0.0, 0.0), wpv1 = wv1;
            float2 gs1 = make_float2(0.f, 0.f), fv1 = make_float2(1.f, 1.f);
            if (more) {
                wv1 = w2[qn]; wpv1 = wp2[qn]; gs1 = g2[qn]; fv1 = f2p[qn];
                for (int kk = 1; kk < a.groups; ++kk) { const float2 t = g2[kk * gq + qn]; gs1.x += t.x; gs1.y += t.y; }
            }
            double2 z;
            if (a.idiv || !FOE_K2_LOCKSTEP) {
                z.x = k2_pixel(wv.x, wpv.x, (double)gs.x, (double)fv.x, fv.x, im.alpha, im.beta, im.l1, im.l2, im.pf, a.sp, a.idiv, acc);
                z.y = k2_pixel(wv.y, wpv.y, (double)gs.y, (double)fv.y, fv.y, im.alpha, im.beta, im.l1, im.l2, im.pf, a.sp, a.idiv, acc);
            } else {
                z = k2_pair(wv, wpv, gs, fv, im.alpha, im.beta, im.l1, im.l2, im.pf, a.sp, acc);
            }
            wn2[q] = z;
            if (a.halo_up != nullptr) {
                const size_t p = base + 2 * (size_t)q;
                if (p < a.halo_px) { a.halo_up[p] = z.x; a.halo_up[p + 1] = z.y; }
                else if (p >= a.HW - a.halo_px) {
                    a.halo_dn[p - (a.HW - a.halo_px)] = z.x; a.halo_dn[p + 1 - (a.HW - a.halo_px)] = z.y;
                }
            }
            if (!more) break;
            q = qn; wv = wv1; wpv = wpv1; gs = gs1; fv = fv1;
        }
    }
    if (a.halo_sys_fence) __threadfence_system();
    k2_block_partials(acc, a.ppart + ((size_t)b * a.nblk + bx) * kNumPart);
}

// L2 prefetch of bytes [p, p + n) by one bulk request (the 16-B aligned interior; a hint: the
// loads that follow read the same addresses)
__device__ __forceinline__ void l2_prefetch_range(const void* p, size_t n) {
    const uintptr_t s = ((uintptr_t)p + 15) & ~(uintptr_t)15, e = ((uintptr_t)p + n) & ~(uintptr_t)15;
    if (e > s)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(s), "r"((uint32_t)(e - s)) : "memory");
}

#ifndef FOE_K2_L2PF
#define FOE_K2_L2PF 0   // measured with the pair path: 158.7 us with, 153.9 without
#endif
template <int PXT>
__global__ void __launch_bounds__(kThreads, FOE_K2_CTAS)
k_inertial_prox(const K2Args a) {
#if FOE_K2_ETAB && !FOE_K2_ETAB_G
    k2_etab_init();
    __syncthreads();
#endif
    pdl_wait();   // programmatic launch after K3: its control blocks must be complete
#if FOE_K2_L2PF
    // K2 is latency-bound on its loads (long-scoreboard stalls at the first use of g and f~): one
    // thread asks L2 for the block's whole range of w, w-, g, f~ up front, so that the per-pixel
    // loads after the first unrolled pair hit L2 (~250 cycles) instead of HBM
    if (threadIdx.x == 0) {
        const ImgCtl& c = a.ctl[blockIdx.y];
        const size_t base = (size_t)blockIdx.x * (kThreads * PXT);
        if (c.active && base < a.HW) {
            const size_t n = min((size_t)(kThreads * PXT), a.HW - base), o = (size_t)blockIdx.y * a.HW + base;
            l2_prefetch_range(a.w + (size_t)c.cur * a.w_slot_stride + o, n * 8);
            l2_prefetch_range(a.w + (size_t)c.prev * a.w_slot_stride + o, n * 8);
            for (int q = 0; q < a.groups; ++q)
                l2_prefetch_range(a.g + (size_t)c.gcur * a.g_slot_stride + (size_t)q * a.g_group_stride + o, n * 4);
            l2_prefetch_range(a.ft + o, n * 4);
        }
    }
#endif
    if (PXT % 2 == 0 && a.pairs) {
        __shared__ K2Img im;
        const ImgCtl& c = a.ctl[blockIdx.y];
        if (c.active) {
            if (threadIdx.x == 0) {
                im.alpha = a.sp.safety * 2.0 * (1.0 - a.sp.beta) / c.L;
                im.beta = a.sp.beta; im.l1 = c.lam1; im.l2 = c.lam2;
                im.pf = ProxF{(float)(im.alpha * c.lam1), (float)(im.alpha * c.lam2)};
            }
            __syncthreads();
            inertial_prox_pairs<PXT>(a, im, blockIdx.x, blockIdx.y);
        }
    } else {
        inertial_prox_blk<PXT>(a, blockIdx.x, blockIdx.y);
    }
    pdl_trigger();
}

// ---------------------------------------------------------------------------------
// K3: decision, rotation, Lipschitz update, trace (one CTA per image).
// ---------------------------------------------------------------------------------
struct K3Args {
    ImgCtl* ctl;
    const double* epart;  // [B][ne] (element i at epart[(b ne + i) estride])
    const double* ppart;  // [B][nblk][kNumPart]
    double* trace;        // [B][max_iters+1][8]
    int ne, nblk, estride;
    SolverParams sp;
};

enum { ST_OK = 0, ST_NONFINITE = 4, ST_BACKTRACK = 5, ST_PROX = 6, ST_DOMAIN = 7 };

// the decision of image b by one CTA (trace == nullptr: not recorded by this CTA)
__device__ __forceinline__ void decide_img(const K3Args& a, const int b) {
    ImgCtl& c = a.ctl[b];
    if (!c.active) return;
    double e = 0.0;
    for (int i = threadIdx.x; i < a.ne; i += kThreads) e += a.epart[((size_t)b * a.ne + i) * a.estride];
    double s[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int i = threadIdx.x; i < a.nblk; i += kThreads) {
        const double* p = a.ppart + ((size_t)b * a.nblk + i) * kNumPart;
        s[0] += p[0]; s[1] += p[1]; s[2] += p[2]; s[3] += p[3];
        s[4] = fmax(s[4], p[4]); s[5] = fmax(s[5], p[5]); s[6] += p[6];
    }
    // the 8 reductions in one pass (per value the order of block_sum_d / block_max_d: xor
    // butterfly in the warp, then the warps in index order), one CTA barrier
    double v[8] = {e, s[0], s[1], s[2], s[3], s[4], s[5], s[6]};
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = (k == 5 || k == 6) ? warp_max_d(v[k]) : warp_sum_d(v[k]);
    __shared__ double wred8[kThreads / 32][8];
    __syncthreads();
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int k = 0; k < 8; ++k) wred8[threadIdx.x >> 5][k] = v[k];
    __syncthreads();
    if (threadIdx.x != 0) return;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        double t = (k == 5 || k == 6) ? wred8[0][k] : 0.0 + wred8[0][k];
        for (int i = 1; i < kThreads / 32; ++i) t = (k == 5 || k == 6) ? fmax(t, wred8[i][k]) : t + wred8[i][k];
        v[k] = t;
    }
    const double Fp = v[0], gd = v[1], dd = v[2], Gp = v[3], ww = v[4], wmax = v[5], nit = v[6], fail = v[7];
    c.trials += 1;
    c.total_trials += 1;
    if (fail > 0.0) {
        c.status = ST_PROX;
        c.active = 0;
        return;
    }
    const double L = c.L;
    const double margin = c.F + gd + 0.5 * L * dd - Fp;
    const bool ok = isfinite(Fp) && isfinite(gd) && isfinite(dd) && isfinite(Gp) && margin >= 0.0;
    if (ok) {
        if (!(wmax <= a.sp.w_guard)) c.status = isfinite(wmax) ? ST_DOMAIN : ST_NONFINITE;  // R-11
        const int old_prev = c.prev;
        c.prev = c.cur; c.cur = c.cand; c.cand = old_prev;
        const int og = c.gcur; c.gcur = c.gcand; c.gcand = og;
        c.F = Fp;
        c.n += 1;
        const double relchg = sqrt(dd) / fmax(sqrt(ww), 1.0);
        if (a.sp.record_trace && a.trace != nullptr) {
            double* r = a.trace + ((size_t)b * (a.sp.max_iters + 1) + c.n) * 8;
            r[0] = Fp; r[1] = Gp; r[2] = Fp + Gp; r[3] = L; r[4] = (double)c.trials;
            r[5] = margin; r[6] = nit; r[7] = relchg;
        }
        c.trials = 0;
        c.L = L * a.sp.shrink;                                        // R-9
        if (a.sp.rel_tol > 0.0 && relchg < a.sp.rel_tol) c.done = 1;
    } else {
        if (c.trials > a.sp.max_backtracks) c.status = ST_BACKTRACK;
        c.L = L * a.sp.eta;
    }
    c.active = (c.status == ST_OK && !c.done && c.n < c.target) ? 1 : 0;
}

__global__ void __launch_bounds__(kThreads) k_decide(const K3Args a) {
    pdl_wait();
    decide_img(a, blockIdx.x);
    pdl_trigger();
}

// ---------------------------------------------------------------------------------
// Setup / helper kernels
// ---------------------------------------------------------------------------------

// f~ = max(f,1) (R-4); w^0 = log f~ into slots 0 and 1 (w^{-1} = w^0, R-8); per-block
// partials of G(w^0) (slot 2 of ppart).
__global__ void __launch_bounds__(kThreads)
k_init(const float* f, float* ft, double* w, size_t w_slot_stride, double* ppart, int nblk,
       const ImgCtl* ctl, size_t HW, int pxt, double* halo_up, double* halo_dn, size_t halo_px, int idiv) {
    __shared__ double red[32];
    const int b = blockIdx.y;
    const double l1 = ctl[b].lam1, l2 = ctl[b].lam2;
    double G = 0.0;
    const size_t base = (size_t)blockIdx.x * kThreads * pxt;
    for (int k = 0; k < pxt; ++k) {
        const size_t p = base + (size_t)k * kThreads + threadIdx.x;
        if (p >= HW) break;
        const size_t gi = (size_t)b * HW + p;
        const float fv = fmaxf(f[gi], 1.0f);
        ft[gi] = fv;
        const double fd = (double)fv;
        const double z = idiv ? fd : log(fd);          // u^0 = f~ (model (6)) or w^0 = log f~
        w[gi] = z;
        w[w_slot_stride + gi] = z;
        if (halo_up != nullptr) {   // row slab (B = 1): rows the ring neighbours need (as K2)
            if (p < halo_px) halo_up[p] = z;
            else if (p >= HW - halo_px) halo_dn[p - (HW - halo_px)] = z;
        }
        const double f2 = fd * fd;
        G += idiv ? 0.5 * l1 * (z * z - 2.0 * f2 * log(z))
                  : 0.5 * l1 * (2.0 * z + f2 * exp(-2.0 * z)) + 0.5 * l2 * (exp(2.0 * z) - 2.0 * f2 * z);
    }
    if (halo_up != nullptr) __threadfence_system();
    const double s = block_sum_d(G, red);
    if (threadIdx.x == 0) {
        double* out = ppart + ((size_t)b * nblk + blockIdx.x) * kNumPart;
        for (int i = 0; i < kNumPart; ++i) out[i] = 0.0;
        out[2] = s;
    }
}

// F(w^0), G(w^0) -> ctl, trace row 0.
__global__ void __launch_bounds__(kThreads)
k_init_finalize(ImgCtl* ctl, const double* epart, int ne, int estride, const double* ppart, int nblk,
                double* trace, int max_iters, int record) {
    __shared__ double red[32];
    const int b = blockIdx.x;
    double e = 0.0, g = 0.0;
    for (int i = threadIdx.x; i < ne; i += kThreads) e += epart[((size_t)b * ne + i) * estride];
    for (int i = threadIdx.x; i < nblk; i += kThreads) g += ppart[((size_t)b * nblk + i) * kNumPart + 2];
    const double F = block_sum_d(e, red);
    const double G = block_sum_d(g, red);
    if (threadIdx.x == 0) {
        ctl[b].F = F;
        if (!isfinite(F)) ctl[b].status = ST_NONFINITE;
        if (record) {
            double* r = trace + (size_t)b * (max_iters + 1) * 8;
            r[0] = F; r[1] = G; r[2] = F + G; r[3] = ctl[b].L;
            r[4] = 0; r[5] = 0; r[6] = 0; r[7] = 0;
        }
    }
}

__global__ void k_set_target(ImgCtl* ctl, int B, int target) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    ImgCtl& c = ctl[b];
    c.target = target;
    c.active = (c.status == ST_OK && !c.done && c.n < target) ? 1 : 0;
}

// out[b][k] = fixed-order sum over blocks of part[b][blk][k] (k < K) -- generic finaliser.
__global__ void __launch_bounds__(kThreads)
k_reduce_rows(const double* part, int nblk, int stride, int K, double* out) {
    __shared__ double red[32];
    const int b = blockIdx.x;
    for (int k = 0; k < K; ++k) {
        double s = 0.0;
        for (int i = threadIdx.x; i < nblk; i += kThreads) s += part[((size_t)b * nblk + i) * stride + k];
        s = block_sum_d(s, red);
        if (threadIdx.x == 0) out[(size_t)b * K + k] = s;
    }
}

// Row slab (B = 1): per-band partials of one slab, band k = slab rows [64k, 64k+64) = tile row
// k = K2 blocks [k bpb, (k+1) bpb).  out[k][0..6] = the K2 partials of the band (sums; slots
// 4/5 max), out[k][7] = the band's K1 energy partials.  Bands are a fixed global partition of
// the scene, so the decision's sums do not depend on how many slabs it is cut into.
__global__ void __launch_bounds__(kThreads)
k_band_reduce(const double* epart, int e_per_band, const double* ppart, int bpb, double* out) {
    __shared__ double red[32];
    const int k = blockIdx.x;
    double e = 0.0;
    for (int i = threadIdx.x; i < e_per_band; i += kThreads) e += epart[(size_t)k * e_per_band + i];
    double s[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int i = threadIdx.x; i < bpb; i += kThreads) {
        const double* p = ppart + ((size_t)k * bpb + i) * kNumPart;
        s[0] += p[0]; s[1] += p[1]; s[2] += p[2]; s[3] += p[3];
        s[4] = fmax(s[4], p[4]); s[5] = fmax(s[5], p[5]); s[6] += p[6];
    }
    double r[8];
    r[0] = block_sum_d(s[0], red);
    r[1] = block_sum_d(s[1], red);
    r[2] = block_sum_d(s[2], red);
    r[3] = block_sum_d(s[3], red);
    r[4] = block_max_d(s[4], red);
    r[5] = block_max_d(s[5], red);
    r[6] = block_sum_d(s[6], red);
    r[7] = block_sum_d(e, red);
    if (threadIdx.x < 8) out[(size_t)k * kNumPart + threadIdx.x] = r[threadIdx.x];
}

// data energy partials of a given w (foe_energy_grad): part[b][blk][0]
__global__ void __launch_bounds__(kThreads)
k_data_energy(const double* w, const float* f, const double* lam, double* part, int nblk, size_t HW, int pxt,
              int idiv) {
    __shared__ double red[32];
    const int b = blockIdx.y;
    const double l1 = lam[2 * b], l2 = lam[2 * b + 1];
    double G = 0.0;
    const size_t base = (size_t)blockIdx.x * kThreads * pxt;
    for (int k = 0; k < pxt; ++k) {
        const size_t p = base + (size_t)k * kThreads + threadIdx.x;
        if (p >= HW) break;
        const size_t gi = (size_t)b * HW + p;
        const double fd = (double)fmaxf(f[gi], 1.0f);
        const double z = w[gi];
        const double f2 = fd * fd;
        G += idiv ? 0.5 * l1 * (z * z - 2.0 * f2 * log(z))
                  : 0.5 * l1 * (2.0 * z + f2 * exp(-2.0 * z)) + 0.5 * l2 * (exp(2.0 * z) - 2.0 * f2 * z);
    }
    const double s = block_sum_d(G, red);
    if (threadIdx.x == 0) part[(size_t)b * nblk + blockIdx.x] = s;
}

// g = sum over groups of the partial gradient planes (fixed order)
__global__ void k_sum_groups(const float* gparts, size_t group_stride, int groups, float* out, size_t n) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float s = gparts[i];
    for (int q = 1; q < groups; ++q) s += gparts[(size_t)q * group_stride + i];
    out[i] = s;
}

// power iteration helpers: part[b][blk] = {<v,h>, <h,h>, <v0,v0>}
__global__ void __launch_bounds__(kThreads)
k_dot3(const double* v, const float* h, double* part, int nblk, size_t HW, int pxt) {
    __shared__ double red[32];
    const int b = blockIdx.y;
    double vh = 0.0, hh = 0.0, vv = 0.0;
    const size_t base = (size_t)blockIdx.x * kThreads * pxt;
    for (int k = 0; k < pxt; ++k) {
        const size_t p = base + (size_t)k * kThreads + threadIdx.x;
        if (p >= HW) break;
        const size_t gi = (size_t)b * HW + p;
        const double a = v ? v[gi] : 0.0;    // (v == nullptr: only <h,h>, the power iteration's
        const double c = h ? (double)h[gi] : 0.0;   //  steps before the last)
        vh += a * c; hh += c * c; vv += a * a;
    }
    const double s0 = block_sum_d(vh, red), s1 = block_sum_d(hh, red), s2 = block_sum_d(vv, red);
    if (threadIdx.x == 0) {
        double* o = part + ((size_t)b * nblk + blockIdx.x) * 3;
        o[0] = s0; o[1] = s1; o[2] = s2;
    }
}

// v <- src / sqrt(norm2[b*K + k]) (grid: x = chunks of image b = blockIdx.y; the norm once per thread)
template <typename T>
__global__ void k_normalize(const T* src, double* v, const double* sums, int K, int k, size_t HW, int B) {
    const int b = blockIdx.y;
    const double nrm = sqrt(sums[(size_t)b * K + k]);
    const T* sp = src + (size_t)b * HW;
    double* vp = v + (size_t)b * HW;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < HW; i += (size_t)gridDim.x * blockDim.x)
        vp[i] = (double)sp[i] / nrm;
}

__global__ void k_log_ftilde(const float* f, double* w, size_t n, int idiv) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) w[i] = idiv ? (double)fmaxf(f[i], 1.0f) : log((double)fmaxf(f[i], 1.0f));
}

// a13: u = e^w of each image's current slot (and/or a copy of w)
__global__ void k_iterate_out(const ImgCtl* ctl, const double* w, size_t slot_stride, double* w_out,
                              float* u_out, size_t HW, int udom) {
    const int b = blockIdx.y;
    const double* src = w + (size_t)ctl[b].cur * slot_stride + (size_t)b * HW;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < HW; i += (size_t)gridDim.x * blockDim.x) {
        const double v = src[i];
        if (w_out) w_out[(size_t)b * HW + i] = v;
        if (u_out) u_out[(size_t)b * HW + i] = (float)(udom ? v : exp(v));
    }
}

}  // namespace foe
