// foe_tc.cuh -- K8: the fused FoE prior energy + gradient (rows a2-a7 of SURVEY.md 8(a)) on the
// sm_100a tensor cores (tcgen05, TF32 with a 3-pass hi/lo split for fp32-level accuracy).
//
// The two correlations of grad_w F = W sum_i theta_i K_i^T rho'(K_i e^w)
// are written as GEMMs over one row of 128 response pixels at a time (M = 128 TMEM lanes):
//
//   forward   R[q, i] = sum_t U[q, t] Kf[t, i]      U = im2col of u - c (taps t = a*m + b of
//                                                   the m x m window, K padded to KT = 8k),
//                                                   Kf = flipped taps (true convolution, R-2)
//   backward  Z[q, t] = sum_i P[q, i] Kb[i, t]      P = rho'(r)/2 = r/(1+r^2), Kb = 2 theta_i k_i
//             s[p]    = sum_t Z[p + off(t), t]      (col2im: a 49-term gather through smem)
//
// A operands (U, P) live in TMEM, written by the epilogue threads (one pixel = one TMEM lane);
// B operands (Kf, Kb; hi and lo tf32 halves) are staged once per CTA in shared memory in the
// K-major no-swizzle canonical layout; accumulators R and Z are in TMEM.  Each product x.y is
// evaluated as x_hi y_hi + x_hi y_lo + x_lo y_hi with x_hi = tf32(x), x_lo = x - x_hi (its top
// 11 bits are what the tensor core reads):
// error ~2^-21 relative, i.e. fp32-level (the path's tolerance is 1e-5 relative L2,
// BASELINE.json north_star).  The im2col subtracts each response pixel's own window centre
// u_q (a per-pixel DC shift, restored as u_q sum_t k in the epilogue), so the tensor-core
// operands are local differences; the tile-wide shift of K1 was not enough here (the tensor
// core's fp32 accumulation gave 1.2e-5 gradient error on smooth tiles).
//
// One CTA (256 threads = 2 warp groups x 4 warps; warp w reaches TMEM lanes 32 (w % 4) ..) =
// an output tile of R rows x (128 - 2C) columns = (R + 2C) response rows of 128 lanes + a
// (R + 4C) x (128 + 2C) u tile.  Per response row: im2col -> 3*(KT/8) forward MMAs -> rho,
// rho' epilogue -> 3*(NP/8) backward MMAs -> Z through smem -> rolling col2im sums of the
// 2C+1 output rows it touches; the two warp groups split every phase (tap chunks, filter
// chunks, col2im rows).  Two CTAs per SM overlap one CTA's MMAs with the other's epilogue.
#pragma once

#include "foe_kernels.cuh"
#include "tc_ptx.cuh"

// rows of the u tile a warp stages at a time (their loads all in flight before the exponentials)
#ifndef FOE_STAGE_ROWS
#define FOE_STAGE_ROWS 2
#endif

// 1: K8's epilogue takes one MUFU reciprocal per filter pair (the XU pipe is K8's busiest
// thread-work pipe); 0: one per filter
#ifndef FOE_K8_PAIR_RCP
#define FOE_K8_PAIR_RCP 1
#endif

namespace foe {

template <int M, int NP, int R>
struct TcGeom {
    static constexpr int C = (M - 1) / 2;
    static constexpr int TAPS = M * M;
    static constexpr int KT = ((TAPS + 7) / 8) * 8;     // forward K (taps), backward N
    static constexpr int LANES = 128;                   // response pixels per row (TMEM lanes)
    static constexpr int OW = LANES - 2 * C;            // output columns per tile
    static constexpr int RR = R + 2 * C;                // response rows per tile
    static constexpr int UY = R + 4 * C;                // staged u rows
    static constexpr int UX = LANES + 2 * C;            // staged u columns
    static constexpr int UP = UX + 2;                   // u pitch (floats)
    // backward GEMM covers taps [0, NB); the last tap (TAPS = 1 mod 8 for odd m) is a 1-column
    // dot product done in the epilogue on CUDA cores, so Z (NB <= NP columns) can reuse D's
    // columns and the A columns stay free for the next row's im2col while the backward MMA runs
    static constexpr int NB = (TAPS / 8) * 8;
    // TMEM columns
    static constexpr int COL_AHI = 0, COL_ALO = KT, COL_D = 2 * KT, COL_PHI = 2 * KT + NP, COL_PLO = 2 * KT + 2 * NP;
    static constexpr int COL_Z = COL_D;
    static constexpr int TCOLS_USED = 2 * KT + 3 * NP;
    static constexpr int TCOLS = TCOLS_USED <= 32 ? 32 : TCOLS_USED <= 64 ? 64 : TCOLS_USED <= 128 ? 128
                                 : TCOLS_USED <= 256 ? 256 : 512;
    // B operand images (floats): Kf [KT/4][NP][4] and Kb [NP/4][NB][4], hi then lo, then the
    // last tap of Kb as a plain vector [NP]
    static constexpr int BF_FLOATS = KT * NP;
    static constexpr int BB_FLOATS = NP * NB;
    static constexpr int B_FLOATS = 2 * BF_FLOATS + 2 * BB_FLOATS + NP;
    // shared memory (floats): B images | u tile | Z transpose [TAPS][LANES] | col2im hand-off
    // ring [8][LANES] | last-tap partials [2 rows][2 groups][LANES] | sum k | theta ln2
    static constexpr int SM_B = 0;
    static constexpr int SM_U = SM_B + B_FLOATS;
    static constexpr int SM_Z = SM_U + UY * UP;
    static constexpr int SM_HAND = SM_Z + TAPS * LANES;
    static constexpr int SM_ZL = SM_HAND + 8 * LANES;
    static constexpr int SM_CS = SM_ZL + 4 * LANES;
    static constexpr int SM_TH = SM_CS + NP;
    static constexpr int SM_FLOATS = SM_TH + NP;
    static constexpr int SMEM_BYTES = SM_FLOATS * 4 + 64;
    static_assert(NB <= NP && TAPS - NB == 1, "one CUDA-core tap, Z inside D");
    static_assert(TCOLS_USED <= 512, "TMEM budget");
    static_assert(NP % 16 == 0 && KT % 8 == 0, "MMA shape");
    static_assert((B_FLOATS * 4) % 16 == 0, "B images: one TMA bulk copy (multiple of 16 bytes)");
};

// Per-filter constants of K8's epilogue, in the kernel-parameter constant bank (FFMA operands
// straight from c[], no shared-memory loads): sum_t k_i (DC restore), theta_i ln 2 (energy),
// and the last tap of Kb (the CUDA-core column of the backward GEMM); zero past N_f.
struct TcConst {
    float sumk[kMaxFilters];
    float thl[kMaxFilters];
    float kbl[kMaxFilters];
};

struct TcArgs {
    K1Args k;                 // image geometry, slots, control, outputs (as K1)
    const float* bimg;        // [B_FLOATS] B operand images (hi/lo), built at model creation
    const float* sumk;        // [NP] sum_t k_i (fp64-summed, fp32) for the DC restore (0 past N_f)
    const float* theta_ln2;   // [NP] theta_i ln 2 (0 past N_f)
    int tiles_x;              // column tiles of OW
};

// expm1(t) in fp64 to ~1e-9 relative (fp32 staging needs 2^-25): t = n ln2 + r, |r| <= ln2/2,
// expm1(t) = 2^n expm1(r) + (2^n - 1), expm1(r) by its Taylor series to r^8 (remainder
// < 6e-10 relative); branch-free, no special cases (|t| < 700; a non-finite t propagates)
__device__ __forceinline__ double expm1_stage(double t) {
    const double n = rint(t * 1.4426950408889634);
    const double r = fma(-n, 6.93147180559945286e-01, t);
    double p = fma(r, 1.0 / 40320.0, 1.0 / 5040.0);
    p = fma(p, r, 1.0 / 720.0);
    p = fma(p, r, 1.0 / 120.0);
    p = fma(p, r, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p * r, r, r);
    const double s = __longlong_as_double((long long)((int)n + 1023) << 52);   // 2^n
    return fma(s, p, s - 1.0);
}
// one staged value u - c of the fp64 iterate x (w, or u for the u-domain model (6)), c = cst
// (the fp32 tile constant), ec = e^{wc} (fp64): ec expm1(x - wc) + (ec - c) in fp64, rounded once
// to fp32.  (An fp32 expm1 of the fp32-rounded difference was 2.5x less accurate: on c4 image 37
// the staging alone gave 2.9e-6 gradient error against 1.2e-6 rounded once, and K8's P2 update
// error crossed the 1e-5 bar.)
__device__ __forceinline__ float tc_stage_val(double x, bool udom, float cst, double wc, double ec) {
    if (udom) return (float)(x - (double)cst);
    return (float)fma(ec, expm1_stage(x - wc), ec - (double)cst);
}

// u tile staging (a2): UY rows x UX columns of u - c from the fp64 iterate, one warp per row at a
// time with all of a lane's loads of the row in flight; columns wrap periodically (their indices
// are the same for every row), rows wrap or come from the slab's ghost rows
template <int UY, int UX, int UP, int NWARPS>
__device__ __forceinline__ void tc_stage_u(float* us, const double* w, const double* halo, int H, int W, int y0,
                                           int x0, int c2, bool udom, float cst, double wc, int warp, int lane) {
    constexpr int NX = (UX + 31) / 32;
    const double ec = udom ? 0.0 : exp(wc);
    int gx[NX];
#pragma unroll
    for (int k = 0; k < NX; ++k) gx[k] = wrap_idx(x0 - c2 + lane + 32 * k, W);
    // FOE_STAGE_ROWS rows per warp in flight (all their loads issued before any exponential)
    constexpr int NRB = FOE_STAGE_ROWS;
    for (int uy0 = warp * NRB; uy0 < UY; uy0 += NWARPS * NRB) {
        double v[NRB][NX];
#pragma unroll
        for (int r = 0; r < NRB; ++r) {
            const int uy = uy0 + r;
            const int y = y0 - c2 + uy;
            const double* src;
            if (halo == nullptr) src = w + (size_t)wrap_idx(y, H) * W;
            else if (y < 0) src = halo + (size_t)(kHalo + y) * W;
            else if (y >= H) src = halo + (size_t)(kHalo + y - H) * W;
            else src = w + (size_t)y * W;
#pragma unroll
            for (int k = 0; k < NX; ++k) v[r][k] = (uy < UY && lane + 32 * k < UX) ? src[gx[k]] : wc;
        }
#pragma unroll
        for (int r = 0; r < NRB; ++r) {
            const int uy = uy0 + r;
            if (uy >= UY) break;
#pragma unroll
            for (int k = 0; k < NX; ++k) {
                const int ux = lane + 32 * k;
                if (ux < UX) us[uy * UP + ux] = tc_stage_val(v[r][k], udom, cst, wc, ec);
            }
        }
    }
}

// u tile staging of a PACKED tile: strip s (lanes [s SP, s SP + SP), SP = rem + 4C) holds the
// last rem output columns (x0r ..) of band band0 + s; columns past the strips and strips past
// the last band are filled with c (u - c = 0)
template <int UY, int UX, int UP, int NWARPS>
__device__ __forceinline__ void tc_stage_u_packed(float* us, const double* w, int H, int W, int R, int x0r, int c2,
                                                  int SP, int spt, int band0, int nbands, bool udom, float cst,
                                                  double wc, int warp, int lane) {
    constexpr int NX = (UX + 31) / 32;
    const double ec = udom ? 0.0 : exp(wc);
    int gx[NX], yb[NX];
    bool ok[NX];
#pragma unroll
    for (int k = 0; k < NX; ++k) {
        const int ux = lane + 32 * k, st = ux / SP, band = band0 + st;
        ok[k] = ux < UX && st < spt && band < nbands;
        gx[k] = wrap_idx(x0r - c2 + (ux - st * SP), W);
        yb[k] = band * R - c2;
    }
    for (int uy = warp; uy < UY; uy += NWARPS) {
        double v[NX];
#pragma unroll
        for (int k = 0; k < NX; ++k) v[k] = ok[k] ? w[(size_t)wrap_idx(yb[k] + uy, H) * W + gx[k]] : wc;
#pragma unroll
        for (int k = 0; k < NX; ++k) {
            const int ux = lane + 32 * k;
            if (ux < UX) us[uy * UP + ux] = tc_stage_val(v[k], udom, cst, wc, ec);
        }
    }
}

// ---- per-row thread work of K8, on compile-time chunk ranges (one call per warp group) ------
// im2col chunks [C0, C1) of 8 taps: U = u(window) - u_q split into tf32 hi / lo, to TMEM
template <int M, int UP, int C0, int C1>
__device__ __forceinline__ void tc_im2col(const float* up, float vc, uint32_t t_hi, uint32_t t_lo) {
#pragma unroll
    for (int c8 = C0; c8 < C1; ++c8) {
        float h[8], lo[8];
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
            const int t0 = c8 * 8 + e, t1 = t0 + 1;
            const float2 u2 = make_float2(t0 < M * M ? up[(t0 / M) * UP + (t0 % M)] : vc,
                                          t1 < M * M ? up[(t1 / M) * UP + (t1 % M)] : vc);
            const float2 v = __fadd2_rn(u2, make_float2(-vc, -vc));     // taps past m*m -> 0
            float2 hi2, lo2;
            tc::tf32_split2(v, hi2, lo2);
            h[e] = hi2.x; h[e + 1] = hi2.y;
            lo[e] = lo2.x; lo[e + 1] = lo2.y;
        }
        tc::tmem_st8(t_hi + c8 * 8, h);
        tc::tmem_st8(t_lo + c8 * 8, lo);
    }
}
// epilogue of filter chunks [F0, F1): r = R + u_q sum k; energy sum theta ln2 lg2(1 + r^2);
// P = r / (1 + r^2) (= rho'/2) split into tf32 hi / lo, to TMEM; zlast += P kb_last
template <int F0, int F1>
__device__ __forceinline__ float tc_epilogue(uint32_t t_d, uint32_t t_phi, uint32_t t_plo, float uq,
                                             const float* css, const float* ths, const float* kbl, float& zlast) {
    float r[(F1 - F0) * 8];
#pragma unroll
    for (int f8 = F0; f8 < F1; ++f8) {
        float* rr = r + (f8 - F0) * 8;
        tc::tmem_ld8(t_d + f8 * 8, *reinterpret_cast<float(*)[8]>(rr));
    }
    tc::wait_ld();
    // filters in pairs on the FP32x2 pipes (FFMA2 / FMUL2 / FADD2); MUFU stays scalar
    const float2 uq2 = make_float2(uq, uq), one2 = make_float2(1.f, 1.f);
    float2 el2 = make_float2(0.f, 0.f), zl2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int f8 = F0; f8 < F1; ++f8) {
        float ph[8], pl[8];
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
            const int i = f8 * 8 + e;
            const float2 r2 = make_float2(r[(f8 - F0) * 8 + e], r[(f8 - F0) * 8 + e + 1]);
            const float2 rv = __ffma2_rn(uq2, make_float2(css[i], css[i + 1]), r2);
            const float2 d = __ffma2_rn(rv, rv, one2);
            el2 = __ffma2_rn(make_float2(ths[i], ths[i + 1]), make_float2(lg2_approx(d.x), lg2_approx(d.y)), el2);
#if FOE_K8_PAIR_RCP
            // one MUFU reciprocal per filter pair: 1/d_A = d_B / (d_A d_B), 1/d_B = d_A / (d_A d_B)
            // (d >= 1; d_A d_B overflows only for |r| > ~4e9 -- u ~ 1e9 -- where rho'/2 ~ 1/r
            // flushes to 0; an infinite d (u past the w guard) makes the energy infinite, so the
            // trial is rejected either way)
            const float q = rcp_approx(d.x * d.y);
            const float2 pv = __fmul2_rn(rv, __fmul2_rn(make_float2(d.y, d.x), make_float2(q, q)));
#else
            const float2 pv = __fmul2_rn(rv, make_float2(rcp_approx(d.x), rcp_approx(d.y)));
#endif
            zl2 = __ffma2_rn(pv, make_float2(kbl[i], kbl[i + 1]), zl2);
            float2 hi2, lo2;
            tc::tf32_split2(pv, hi2, lo2);
            ph[e] = hi2.x; ph[e + 1] = hi2.y;
            pl[e] = lo2.x; pl[e + 1] = lo2.y;
        }
        tc::tmem_st8(t_phi + f8 * 8, ph);
        tc::tmem_st8(t_plo + f8 * 8, pl);
    }
    zlast = zl2.x + zl2.y;
    return el2.x + el2.y;
}
// Z chunks [C0, C1) of 8 taps -> zs[tap][lane]
template <int L, int C0, int C1>
__device__ __forceinline__ void tc_z_to_smem(uint32_t t_z, float* zs, int l) {
    float z[(C1 - C0) * 8];
#pragma unroll
    for (int c8 = C0; c8 < C1; ++c8) tc::tmem_ld8(t_z + c8 * 8, *reinterpret_cast<float(*)[8]>(z + (c8 - C0) * 8));
    tc::wait_ld();
#pragma unroll
    for (int k = 0; k < (C1 - C0) * 8; ++k) zs[(C0 * 8 + k) * L + l] = z[k];
}

template <int M, int NP, int R>
__global__ void __launch_bounds__(256, 2) k_prior_grad_tc(const TcArgs ta, const __grid_constant__ TcConst cc) {
    using G = TcGeom<M, NP, R>;
    constexpr int C = G::C, KT = G::KT, TAPS = G::TAPS, L = G::LANES;
    extern __shared__ __align__(128) float sm[];
    float* bsm = sm + G::SM_B;
    float* us = sm + G::SM_U;
    float* zs = sm + G::SM_Z;
    float* css = sm + G::SM_CS;
    float* ths = sm + G::SM_TH;
    __shared__ uint32_t tbase_s;
    __shared__ __align__(8) uint64_t mbar_f, mbar_b;   // forward / backward MMA completion
    __shared__ __align__(8) uint64_t mbar_bimg;        // TMA bulk copy of the B images
    __shared__ double red[32];

    const K1Args& args = ta.k;
    const int b = blockIdx.y;
    int wslot = 0, gslot = 0;
    if (args.ctl != nullptr) {
        const ImgCtl& c = args.ctl[b];
        if (!c.active) return;
        wslot = args.which_cur ? c.cur : c.cand;
        gslot = args.which_cur ? c.gcur : c.gcand;
    }
    const int H = args.H, W = args.W;
    const size_t HW = (size_t)H * W;
    const int tile = blockIdx.x;
    const double* w = args.w + (size_t)wslot * args.w_slot_stride + (size_t)b * HW;
    // warp index broadcast from lane 0: provably warp-uniform, so TMEM addresses and the warp
    // group branch stay in uniform registers (no per-op R2UR / collective fix-up code)
    const int t = threadIdx.x, warp = __shfl_sync(0xffffffffu, t >> 5, 0);
    const int wg = warp >> 2;                                   // warp group (0, 1)
    const int l = (warp & 3) * 32 + (t & 31);                   // TMEM lane = response pixel
    // tile geometry: a full tile (band ty, columns x0 ..), or a packed tile whose lane strips
    // carry the remainder columns of several bands (args.tc_rem > 0).  Per lane: its strip's
    // band origin sy0, its column ocol inside the strip / tile, and whether the strip exists.
    const int nbands = (H + R - 1) / R;
    const int nnorm = nbands * ta.tiles_x;
    const bool packed = tile >= nnorm;
    int y0, x0, sy0, ocol;
    bool svalid = true;
    const int SP = args.tc_rem + 4 * C;                         // strip pitch in lanes (packed)
    if (!packed) {
        const int ty = tile / ta.tiles_x, tx = tile - ty * ta.tiles_x;
        y0 = ty * R; x0 = tx * G::OW; sy0 = y0; ocol = l;
    } else {
        const int band0 = (tile - nnorm) * args.tc_spt;
        const int st = l / SP;
        ocol = l - st * SP;
        svalid = st < args.tc_spt && band0 + st < nbands;
        y0 = band0 * R; x0 = ta.tiles_x * G::OW; sy0 = (band0 + st) * R;
    }

    // ---- prologue: TMEM, mbarrier, B images, u tile ------------------------------------
    if (warp == 0) tc::tmem_alloc<G::TCOLS>(&tbase_s);
    if (t == 0) {
        tc::mbar_init(&mbar_f, 1);
        tc::mbar_init(&mbar_b, 1);
        tc::mbar_init(&mbar_bimg, 1);
        tc::mbar_fence_init();
        // the B images (taps, hi/lo, K-major) by one TMA bulk copy, overlapped with the u staging
        tc::bulk_g2s(bsm, ta.bimg, (uint32_t)(G::B_FLOATS * 4), &mbar_bimg);
    }
    const int yc = min(y0 + R / 2, H - 1), xc = min(x0 + (packed ? args.tc_rem : G::OW) / 2, W - 1);
    // u - c = c (e^{w - w_c} - 1) with c = e^{w_c} at a pixel of the tile: one fp64 exp per CTA,
    // then fp32 expm1 of the small fp64 difference -- accurate relative to u - c (what the
    // stencil needs), and far cheaper than K1's fp64 exp per staged pixel
    const bool udom = args.udom != 0;
    const double wc = w[(size_t)yc * W + xc];
    const float cst = (float)(udom ? wc : exp(wc));
    if (t < NP) {
        css[t] = __ldg(ta.sumk + t);
        ths[t] = __ldg(ta.theta_ln2 + t);
    }
    const double* halo = args.halo;
    if (!packed) tc_stage_u<G::UY, G::UX, G::UP, 8>(us, w, halo, H, W, y0, x0, 2 * C, udom, cst, wc, warp, t & 31);
    else tc_stage_u_packed<G::UY, G::UX, G::UP, 8>(us, w, H, W, R, x0, 2 * C, SP, args.tc_spt, y0 / R, nbands,
                                                   udom, cst, wc, warp, t & 31);
    tc::fence_proxy_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    tc::mbar_wait(&mbar_bimg, 0);   // B images landed (async proxy; read by the MMAs and kbl below)
    const uint32_t tb = tbase_s;
    const uint32_t tl = tb + ((uint32_t)((warp & 3) * 32) << 16);   // this warp's TMEM lane base
    const uint32_t idf = tc::idesc_tf32(128, NP);              // forward: N = filters
    const uint32_t idb = tc::idesc_tf32(128, G::NB);           // backward: N = taps [0, NB)
    const uint32_t b_base = tc::smem_u32(bsm);
    const float* kbl = bsm + 2 * G::BF_FLOATS + 2 * G::BB_FLOATS;   // last tap of Kb

    // energy ownership of this lane's response column, output column of this thread
    const int ow = packed ? args.tc_rem : G::OW;                // output columns of this lane's strip
    const bool col_own = svalid && (ocol >= C) && (ocol < C + ow) && (x0 - C + ocol < W);
    const bool out_col = svalid && (ocol < ow) && (x0 + ocol < W);   // output column ocol of the strip

    double e_acc = 0.0;
    // Two warp groups share every row: wg 0 takes the first half of the tap chunks (im2col,
    // Z), filters (epilogue) and filter rows a < C+1 (col2im); wg 1 the rest.  Warp w reaches
    // TMEM lanes 32 (w % 4) .. +31, so both groups cover all 128 pixels.
    constexpr int NC8 = KT / 8, H8 = (NC8 + 1) / 2;        // im2col tap chunks: wg0 [0,H8), wg1 [H8,NC8)
    constexpr int NZ8 = G::NB / 8, HZ8 = (NZ8 + 1) / 2;    // Z tap chunks: wg0 [0,HZ8), wg1 [HZ8,NZ8)
    constexpr int NF8 = NP / 8, HF8 = NF8 / 2;             // filter chunks: wg0 [0,HF8), wg1 [HF8,NF8)
    constexpr int A0 = C + 1, A1 = M - A0;                 // col2im rows: wg0 a < A0, wg1 a >= A0
    float acc[A0 > A1 ? A0 : A1];
#pragma unroll
    for (int k = 0; k < (A0 > A1 ? A0 : A1); ++k) acc[k] = 0.f;
    float* gout = args.g + (size_t)gslot * args.g_slot_stride + (size_t)b * HW;
    float* hand = sm + G::SM_HAND;                         // [8][L] wg0 -> wg1 partial sums
    float* zls = sm + G::SM_ZL;                            // [2 rows][2 groups][L] last-tap partials

    // Software pipeline over response rows (iteration j):
    //   im2col(j) | wait MMAb(j-1), Z(j-1) -> smem | sync | issue MMAf(j) |
    //   col2im(j-1) (overlaps MMAf(j)) | wait MMAf(j), epilogue(j) | sync | issue MMAb(j)
    // MMAb(j) then runs under the next iteration's im2col.  Z(j) lands in D's columns (D is
    // consumed by epilogue(j) before MMAb(j) is issued; MMAf(j+1) is issued after Z(j) is read).
#pragma unroll 1
    for (int j = 0; j <= G::RR; ++j) {
        float uq = 0.f;
        if (j < G::RR) {
            // (a2, a3) im2col of response pixel (row j, lane l): taps a*M + b minus the window
            // centre u_q (per-pixel DC shift: K(u - u_q) + u_q sum k = K u)
            const float* up = us + j * G::UP + l;
            const float vc = up[C * G::UP + C];
            uq = vc + cst;
            if (wg == 0) tc_im2col<M, G::UP, 0, H8>(up, vc, tl + G::COL_AHI, tl + G::COL_ALO);
            else tc_im2col<M, G::UP, H8, NC8>(up, vc, tl + G::COL_AHI, tl + G::COL_ALO);
        }
        if (j > 0) {
            tc::mbar_wait(&mbar_b, (uint32_t)((j - 1) & 1));
            tc::fence_after_sync();
            if (wg == 0) tc_z_to_smem<L, 0, HZ8>(tl + G::COL_Z, zs, l);
            else tc_z_to_smem<L, HZ8, NZ8>(tl + G::COL_Z, zs, l);
        }
        tc::wait_st();
        tc::fence_before_sync();
        __syncthreads();
        if (warp == 0 && j < G::RR) {
            tc::fence_after_sync();
            // the small cross terms first, then hi.hi: the fp32 accumulator loses less of them
#pragma unroll
            for (int s = 0; s < NC8; ++s) {
                const uint32_t off = (uint32_t)(s * 2 * NP * 16);
                const uint64_t bh = tc::sdesc_kmajor(b_base + off, NP * 16, 128);
                const uint64_t bl = tc::sdesc_kmajor(b_base + G::BF_FLOATS * 4 + off, NP * 16, 128);
                tc::mma_tf32_ts_warp(tb + G::COL_D, tb + G::COL_AHI + s * 8, bl, idf, s > 0);
                tc::mma_tf32_ts_warp(tb + G::COL_D, tb + G::COL_ALO + s * 8, bh, idf, 1);
            }
#pragma unroll
            for (int s = 0; s < NC8; ++s) {
                const uint32_t off = (uint32_t)(s * 2 * NP * 16);
                const uint64_t bh = tc::sdesc_kmajor(b_base + off, NP * 16, 128);
                tc::mma_tf32_ts_warp(tb + G::COL_D, tb + G::COL_AHI + s * 8, bh, idf, 1);
            }
            tc::mma_commit_warp(&mbar_f);
        }
        if (j > 0) {
            // col2im of row jz = j - 1: Z row jz feeds output rows o = jz - a at column ox = l:
            //   s[o][ox] += sum_b Z[(jz, ox + b), (a, b)];  acc[k] holds row jz - (a0 + k)
            const int jz = j - 1;
            if (wg == 0) {
                // two filter rows per FP32x2 add (a, a + 1)
#pragma unroll
                for (int a = 0; a + 1 < A0; a += 2) {
                    float2 sa = make_float2(0.f, 0.f);
#pragma unroll
                    for (int bb = 0; bb < M; ++bb)
                        sa = __fadd2_rn(sa, make_float2(zs[(a * M + bb) * L + l + bb], zs[((a + 1) * M + bb) * L + l + bb]));
                    acc[a] += sa.x;
                    acc[a + 1] += sa.y;
                }
                if constexpr (A0 % 2 == 1) {
                    float sa = 0.f;
#pragma unroll
                    for (int bb = 0; bb < M; ++bb) sa += zs[((A0 - 1) * M + bb) * L + l + bb];
                    acc[A0 - 1] += sa;
                }
                const int o = jz - (A0 - 1);                    // wg0's share of row o is complete
                if (o >= 0) hand[(o & 7) * L + l] = acc[A0 - 1];
#pragma unroll
                for (int k = A0 - 1; k > 0; --k) acc[k] = acc[k - 1];
                acc[0] = 0.f;
            } else {
                const float* zl = zls + (jz & 1) * 2 * L;
                // rows A0 .. M-2 in FP32x2 pairs (all their taps are in Z), the last row (it holds
                // the CUDA-core tap) scalar
                constexpr int NPR = (A1 - 1) / 2;
#pragma unroll
                for (int q = 0; q < NPR; ++q) {
                    const int a = A0 + 2 * q;
                    float2 sa = make_float2(0.f, 0.f);
#pragma unroll
                    for (int bb = 0; bb < M; ++bb)
                        sa = __fadd2_rn(sa, make_float2(zs[(a * M + bb) * L + l + bb], zs[((a + 1) * M + bb) * L + l + bb]));
                    acc[2 * q] += sa.x;
                    acc[2 * q + 1] += sa.y;
                }
#pragma unroll
                for (int k = 2 * NPR; k < A1; ++k) {
                    const int a = A0 + k;
                    float sa = 0.f;
#pragma unroll
                    for (int bb = 0; bb < M; ++bb) {
                        const int tap = a * M + bb;
                        sa += tap < G::NB ? zs[tap * L + l + bb] : zl[l + bb] + zl[L + l + bb];
                    }
                    acc[k] += sa;
                }
                // (a6) row o = jz - 2C is complete: g = u (.) s
                const int o = jz - 2 * C;
                if (o >= 0 && o < R && out_col && sy0 + o < H) {
                    const float s_tot = acc[A1 - 1] + hand[(o & 7) * L + l];
                    const float u = udom ? 1.0f : us[(o + 2 * C) * G::UP + l + 2 * C] + cst;   // W = diag(e^w)
                    gout[(size_t)(sy0 + o) * W + x0 + ocol] = u * s_tot;
                }
#pragma unroll
                for (int k = A1 - 1; k > 0; --k) acc[k] = acc[k - 1];
                acc[0] = 0.f;
            }
        }
        if (j < G::RR) {
            tc::mbar_wait(&mbar_f, (uint32_t)(j & 1));
            tc::fence_after_sync();
            // (a4, a7) responses r = R + u_q sum k, rho (owned responses), rho'/2 -> P (hi/lo)
            const bool own = col_own && (j >= C) && (j < C + R) && (sy0 - C + j < H);
            float zl;
            const float el = wg == 0
                ? tc_epilogue<0, HF8>(tl + G::COL_D, tl + G::COL_PHI, tl + G::COL_PLO, uq, cc.sumk, cc.thl, cc.kbl, zl)
                : tc_epilogue<HF8, NF8>(tl + G::COL_D, tl + G::COL_PHI, tl + G::COL_PLO, uq, cc.sumk, cc.thl, cc.kbl, zl);
            zls[(j & 1) * 2 * L + wg * L + l] = zl;
            if (own) e_acc += (double)el;
            tc::wait_st();
            tc::fence_before_sync();
            __syncthreads();
            if (warp == 0) {
                tc::fence_after_sync();
#pragma unroll
                for (int s = 0; s < NF8; ++s) {
                    const uint32_t off = (uint32_t)(s * 2 * G::NB * 16);
                    const uint64_t bh = tc::sdesc_kmajor(b_base + 2 * G::BF_FLOATS * 4 + off, G::NB * 16, 128);
                    const uint64_t bl = tc::sdesc_kmajor(b_base + (2 * G::BF_FLOATS + G::BB_FLOATS) * 4 + off,
                                                         G::NB * 16, 128);
                    tc::mma_tf32_ts_warp(tb + G::COL_Z, tb + G::COL_PHI + s * 8, bl, idb, s > 0);
                    tc::mma_tf32_ts_warp(tb + G::COL_Z, tb + G::COL_PLO + s * 8, bh, idb, 1);
                }
#pragma unroll
                for (int s = 0; s < NF8; ++s) {
                    const uint32_t off = (uint32_t)(s * 2 * G::NB * 16);
                    const uint64_t bh = tc::sdesc_kmajor(b_base + 2 * G::BF_FLOATS * 4 + off, G::NB * 16, 128);
                    tc::mma_tf32_ts_warp(tb + G::COL_Z, tb + G::COL_PHI + s * 8, bh, idb, 1);
                }
                tc::mma_commit_warp(&mbar_b);
            }
        }
    }
    // (a7) per-CTA energy partial (fixed order)
    const double e = block_sum_d(e_acc, red);
    if (t == 0) args.epart[(size_t)b * args.ntiles * args.groups + blockIdx.x] = e;
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<G::TCOLS>(tb);
}

}  // namespace foe
