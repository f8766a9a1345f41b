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
    int nimg;                 // images in the batch (persistent variant: grid = min(items, SMs))
    // fused trial (K2 inside K8's staging, FUSED instantiation): f~, the test partials
    // [B][ntiles][8] of the tile's owned pixels, and the solver parameters
    const float* ft;
    double* ppart;
    SolverParams sp;
};

// u tile staging (a2): UY rows x UX columns of u - c from the fp64 iterate, one warp per row at a
// time with all of a lane's loads of the row in flight; columns wrap periodically (their indices
// are the same for every row), rows wrap or come from the slab's ghost rows
template <int UY, int UX, int UP, int NWARPS>
__device__ __forceinline__ void tc_stage_u(float* us, const double* w, const double* halo, int H, int W, int y0,
                                           int x0, int c2, bool udom, float cst, double wc, int warp, int lane) {
    constexpr int NX = (UX + 31) / 32;
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
                if (ux < UX) us[uy * UP + ux] = udom ? (float)(v[r][k] - (double)cst) : cst * expm1f((float)(v[r][k] - wc));
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
            if (ux < UX) us[uy * UP + ux] = udom ? (float)(v[k] - (double)cst) : cst * expm1f((float)(v[k] - wc));
        }
    }
}

// Fused trial staging (K2 inside K8, rows a8-a10 on the staged pixels): for every staged pixel
// the inertial point and prox of K2 (k2_pixel, the same arithmetic as k_inertial_prox) give w+,
// staged as u+ - c; pixels the tile owns store w+ and enter the test partials.  Column
// geometry per lane slot k: image column gx, unwrapped row origin yb (band - 2C), strip origin
// (ownership window [ox0, ox1) in unwrapped columns, rows [oy0, oy1)).
struct FuseCtx {
    const double *w, *wp;
    double* wn;
    const float *g, *ft;
    double alpha, beta, l1, l2;
};
template <int UY, int UX, int UP, int NWARPS>
__device__ __forceinline__ void tc_stage_fused(float* us, const FuseCtx& fc, const SolverParams& sp, int idiv, int H,
                                               int W, const int (&gx)[(UX + 31) / 32], const int (&yb)[(UX + 31) / 32],
                                               const bool (&ok)[(UX + 31) / 32], const bool (&cown)[(UX + 31) / 32],
                                               const int (&oy0)[(UX + 31) / 32], float cst, double wc, int warp,
                                               int lane, int R, K2Acc& acc) {
    constexpr int NX = (UX + 31) / 32;
    for (int uy = warp; uy < UY; uy += NWARPS) {
        double wv[NX], wpv[NX];
        float gv[NX], fv[NX];
        size_t pix[NX];
#pragma unroll
        for (int k = 0; k < NX; ++k) {
            pix[k] = (size_t)wrap_idx(yb[k] + uy, H) * W + gx[k];
            wv[k] = ok[k] ? fc.w[pix[k]] : wc;
            wpv[k] = ok[k] ? fc.wp[pix[k]] : wc;
            gv[k] = ok[k] ? fc.g[pix[k]] : 0.f;
            fv[k] = ok[k] ? fc.ft[pix[k]] : 1.f;
        }
#pragma unroll
        for (int k = 0; k < NX; ++k) {
            const int ux = lane + 32 * k;
            if (ux >= UX) continue;
            float val = 0.f;
            if (ok[k]) {
                const int yu = yb[k] + uy;                     // unwrapped image row
                const bool own = cown[k] && yu >= oy0[k] && yu < oy0[k] + R && yu < H;
                const double z = k2_pixel(wv[k], wpv[k], (double)gv[k], (double)fv[k], fc.alpha, fc.beta, fc.l1,
                                          fc.l2, sp, idiv, acc, own);
                if (own) fc.wn[pix[k]] = z;
                val = idiv ? (float)(z - (double)cst) : cst * expm1f((float)(z - wc));
            }
            us[uy * UP + ux] = val;
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

// FUSED: one trial in one kernel -- K2 (inertial point + prox + test partials) on the staged
// pixels, then the prior energy + gradient at the candidate (ctl required, evaluates ctl.cand)
template <int M, int NP, int R, bool FUSED = false>
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
    FuseCtx fc{};
    if constexpr (FUSED) {
        const ImgCtl& c = args.ctl[b];
        fc.w = args.w + (size_t)c.cur * args.w_slot_stride + (size_t)b * HW;
        fc.wp = args.w + (size_t)c.prev * args.w_slot_stride + (size_t)b * HW;
        fc.wn = const_cast<double*>(args.w) + (size_t)c.cand * args.w_slot_stride + (size_t)b * HW;
        fc.g = args.g + (size_t)c.gcur * args.g_slot_stride + (size_t)b * HW;
        fc.ft = ta.ft + (size_t)b * HW;
        fc.alpha = ta.sp.safety * 2.0 * (1.0 - ta.sp.beta) / c.L;
        fc.beta = ta.sp.beta;
        fc.l1 = c.lam1;
        fc.l2 = c.lam2;
    }
    __shared__ double zc_s;
    if constexpr (FUSED) {
        if (t == 0) {   // the DC centre's w+ (the same k2_pixel as its staged copy)
            K2Acc dummy;
            const size_t pc = (size_t)yc * W + xc;
            zc_s = k2_pixel(fc.w[pc], fc.wp[pc], (double)fc.g[pc], (double)fc.ft[pc], fc.alpha, fc.beta, fc.l1, fc.l2,
                            ta.sp, udom, dummy, false);
        }
        __syncthreads();
    }
    const double wc = FUSED ? zc_s : w[(size_t)yc * W + xc];
    const float cst = (float)(udom ? wc : exp(wc));
    if constexpr (FUSED) {
        constexpr int NX = (G::UX + 31) / 32;
        int gx[NX], yb[NX], oy0[NX];
        bool ok[NX], cown[NX];
        const int lane = t & 31;
#pragma unroll
        for (int k = 0; k < NX; ++k) {
            const int ux = lane + 32 * k;
            if (!packed) {
                const int xu = x0 - 2 * C + ux;
                ok[k] = ux < G::UX;
                gx[k] = wrap_idx(xu, W);
                yb[k] = y0 - 2 * C;
                oy0[k] = y0;
                cown[k] = xu >= x0 && xu < x0 + G::OW && xu < W;
            } else {
                const int st = ux / SP, band = y0 / R + st;
                const int xu = x0 - 2 * C + (ux - st * SP);
                ok[k] = ux < G::UX && st < args.tc_spt && band < nbands;
                gx[k] = wrap_idx(xu, W);
                yb[k] = band * R - 2 * C;
                oy0[k] = band * R;
                cown[k] = xu >= x0 && xu < W;
            }
        }
        K2Acc acc;
        tc_stage_fused<G::UY, G::UX, G::UP, 8>(us, fc, ta.sp, udom, H, W, gx, yb, ok, cown, oy0, cst, wc, warp, lane, R,
                                               acc);
        __syncthreads();
        k2_block_partials(acc, ta.ppart + ((size_t)b * args.ntiles + blockIdx.x) * kNumPart);
    }
    if (t < NP) {
        css[t] = __ldg(ta.sumk + t);
        ths[t] = __ldg(ta.theta_ln2 + t);
    }
    const double* halo = args.halo;
    if constexpr (!FUSED) {
        if (!packed) tc_stage_u<G::UY, G::UX, G::UP, 8>(us, w, halo, H, W, y0, x0, 2 * C, udom, cst, wc, warp, t & 31);
        else tc_stage_u_packed<G::UY, G::UX, G::UP, 8>(us, w, H, W, R, x0, 2 * C, SP, args.tc_spt, y0 / R, nbands,
                                                       udom, cst, wc, warp, t & 31);
    }
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

namespace foe {

// =============================================================================================
// K8 v4: the same computation, warp-specialised so that the rows of a tile flow through a
// pipeline instead of a lock-step loop (one CTA per SM, 512 TMEM columns):
//
//   IM  warps 0-7   im2col of row j into A[j%2]                    (waits A_empty: MMAf(j-2) done)
//   MMA warp 20     MMAf(j): A[j%2] -> D[j%2]; MMAb(j-1): P -> Z(j-1) in D[(j-1)%2]
//   EP  warps 8-15  rho, rho' of row j from D[j%2] -> P, last-tap partial -> TMEM (zl[j%2])
//                   (waits D_full[j%2]; writes P after P_empty: MMAb(j-1) done)
//   ZC  warps 16-19 Z(j) -> smem, col2im, g rows                   (waits Z_full[j%2])
//
// mbarriers: A_full[2] (8 IM warps), A_empty[2] / D_full[2] / Z_full[2] / P_empty (tcgen05
// commits), P_full (8 EP warps), D_empty[2] (4 ZC warps).  Parity of the k-th completion of a
// two-slot barrier is (k & 1) with k = j / 2; of a one-slot barrier, j & 1.
// =============================================================================================
// v4 epilogue math for one half of the filters (HALF), from the D row in TMEM
template <int NP, int HALF>
__device__ __forceinline__ void tc4_ep_half(uint32_t t_d, float uq, const TcConst& cc, float& el, float& zl,
                                            float (&ph)[NP / 2], float (&pl)[NP / 2], bool knockout) {
    constexpr int HF = NP / 2;
    float r[HF];
    tc::tmem_ld16(t_d + HALF * HF, *reinterpret_cast<float(*)[16]>(r));
    if constexpr (HF > 16) tc::tmem_ld8(t_d + HALF * HF + 16, *reinterpret_cast<float(*)[8]>(r + 16));
    tc::wait_ld();
    el = 0.f;
    zl = 0.f;
#pragma unroll
    for (int e = 0; e < HF; ++e) {
        if (knockout) { ph[e] = r[e]; pl[e] = 0.f; continue; }
        const int i = HALF * HF + e;
        const float rv = fmaf(uq, cc.sumk[i], r[e]);
        const float d = fmaf(rv, rv, 1.f);
        el = fmaf(cc.thl[i], lg2_approx(d), el);
        const float pv = rv * rcp_approx(d);
        zl = fmaf(pv, cc.kbl[i], zl);
        ph[e] = tc::tf32_hi(pv);
        pl[e] = tc::tf32_hi(pv - ph[e]);
    }
}

template <int M, int NP, int R>
struct Tc4Geom {
    using B = TcGeom<M, NP, R>;
    static constexpr int KT = B::KT, NB = B::NB, TAPS = B::TAPS, LANES = 128;
    // TMEM columns
    static constexpr int ND = 3;                     // D / Z ring depth
    static constexpr int COL_A0 = 0;                 // A[s]: hi [s*2KT, s*2KT+KT), lo [+KT, +2KT)
    static constexpr int COL_D0 = 4 * KT;            // D[s] at COL_D0 + s*NP, s = j % ND (Z(j) reuses it)
    static constexpr int COL_P = COL_D0 + ND * NP;   // P hi [COL_P, +NP), lo [+NP, +2NP)
    static constexpr int COL_ZL = COL_P + 2 * NP;    // last-tap partials: [slot][half] (2 ND columns)
    static constexpr int TCOLS_USED = COL_ZL + 2 * ND;
    static_assert(TCOLS_USED <= 512, "TMEM budget");
    // shared memory (floats): B images | u tile | Zs[2][TAPS][LANES] | sum k | theta ln2
    static constexpr int SM_B = 0;
    static constexpr int SM_U = B::B_FLOATS;
    static constexpr int SM_Z = SM_U + B::UY * B::UP;
    static constexpr int SM_CS = SM_Z + 2 * TAPS * LANES;
    static constexpr int SM_TH = SM_CS + NP;
    static constexpr int SM_FLOATS = SM_TH + NP;
    static constexpr int SMEM_BYTES = SM_FLOATS * 4 + 64;
    static constexpr int THREADS = 21 * 32;      // 8 IM + 8 EP + 4 ZC + 1 MMA warps
};

// KO (profiling only, never selected by the library's API): 0 = full kernel; 1/2/3/4 skip the
// work of IM / EP / ZC / the MMAs (barriers kept) to find the pipeline's limiting role.
template <int M, int NP, int R, int KO = 0>
__global__ void __launch_bounds__(21 * 32, 1) k_prior_grad_tc4(const TcArgs ta, const __grid_constant__ TcConst cc) {
    using G = TcGeom<M, NP, R>;
    using G4 = Tc4Geom<M, NP, R>;
    constexpr int C = G::C, KT = G::KT, TAPS = G::TAPS, L = G::LANES, NB = G::NB;
    extern __shared__ __align__(128) float sm[];
    float* bsm = sm + G4::SM_B;
    float* us = sm + G4::SM_U;
    float* zs = sm + G4::SM_Z;
    float* css = sm + G4::SM_CS;
    float* ths = sm + G4::SM_TH;
    __shared__ uint32_t tbase_s;
    constexpr int ND = G4::ND;
    __shared__ __align__(8) uint64_t bar_afull[2], bar_aempty[2], bar_dfull[ND], bar_dempty[ND], bar_zfull[ND];
    __shared__ __align__(8) uint64_t bar_pfull, bar_pempty;
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
    const int ty = tile / ta.tiles_x, tx = tile - ty * ta.tiles_x;
    const int y0 = ty * R, x0 = tx * G::OW;
    const double* w = args.w + (size_t)wslot * args.w_slot_stride + (size_t)b * HW;
    const int t = threadIdx.x, warp = __shfl_sync(0xffffffffu, t >> 5, 0), lane = t & 31;   // warp-uniform
    const int l = (warp & 3) * 32 + lane;                       // TMEM lane = response pixel
    const bool udom = args.udom != 0;

    // ---- prologue (all warps): TMEM, barriers, B images, u tile ------------------------------
    if (warp == 0) tc::tmem_alloc<512>(&tbase_s);
    if (t == 0) {
        for (int s = 0; s < 2; ++s) {
            tc::mbar_init(&bar_afull[s], 8);
            tc::mbar_init(&bar_aempty[s], 1);
        }
        for (int s = 0; s < ND; ++s) {
            tc::mbar_init(&bar_dfull[s], 1);
            tc::mbar_init(&bar_dempty[s], 4);
            tc::mbar_init(&bar_zfull[s], 1);
        }
        tc::mbar_init(&bar_pfull, 8);
        tc::mbar_init(&bar_pempty, 1);
        tc::mbar_fence_init();
    }
    {
        const float4* src = reinterpret_cast<const float4*>(ta.bimg);
        float4* dst = reinterpret_cast<float4*>(bsm);
        for (int i = t; i < G::B_FLOATS / 4; i += G4::THREADS) dst[i] = __ldg(src + i);
    }
    const int yc = min(y0 + R / 2, H - 1), xc = min(x0 + G::OW / 2, W - 1);
    const double wc = w[(size_t)yc * W + xc];
    const float cst = (float)(udom ? wc : exp(wc));
    if (t < NP) {
        css[t] = __ldg(ta.sumk + t);
        ths[t] = __ldg(ta.theta_ln2 + t);
    }
    const double* halo = args.halo;
    tc_stage_u<G::UY, G::UX, G::UP, G4::THREADS / 32>(us, w, halo, H, W, y0, x0, 2 * C, udom, cst, wc, warp, lane);
    tc::fence_proxy_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tb = tbase_s;
    const uint32_t tl = tb + ((uint32_t)((warp & 3) * 32) << 16);
    double e_acc = 0.0;

    if (warp < 8) {
        // ================================ IM: im2col ================================
        // two warp groups: taps chunks [0, H8) and [H8, KT/8)
        constexpr int H8 = (KT / 8 + 1) / 2;
        const int ig = warp >> 2;
#pragma unroll 1
        for (int j = 0; j < G::RR; ++j) {
            const int s = j & 1;
            if (j >= 2) {
                tc::mbar_wait(&bar_aempty[s], (uint32_t)(((j >> 1) - 1) & 1));
                tc::fence_after_sync();
            }
            const float* up = us + j * G::UP + l;
            const float vc = up[C * G::UP + C];
            const uint32_t a_hi = tl + G4::COL_A0 + s * 2 * KT, a_lo = a_hi + KT;
            if (KO != 1) {
                if (ig == 0) tc_im2col<M, G::UP, 0, H8>(up, vc, a_hi, a_lo);
                else tc_im2col<M, G::UP, H8, KT / 8>(up, vc, a_hi, a_lo);
            }
            tc::wait_st();
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&bar_afull[s]);
        }
    } else if (warp < 16) {
        // ================================ EP: rho, rho' =============================
        const int half = (warp - 8) >> 2;                   // filters [half*NP/2, (half+1)*NP/2)
        const int lx = x0 - C + l;
        const bool col_own = (l >= C) && (l < C + G::OW) && (lx < W);
#pragma unroll 1
        for (int j = 0; j < G::RR; ++j) {
            const int s = j % ND;
            tc::mbar_wait(&bar_dfull[s], (uint32_t)((j / ND) & 1));
            tc::fence_after_sync();
            const float uq = us[(j + C) * G::UP + l + C] + cst;   // window centre u_q (DC restore)
            constexpr int HF = NP / 2;
            float el, zl, ph[HF], pl[HF];
            if (half == 0) tc4_ep_half<NP, 0>(tl + G4::COL_D0 + s * NP, uq, cc, el, zl, ph, pl, KO == 2);
            else tc4_ep_half<NP, 1>(tl + G4::COL_D0 + s * NP, uq, cc, el, zl, ph, pl, KO == 2);
            const bool own = col_own && (j >= C) && (j < C + R) && (y0 - C + j < H);
            if (own) e_acc += (double)el;
            if (j >= 1) {                                       // P is free once MMAb(j-1) is done
                tc::mbar_wait(&bar_pempty, (uint32_t)((j - 1) & 1));
                tc::fence_after_sync();
            }
#pragma unroll
            for (int c8 = 0; c8 < HF / 8; ++c8) {
                tc::tmem_st8(tl + G4::COL_P + half * HF + c8 * 8, *reinterpret_cast<float(*)[8]>(ph + c8 * 8));
                tc::tmem_st8(tl + G4::COL_P + NP + half * HF + c8 * 8, *reinterpret_cast<float(*)[8]>(pl + c8 * 8));
            }
            tc::tmem_st1(tl + G4::COL_ZL + s * 2 + half, zl);
            tc::wait_st();
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&bar_pfull);
        }
    } else if (warp < 20) {
        // ================================ ZC: Z, col2im, g ==========================
        float acc[M];
#pragma unroll
        for (int k = 0; k < M; ++k) acc[k] = 0.f;
        float* gout = args.g + (size_t)gslot * args.g_slot_stride + (size_t)b * HW;
        const bool out_col = (l < G::OW) && (x0 + l < W);
#pragma unroll 1
        for (int j = 0; j < G::RR; ++j) {
            const int s = j % ND, zb = j & 1;
            tc::mbar_wait(&bar_zfull[s], (uint32_t)((j / ND) & 1));
            tc::fence_after_sync();
            static_assert(NB == 48 || NB == 24 || NB == 8, "Z readout shapes");
            float z[NB < 32 ? 32 : NB];
            if constexpr (NB == 48) {
                tc::tmem_ld32(tl + G4::COL_D0 + s * NP, z);
                tc::tmem_ld16(tl + G4::COL_D0 + s * NP + 32, *reinterpret_cast<float(*)[16]>(z + 32));
            } else if constexpr (NB == 24) {
                tc::tmem_ld16(tl + G4::COL_D0 + s * NP, *reinterpret_cast<float(*)[16]>(z));
                tc::tmem_ld8(tl + G4::COL_D0 + s * NP + 16, *reinterpret_cast<float(*)[8]>(z + 16));
            } else {
                tc::tmem_ld8(tl + G4::COL_D0 + s * NP, *reinterpret_cast<float(*)[8]>(z));
            }
            float zl0, zl1;
            tc::tmem_ld2(tl + G4::COL_ZL + s * 2, zl0, zl1);
            tc::wait_ld();
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&bar_dempty[s]);   // D[s] may take MMAf(j+2)
            float* zr = zs + zb * TAPS * L;
            if (KO == 3) { acc[0] += z[0] + zl0 + zl1; continue; }
#pragma unroll
            for (int k = 0; k < NB; ++k) zr[k * L + l] = z[k];
            zr[NB * L + l] = zl0 + zl1;
            tc::named_sync(1, 128);
            // col2im of row j: output rows o = j - a; acc[a] holds row j - a (shifted each row)
#pragma unroll
            for (int a = 0; a < M; ++a) {
                float sa = 0.f;
#pragma unroll
                for (int bb = 0; bb < M; ++bb) sa += zr[(a * M + bb) * L + l + bb];
                acc[a] += sa;
            }
            const int o = j - 2 * C;
            if (o >= 0 && o < R && out_col && y0 + o < H) {
                const float u = udom ? 1.0f : us[(o + 2 * C) * G::UP + l + 2 * C] + cst;   // W = diag(e^w)
                gout[(size_t)(y0 + o) * W + x0 + l] = u * acc[M - 1];
            }
#pragma unroll
            for (int k = M - 1; k > 0; --k) acc[k] = acc[k - 1];
            acc[0] = 0.f;
        }
    } else {
        // ================================ MMA issuer (whole warp; one elected lane issues) ===
        const uint32_t idf = tc::idesc_tf32(128, NP), idb = tc::idesc_tf32(128, NB);
        const uint32_t b_base = tc::smem_u32(bsm);
#pragma unroll 1
        for (int j = 0; j <= G::RR; ++j) {
            if (j < G::RR) {
                const int s = j & 1, sd = j % ND;
                tc::mbar_wait(&bar_afull[s], (uint32_t)((j >> 1) & 1));
                if (j >= ND) tc::mbar_wait(&bar_dempty[sd], (uint32_t)(((j / ND) - 1) & 1));
                tc::fence_after_sync();
                const uint32_t a_hi = tb + G4::COL_A0 + s * 2 * KT, a_lo = a_hi + KT, d = tb + G4::COL_D0 + sd * NP;
#pragma unroll
                for (int k = 0; k < KT / 8; ++k) {
                    const uint32_t off = (uint32_t)(k * 2 * NP * 16);
                    const uint64_t bh = tc::sdesc_kmajor(b_base + off, NP * 16, 128);
                    const uint64_t bl = tc::sdesc_kmajor(b_base + G::BF_FLOATS * 4 + off, NP * 16, 128);
                    if (KO != 4) tc::mma_tf32_ts_warp(d, a_hi + k * 8, bl, idf, k > 0);
                    if (KO != 4) tc::mma_tf32_ts_warp(d, a_lo + k * 8, bh, idf, 1);
                }
#pragma unroll
                for (int k = 0; k < KT / 8; ++k) {
                    const uint64_t bh = tc::sdesc_kmajor(b_base + (uint32_t)(k * 2 * NP * 16), NP * 16, 128);
                    if (KO != 4) tc::mma_tf32_ts_warp(d, a_hi + k * 8, bh, idf, 1);
                }
                tc::mma_commit_warp(&bar_aempty[s]);
                tc::mma_commit_warp(&bar_dfull[sd]);
            }
            if (j >= 1) {
                const int jb = j - 1, s = jb % ND;
                tc::mbar_wait(&bar_pfull, (uint32_t)(jb & 1));
                tc::fence_after_sync();
                const uint32_t z = tb + G4::COL_D0 + s * NP, p_hi = tb + G4::COL_P, p_lo = p_hi + NP;
#pragma unroll
                for (int k = 0; k < NP / 8; ++k) {
                    const uint32_t off = (uint32_t)(k * 2 * NB * 16);
                    const uint64_t bh = tc::sdesc_kmajor(b_base + 2 * G::BF_FLOATS * 4 + off, NB * 16, 128);
                    const uint64_t bl = tc::sdesc_kmajor(b_base + (2 * G::BF_FLOATS + G::BB_FLOATS) * 4 + off,
                                                         NB * 16, 128);
                    if (KO != 4) tc::mma_tf32_ts_warp(z, p_hi + k * 8, bl, idb, k > 0);
                    if (KO != 4) tc::mma_tf32_ts_warp(z, p_lo + k * 8, bh, idb, 1);
                }
#pragma unroll
                for (int k = 0; k < NP / 8; ++k) {
                    const uint64_t bh = tc::sdesc_kmajor(b_base + 2 * G::BF_FLOATS * 4 + (uint32_t)(k * 2 * NB * 16),
                                                         NB * 16, 128);
                    if (KO != 4) tc::mma_tf32_ts_warp(z, p_hi + k * 8, bh, idb, 1);
                }
                tc::mma_commit_warp(&bar_pempty);
                tc::mma_commit_warp(&bar_zfull[s]);
            }
        }
    }
    // (a7) per-CTA energy partial (fixed order over all threads; only EP threads contribute)
    __syncwarp();
    const double e = block_sum_d(e_acc, red);
    if (t == 0) args.epart[(size_t)b * args.ntiles * args.groups + blockIdx.x] = e;
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<512>(tb);
}

}  // namespace foe

namespace foe {

// =============================================================================================
// K8 v5: the v4 pipeline made persistent -- one CTA per SM loops over (tile, image) work items
// (static stride), so the B images are loaded once per CTA, the pipeline runs on across item
// boundaries (no fill/drain per tile), and a loader warp group stages the next item's u tile
// into a second buffer while the current one is processed:
//
//   IM  warps 0-7, EP 8-15, ZC 16-19, MMA 20 (as v4); LD warps 21-24: u tile of item k into
//   U[k%2] (waits U_empty[k%2]: ZC finished item k-2), arrives U_full[k%2].
//
// Rows are counted globally over the CTA's items (r), so every ring barrier keeps its parity
// arithmetic; per-item energies are reduced over the 8 EP warps (named barrier 2).
// =============================================================================================
template <int M, int NP, int R>
struct Tc5Geom {
    using B = TcGeom<M, NP, R>;
    using G4 = Tc4Geom<M, NP, R>;
    static constexpr int UBUF = B::UY * B::UP;                // floats per u buffer
    static constexpr int SM_B = 0;
    static constexpr int SM_U = B::B_FLOATS;                  // [2][UBUF]
    static constexpr int SM_Z = SM_U + 2 * UBUF;
    static constexpr int SM_FLOATS = SM_Z + 2 * B::TAPS * B::LANES;
    static constexpr int SMEM_BYTES = SM_FLOATS * 4 + 64;
    static constexpr int THREADS = 25 * 32;                   // + 4 loader warps
};

template <int M, int NP, int R>
__global__ void __launch_bounds__(25 * 32, 1) k_prior_grad_tc5(const TcArgs ta, const __grid_constant__ TcConst cc) {
    using G = TcGeom<M, NP, R>;
    using G4 = Tc4Geom<M, NP, R>;
    using G5 = Tc5Geom<M, NP, R>;
    constexpr int C = G::C, KT = G::KT, TAPS = G::TAPS, L = G::LANES, NB = G::NB, ND = G4::ND, RR = G::RR;
    extern __shared__ __align__(128) float sm[];
    float* bsm = sm + G5::SM_B;
    float* ubuf = sm + G5::SM_U;
    float* zs = sm + G5::SM_Z;
    __shared__ uint32_t tbase_s;
    __shared__ __align__(8) uint64_t bar_afull[2], bar_aempty[2], bar_dfull[ND], bar_dempty[ND], bar_zfull[ND];
    __shared__ __align__(8) uint64_t bar_pfull, bar_pempty, bar_ufull[2], bar_uempty[2];
    __shared__ float cst_s[2];
    __shared__ double wc_s[2];
    __shared__ double ep_red[2][8];

    const K1Args& args = ta.k;
    const int H = args.H, W = args.W;
    const size_t HW = (size_t)H * W;
    const int ntiles = args.ntiles, B = ta.nimg;
    const int nitems = ntiles * B;
    const int t = threadIdx.x, warp = __shfl_sync(0xffffffffu, t >> 5, 0), lane = t & 31;
    const int l = (warp & 3) * 32 + lane;
    const bool udom = args.udom != 0;

    if (warp == 0) tc::tmem_alloc<512>(&tbase_s);
    if (t == 0) {
        for (int s = 0; s < 2; ++s) {
            tc::mbar_init(&bar_afull[s], 8);
            tc::mbar_init(&bar_aempty[s], 1);
            tc::mbar_init(&bar_ufull[s], 4);
            tc::mbar_init(&bar_uempty[s], 4);
        }
        for (int s = 0; s < ND; ++s) {
            tc::mbar_init(&bar_dfull[s], 1);
            tc::mbar_init(&bar_dempty[s], 4);
            tc::mbar_init(&bar_zfull[s], 1);
        }
        tc::mbar_init(&bar_pfull, 8);
        tc::mbar_init(&bar_pempty, 1);
        tc::mbar_fence_init();
    }
    {
        const float4* src = reinterpret_cast<const float4*>(ta.bimg);
        float4* dst = reinterpret_cast<float4*>(bsm);
#pragma unroll 4
        for (int i = t; i < G::B_FLOATS / 4; i += G5::THREADS) dst[i] = __ldg(src + i);
    }
    tc::fence_proxy_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tb = tbase_s;
    const uint32_t tl = tb + ((uint32_t)((warp & 3) * 32) << 16);

    // the CTA's items: it = blockIdx.x + k * gridDim.x (blockIdx.y == 0 launches only); an item of
    // an inactive image is skipped identically by every role
    auto item_ok = [&](int it, int& b, int& tile) -> bool {
        b = it / ntiles;
        tile = it - b * ntiles;
        return args.ctl == nullptr || args.ctl[b].active;
    };

    if (warp < 8) {
        // ================================ IM ================================
        constexpr int H8 = (KT / 8 + 1) / 2;
        const int ig = warp >> 2;
        int k = 0, r = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
            int b, tile;
            if (!item_ok(it, b, tile)) continue;
            const int ubi = k & 1;
            tc::mbar_wait(&bar_ufull[ubi], (uint32_t)((k >> 1) & 1));
            const float* us = ubuf + ubi * G5::UBUF;
#pragma unroll 1
            for (int j = 0; j < RR; ++j, ++r) {
                const int s = r & 1;
                if (r >= 2) {
                    tc::mbar_wait(&bar_aempty[s], (uint32_t)(((r >> 1) - 1) & 1));
                    tc::fence_after_sync();
                }
                const float* up = us + j * G::UP + l;
                const float vc = up[C * G::UP + C];
                const uint32_t a_hi = tl + G4::COL_A0 + s * 2 * KT, a_lo = a_hi + KT;
                if (ig == 0) tc_im2col<M, G::UP, 0, H8>(up, vc, a_hi, a_lo);
                else tc_im2col<M, G::UP, H8, KT / 8>(up, vc, a_hi, a_lo);
                tc::wait_st();
                tc::fence_before_sync();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&bar_afull[s]);
            }
            ++k;
        }
    } else if (warp < 16) {
        // ================================ EP ================================
        const int half = (warp - 8) >> 2, ew = warp - 8;
        int k = 0, r = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
            int b, tile;
            if (!item_ok(it, b, tile)) continue;
            const int ubi = k & 1;
            tc::mbar_wait(&bar_ufull[ubi], (uint32_t)((k >> 1) & 1));
            const float* us = ubuf + ubi * G5::UBUF;
            const float cst = cst_s[ubi];
            const int ty = tile / ta.tiles_x, tx = tile - ty * ta.tiles_x;
            const int y0 = ty * R, x0 = tx * G::OW;
            const int lx = x0 - C + l;
            const bool col_own = (l >= C) && (l < C + G::OW) && (lx < W);
            double e_acc = 0.0;
#pragma unroll 1
            for (int j = 0; j < RR; ++j, ++r) {
                const int s = r % ND;
                tc::mbar_wait(&bar_dfull[s], (uint32_t)((r / ND) & 1));
                tc::fence_after_sync();
                const float uq = us[(j + C) * G::UP + l + C] + cst;
                constexpr int HF = NP / 2;
                float el, zl, ph[HF], pl[HF];
                if (half == 0) tc4_ep_half<NP, 0>(tl + G4::COL_D0 + s * NP, uq, cc, el, zl, ph, pl, false);
                else tc4_ep_half<NP, 1>(tl + G4::COL_D0 + s * NP, uq, cc, el, zl, ph, pl, false);
                const bool own = col_own && (j >= C) && (j < C + R) && (y0 - C + j < H);
                if (own) e_acc += (double)el;
                if (r >= 1) {
                    tc::mbar_wait(&bar_pempty, (uint32_t)((r - 1) & 1));
                    tc::fence_after_sync();
                }
#pragma unroll
                for (int c8 = 0; c8 < HF / 8; ++c8) {
                    tc::tmem_st8(tl + G4::COL_P + half * HF + c8 * 8, *reinterpret_cast<float(*)[8]>(ph + c8 * 8));
                    tc::tmem_st8(tl + G4::COL_P + NP + half * HF + c8 * 8, *reinterpret_cast<float(*)[8]>(pl + c8 * 8));
                }
                tc::tmem_st1(tl + G4::COL_ZL + s * 2 + half, zl);
                tc::wait_st();
                tc::fence_before_sync();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&bar_pfull);
            }
            // (a7) the item's energy: fixed-order sum over the 8 EP warps
            const double ew_sum = warp_sum_d(e_acc);
            if (lane == 0) ep_red[k & 1][ew] = ew_sum;
            tc::named_sync(2, 256);
            if (ew == 0 && lane == 0) {
                double e = 0.0;
                for (int i = 0; i < 8; ++i) e += ep_red[k & 1][i];
                args.epart[(size_t)b * ntiles + tile] = e;
            }
            ++k;
        }
    } else if (warp < 20) {
        // ================================ ZC ================================
        int k = 0, r = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
            int b, tile;
            if (!item_ok(it, b, tile)) continue;
            const int ubi = k & 1;
            tc::mbar_wait(&bar_ufull[ubi], (uint32_t)((k >> 1) & 1));
            const float* us = ubuf + ubi * G5::UBUF;
            const float cst = cst_s[ubi];
            const int ty = tile / ta.tiles_x, tx = tile - ty * ta.tiles_x;
            const int y0 = ty * R, x0 = tx * G::OW;
            int gslot = 0;
            if (args.ctl != nullptr) gslot = args.which_cur ? args.ctl[b].gcur : args.ctl[b].gcand;
            float* gout = args.g + (size_t)gslot * args.g_slot_stride + (size_t)b * HW;
            const bool out_col = (l < G::OW) && (x0 + l < W);
            float acc[M];
#pragma unroll
            for (int q = 0; q < M; ++q) acc[q] = 0.f;
#pragma unroll 1
            for (int j = 0; j < RR; ++j, ++r) {
                const int s = r % ND, zb = r & 1;
                tc::mbar_wait(&bar_zfull[s], (uint32_t)((r / ND) & 1));
                tc::fence_after_sync();
                float z[NB < 32 ? 32 : NB];
                if constexpr (NB == 48) {
                    tc::tmem_ld32(tl + G4::COL_D0 + s * NP, z);
                    tc::tmem_ld16(tl + G4::COL_D0 + s * NP + 32, *reinterpret_cast<float(*)[16]>(z + 32));
                } else if constexpr (NB == 24) {
                    tc::tmem_ld16(tl + G4::COL_D0 + s * NP, *reinterpret_cast<float(*)[16]>(z));
                    tc::tmem_ld8(tl + G4::COL_D0 + s * NP + 16, *reinterpret_cast<float(*)[8]>(z + 16));
                } else {
                    tc::tmem_ld8(tl + G4::COL_D0 + s * NP, *reinterpret_cast<float(*)[8]>(z));
                }
                float zl0, zl1;
                tc::tmem_ld2(tl + G4::COL_ZL + s * 2, zl0, zl1);
                tc::wait_ld();
                tc::fence_before_sync();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&bar_dempty[s]);
                float* zr = zs + zb * TAPS * L;
#pragma unroll
                for (int q = 0; q < NB; ++q) zr[q * L + l] = z[q];
                zr[NB * L + l] = zl0 + zl1;
                tc::named_sync(1, 128);
#pragma unroll
                for (int a = 0; a < M; ++a) {
                    float sa = 0.f;
#pragma unroll
                    for (int bb = 0; bb < M; ++bb) sa += zr[(a * M + bb) * L + l + bb];
                    acc[a] += sa;
                }
                const int o = j - 2 * C;
                if (o >= 0 && o < R && out_col && y0 + o < H) {
                    const float u = udom ? 1.0f : us[(o + 2 * C) * G::UP + l + 2 * C] + cst;
                    gout[(size_t)(y0 + o) * W + x0 + l] = u * acc[M - 1];
                }
#pragma unroll
                for (int q = M - 1; q > 0; --q) acc[q] = acc[q - 1];
                acc[0] = 0.f;
            }
            // every role is done with U[ubi] once the last Z row of the item is consumed
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&bar_uempty[ubi]);
            ++k;
        }
    } else if (warp == 20) {
        // ================================ MMA ================================
        const uint32_t idf = tc::idesc_tf32(128, NP), idb = tc::idesc_tf32(128, NB);
        const uint32_t b_base = tc::smem_u32(bsm);
        int r = 0;
        auto issue_b = [&](int rb) {
            const int s = rb % ND;
            tc::mbar_wait(&bar_pfull, (uint32_t)(rb & 1));
            tc::fence_after_sync();
            const uint32_t z = tb + G4::COL_D0 + s * NP, p_hi = tb + G4::COL_P, p_lo = p_hi + NP;
#pragma unroll
            for (int q = 0; q < NP / 8; ++q) {
                const uint32_t off = (uint32_t)(q * 2 * NB * 16);
                const uint64_t bh = tc::sdesc_kmajor(b_base + 2 * G::BF_FLOATS * 4 + off, NB * 16, 128);
                const uint64_t bl = tc::sdesc_kmajor(b_base + (2 * G::BF_FLOATS + G::BB_FLOATS) * 4 + off, NB * 16, 128);
                tc::mma_tf32_ts_warp(z, p_hi + q * 8, bl, idb, q > 0);
                tc::mma_tf32_ts_warp(z, p_lo + q * 8, bh, idb, 1);
            }
#pragma unroll
            for (int q = 0; q < NP / 8; ++q) {
                const uint64_t bh = tc::sdesc_kmajor(b_base + 2 * G::BF_FLOATS * 4 + (uint32_t)(q * 2 * NB * 16), NB * 16, 128);
                tc::mma_tf32_ts_warp(z, p_hi + q * 8, bh, idb, 1);
            }
            tc::mma_commit_warp(&bar_pempty);
            tc::mma_commit_warp(&bar_zfull[s]);
        };
        for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
            int b, tile;
            if (!item_ok(it, b, tile)) continue;
#pragma unroll 1
            for (int j = 0; j < RR; ++j, ++r) {
                const int s = r & 1, sd = r % ND;
                tc::mbar_wait(&bar_afull[s], (uint32_t)((r >> 1) & 1));
                if (r >= ND) tc::mbar_wait(&bar_dempty[sd], (uint32_t)(((r / ND) - 1) & 1));
                tc::fence_after_sync();
                const uint32_t a_hi = tb + G4::COL_A0 + s * 2 * KT, a_lo = a_hi + KT, d = tb + G4::COL_D0 + sd * NP;
#pragma unroll
                for (int q = 0; q < KT / 8; ++q) {
                    const uint32_t off = (uint32_t)(q * 2 * NP * 16);
                    const uint64_t bh = tc::sdesc_kmajor(b_base + off, NP * 16, 128);
                    const uint64_t bl = tc::sdesc_kmajor(b_base + G::BF_FLOATS * 4 + off, NP * 16, 128);
                    tc::mma_tf32_ts_warp(d, a_hi + q * 8, bl, idf, q > 0);
                    tc::mma_tf32_ts_warp(d, a_lo + q * 8, bh, idf, 1);
                }
#pragma unroll
                for (int q = 0; q < KT / 8; ++q) {
                    const uint64_t bh = tc::sdesc_kmajor(b_base + (uint32_t)(q * 2 * NP * 16), NP * 16, 128);
                    tc::mma_tf32_ts_warp(d, a_hi + q * 8, bh, idf, 1);
                }
                tc::mma_commit_warp(&bar_aempty[s]);
                tc::mma_commit_warp(&bar_dfull[sd]);
                if (r >= 1) issue_b(r - 1);
            }
        }
        if (r >= 1) issue_b(r - 1);
    } else {
        // ================================ LD: u tiles ================================
        const int lw = warp - 21;
        int k = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
            int b, tile;
            if (!item_ok(it, b, tile)) continue;
            const int ubi = k & 1;
            if (k >= 2) tc::mbar_wait(&bar_uempty[ubi], (uint32_t)(((k >> 1) - 1) & 1));
            int wslot = 0;
            if (args.ctl != nullptr) wslot = args.which_cur ? args.ctl[b].cur : args.ctl[b].cand;
            const double* w = args.w + (size_t)wslot * args.w_slot_stride + (size_t)b * HW;
            const int ty = tile / ta.tiles_x, tx = tile - ty * ta.tiles_x;
            const int y0 = ty * R, x0 = tx * G::OW;
            const int yc = min(y0 + R / 2, H - 1), xc = min(x0 + G::OW / 2, W - 1);
            const double wc = w[(size_t)yc * W + xc];
            const float cst = (float)(udom ? wc : exp(wc));
            tc_stage_u<G::UY, G::UX, G::UP, 4>(ubuf + ubi * G5::UBUF, w, args.halo, H, W, y0, x0, 2 * C, udom, cst,
                                               wc, lw, lane);
            if (lw == 0 && lane == 0) { cst_s[ubi] = cst; wc_s[ubi] = wc; }
            __threadfence_block();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&bar_ufull[ubi]);
            ++k;
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<512>(tb);
}

// =============================================================================================
// K8 v6: v3's lock-step row loop with THREE warp groups (384 threads, 2 CTAs per SM = 24 warps)
// instead of two, so that more warps hide the latencies of the per-row thread work (ncu of v3:
// issue active 52 %, stalls on fixed-latency dependencies, MIO throttle and the two CTA
// barriers per row).  The row phases are split three ways by compile-time tables (Tc3Part):
// im2col tap chunks, Z tap chunks and epilogue filter chunks over all three groups, the col2im
// rows over groups 0 and 1 (as v3), so group 2 takes a larger share of the im2col and Z
// copies.  Shared memory as v3 minus the unused 49th Z column and the u pitch padding (the
// third group's last-tap partial needs the room; 2 CTAs per SM must still fit).
// =============================================================================================
template <int M>
struct Tc3Part;
template <>
struct Tc3Part<7> {   // KT 56 -> 7 im2col chunks, NB 48 -> 6 Z chunks, NP 48 -> 6 filter chunks
    static constexpr int IM[4] = {0, 1, 3, 7};
    static constexpr int ZC[4] = {0, 1, 2, 6};
    static constexpr int EP[4] = {0, 2, 4, 6};
};
template <>
struct Tc3Part<5> {   // KT 32 -> 4, NB 24 -> 3, NP 32 -> 4
    static constexpr int IM[4] = {0, 1, 2, 4};
    static constexpr int ZC[4] = {0, 1, 2, 3};
    static constexpr int EP[4] = {0, 1, 3, 4};
};

template <int M, int NP, int R>
struct Tc3Geom {
    using B = TcGeom<M, NP, R>;
    static constexpr int C = B::C, TAPS = B::TAPS, KT = B::KT, LANES = B::LANES, OW = B::OW, RR = B::RR;
    static constexpr int UY = B::UY, UX = B::UX, UP = B::UX, NB = B::NB;
    static constexpr int SM_B = 0;
    static constexpr int SM_U = SM_B + B::B_FLOATS;
    static constexpr int SM_Z = SM_U + UY * UP;
    static constexpr int SM_HAND = SM_Z + NB * LANES;
    static constexpr int SM_ZL = SM_HAND + 8 * LANES;     // [2 rows][3 groups][LANES]
    static constexpr int SM_FLOATS = SM_ZL + 6 * LANES;
    static constexpr int SMEM_BYTES = SM_FLOATS * 4 + 64;
    static_assert(2 * (SMEM_BYTES + 1024) <= 228 * 1024, "two CTAs per SM");
};

template <int M, int NP, int R>
__global__ void __launch_bounds__(384, 2) k_prior_grad_tc6(const TcArgs ta, const __grid_constant__ TcConst cc) {
    using G = Tc3Geom<M, NP, R>;
    using GB = TcGeom<M, NP, R>;
    using PT = Tc3Part<M>;
    constexpr int C = G::C, L = G::LANES;
    extern __shared__ __align__(128) float sm[];
    float* bsm = sm + G::SM_B;
    float* us = sm + G::SM_U;
    float* zs = sm + G::SM_Z;
    __shared__ uint32_t tbase_s;
    __shared__ __align__(8) uint64_t mbar_f, mbar_b;
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
    const int ty = tile / ta.tiles_x, tx = tile - ty * ta.tiles_x;
    const int y0 = ty * R, x0 = tx * G::OW;
    const double* w = args.w + (size_t)wslot * args.w_slot_stride + (size_t)b * HW;
    const int t = threadIdx.x, warp = __shfl_sync(0xffffffffu, t >> 5, 0);
    const int wg = warp >> 2;                                   // warp group (0, 1, 2)
    const int l = (warp & 3) * 32 + (t & 31);                   // TMEM lane = response pixel

    if (warp == 0) tc::tmem_alloc<GB::TCOLS>(&tbase_s);
    if (t == 0) {
        tc::mbar_init(&mbar_f, 1);
        tc::mbar_init(&mbar_b, 1);
        tc::mbar_fence_init();
    }
    {
        const float4* src = reinterpret_cast<const float4*>(ta.bimg);
        float4* dst = reinterpret_cast<float4*>(bsm);
#pragma unroll 4
        for (int i = t; i < GB::B_FLOATS / 4; i += 384) dst[i] = __ldg(src + i);
    }
    const int yc = min(y0 + R / 2, H - 1), xc = min(x0 + G::OW / 2, W - 1);
    const bool udom = args.udom != 0;
    const double wc = w[(size_t)yc * W + xc];
    const float cst = (float)(udom ? wc : exp(wc));
    tc_stage_u<G::UY, G::UX, G::UP, 12>(us, w, args.halo, H, W, y0, x0, 2 * C, udom, cst, wc, warp, t & 31);
    tc::fence_proxy_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tb = tbase_s;
    const uint32_t tl = tb + ((uint32_t)((warp & 3) * 32) << 16);
    const uint32_t idf = tc::idesc_tf32(128, NP);
    const uint32_t idb = tc::idesc_tf32(128, G::NB);
    const uint32_t b_base = tc::smem_u32(bsm);

    const int lx = x0 - C + l;
    const bool col_own = (l >= C) && (l < C + G::OW) && (lx < W);
    const bool out_col = (l < G::OW) && (x0 + l < W);

    double e_acc = 0.0;
    constexpr int NC8 = G::KT / 8, NF8 = NP / 8;
    constexpr int A0 = C + 1, A1 = M - A0;                 // col2im rows: wg0 a < A0, wg1 a >= A0
    float acc[A0 > A1 ? A0 : A1];
#pragma unroll
    for (int k = 0; k < (A0 > A1 ? A0 : A1); ++k) acc[k] = 0.f;
    float* gout = args.g + (size_t)gslot * args.g_slot_stride + (size_t)b * HW;
    float* hand = sm + G::SM_HAND;
    float* zls = sm + G::SM_ZL;

#pragma unroll 1
    for (int j = 0; j <= G::RR; ++j) {
        float uq = 0.f;
        if (j < G::RR) {
            const float* up = us + j * G::UP + l;
            const float vc = up[C * G::UP + C];
            uq = vc + cst;
            if (wg == 0) tc_im2col<M, G::UP, PT::IM[0], PT::IM[1]>(up, vc, tl + GB::COL_AHI, tl + GB::COL_ALO);
            else if (wg == 1) tc_im2col<M, G::UP, PT::IM[1], PT::IM[2]>(up, vc, tl + GB::COL_AHI, tl + GB::COL_ALO);
            else tc_im2col<M, G::UP, PT::IM[2], PT::IM[3]>(up, vc, tl + GB::COL_AHI, tl + GB::COL_ALO);
        }
        if (j > 0) {
            tc::mbar_wait(&mbar_b, (uint32_t)((j - 1) & 1));
            tc::fence_after_sync();
            if (wg == 0) tc_z_to_smem<L, PT::ZC[0], PT::ZC[1]>(tl + GB::COL_Z, zs, l);
            else if (wg == 1) tc_z_to_smem<L, PT::ZC[1], PT::ZC[2]>(tl + GB::COL_Z, zs, l);
            else tc_z_to_smem<L, PT::ZC[2], PT::ZC[3]>(tl + GB::COL_Z, zs, l);
        }
        tc::wait_st();
        tc::fence_before_sync();
        __syncthreads();
        if (warp == 0 && j < G::RR) {
            tc::fence_after_sync();
#pragma unroll
            for (int s = 0; s < NC8; ++s) {
                const uint32_t off = (uint32_t)(s * 2 * NP * 16);
                const uint64_t bh = tc::sdesc_kmajor(b_base + off, NP * 16, 128);
                const uint64_t bl = tc::sdesc_kmajor(b_base + GB::BF_FLOATS * 4 + off, NP * 16, 128);
                tc::mma_tf32_ts_warp(tb + GB::COL_D, tb + GB::COL_AHI + s * 8, bl, idf, s > 0);
                tc::mma_tf32_ts_warp(tb + GB::COL_D, tb + GB::COL_ALO + s * 8, bh, idf, 1);
            }
#pragma unroll
            for (int s = 0; s < NC8; ++s) {
                const uint32_t off = (uint32_t)(s * 2 * NP * 16);
                const uint64_t bh = tc::sdesc_kmajor(b_base + off, NP * 16, 128);
                tc::mma_tf32_ts_warp(tb + GB::COL_D, tb + GB::COL_AHI + s * 8, bh, idf, 1);
            }
            tc::mma_commit_warp(&mbar_f);
        }
        if (j > 0 && wg < 2) {
            const int jz = j - 1;
            if (wg == 0) {
#pragma unroll
                for (int a = 0; a < A0; ++a) {
                    float sa = 0.f;
#pragma unroll
                    for (int bb = 0; bb < M; ++bb) sa += zs[(a * M + bb) * L + l + bb];
                    acc[a] += sa;
                }
                const int o = jz - (A0 - 1);
                if (o >= 0) hand[(o & 7) * L + l] = acc[A0 - 1];
#pragma unroll
                for (int k = A0 - 1; k > 0; --k) acc[k] = acc[k - 1];
                acc[0] = 0.f;
            } else {
                const float* zl = zls + (jz & 1) * 3 * L;
#pragma unroll
                for (int k = 0; k < A1; ++k) {
                    const int a = A0 + k;
                    float sa = 0.f;
#pragma unroll
                    for (int bb = 0; bb < M; ++bb) {
                        const int tap = a * M + bb;
                        sa += tap < G::NB ? zs[tap * L + l + bb] : (zl[l + bb] + zl[L + l + bb]) + zl[2 * L + l + bb];
                    }
                    acc[k] += sa;
                }
                const int o = jz - 2 * C;
                if (o >= 0 && o < R && out_col && y0 + o < H) {
                    const float s_tot = acc[A1 - 1] + hand[(o & 7) * L + l];
                    const float u = udom ? 1.0f : us[(o + 2 * C) * G::UP + l + 2 * C] + cst;
                    gout[(size_t)(y0 + o) * W + x0 + l] = u * s_tot;
                }
#pragma unroll
                for (int k = A1 - 1; k > 0; --k) acc[k] = acc[k - 1];
                acc[0] = 0.f;
            }
        }
        if (j < G::RR) {
            tc::mbar_wait(&mbar_f, (uint32_t)(j & 1));
            tc::fence_after_sync();
            const bool own = col_own && (j >= C) && (j < C + R) && (y0 - C + j < H);
            float zl;
            const float el = wg == 0
                ? tc_epilogue<PT::EP[0], PT::EP[1]>(tl + GB::COL_D, tl + GB::COL_PHI, tl + GB::COL_PLO, uq, cc.sumk, cc.thl, cc.kbl, zl)
                : wg == 1
                ? tc_epilogue<PT::EP[1], PT::EP[2]>(tl + GB::COL_D, tl + GB::COL_PHI, tl + GB::COL_PLO, uq, cc.sumk, cc.thl, cc.kbl, zl)
                : tc_epilogue<PT::EP[2], PT::EP[3]>(tl + GB::COL_D, tl + GB::COL_PHI, tl + GB::COL_PLO, uq, cc.sumk, cc.thl, cc.kbl, zl);
            zls[(j & 1) * 3 * L + wg * L + l] = zl;
            if (own) e_acc += (double)el;
            tc::wait_st();
            tc::fence_before_sync();
            __syncthreads();
            if (warp == 0) {
                tc::fence_after_sync();
#pragma unroll
                for (int s = 0; s < NF8; ++s) {
                    const uint32_t off = (uint32_t)(s * 2 * G::NB * 16);
                    const uint64_t bh = tc::sdesc_kmajor(b_base + 2 * GB::BF_FLOATS * 4 + off, G::NB * 16, 128);
                    const uint64_t bl = tc::sdesc_kmajor(b_base + (2 * GB::BF_FLOATS + GB::BB_FLOATS) * 4 + off,
                                                         G::NB * 16, 128);
                    tc::mma_tf32_ts_warp(tb + GB::COL_Z, tb + GB::COL_PHI + s * 8, bl, idb, s > 0);
                    tc::mma_tf32_ts_warp(tb + GB::COL_Z, tb + GB::COL_PLO + s * 8, bh, idb, 1);
                }
#pragma unroll
                for (int s = 0; s < NF8; ++s) {
                    const uint32_t off = (uint32_t)(s * 2 * G::NB * 16);
                    const uint64_t bh = tc::sdesc_kmajor(b_base + 2 * GB::BF_FLOATS * 4 + off, G::NB * 16, 128);
                    tc::mma_tf32_ts_warp(tb + GB::COL_Z, tb + GB::COL_PHI + s * 8, bh, idb, 1);
                }
                tc::mma_commit_warp(&mbar_b);
            }
        }
    }
    const double e = block_sum_d(e_acc, red);
    if (t == 0) args.epart[(size_t)b * args.ntiles * args.groups + blockIdx.x] = e;
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<GB::TCOLS>(tb);
}

// =============================================================================================
// K8 v7: v3's lock-step row loop with the u tile STREAMED through a 16-row shared-memory ring
// instead of staged whole in the prologue, so that a tile can be any number of rows R (runtime,
// ta.rows): one new staged row per response row, loaded one iteration ahead (prefetch register)
// and written before the iteration's second CTA barrier.  Taller tiles cut the halo recompute
// (R + 2C response rows per R output rows: 1.094 at R = 64, 1.023 at R = 256) and the prologue,
// and free 32 KB of shared memory.  Column packing as v3 (strips of the remainder columns of
// tc_spt bands of R rows).  Batch path only (the slab path keeps v3's 64-row bands).
// =============================================================================================
template <int M, int NP>
struct Tc7Geom {
    using B = TcGeom<M, NP, 64>;
    static constexpr int C = B::C, KT = B::KT, LANES = B::LANES, OW = B::OW, UX = B::UX, UP = B::UP, NB = B::NB;
    static constexpr int RING = 16;                       // staged u rows in flight (>= 2C + 3)
    static_assert(RING >= 2 * C + 3, "ring too small");
    static constexpr int SM_B = 0;
    static constexpr int SM_U = SM_B + B::B_FLOATS;
    static constexpr int SM_Z = SM_U + RING * UP;
    static constexpr int SM_HAND = SM_Z + B::TAPS * LANES;
    static constexpr int SM_ZL = SM_HAND + 8 * LANES;
    static constexpr int SM_FLOATS = SM_ZL + 4 * LANES;
    static constexpr int SMEM_BYTES = SM_FLOATS * 4 + 64;
};

// im2col from the ring: rp[a] = row a of the window (lane offset applied)
template <int M, int C0, int C1>
__device__ __forceinline__ void tc_im2col_ring(const float* const (&rp)[M], float vc, uint32_t t_hi, uint32_t t_lo) {
#pragma unroll
    for (int c8 = C0; c8 < C1; ++c8) {
        float h[8], lo[8];
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
            const int t0 = c8 * 8 + e, t1 = t0 + 1;
            const float2 u2 = make_float2(t0 < M * M ? rp[t0 / M][t0 % M] : vc, t1 < M * M ? rp[t1 / M][t1 % M] : vc);
            const float2 v = __fadd2_rn(u2, make_float2(-vc, -vc));
            float2 hi2, lo2;
            tc::tf32_split2(v, hi2, lo2);
            h[e] = hi2.x; h[e + 1] = hi2.y;
            lo[e] = lo2.x; lo[e + 1] = lo2.y;
        }
        tc::tmem_st8(t_hi + c8 * 8, h);
        tc::tmem_st8(t_lo + c8 * 8, lo);
    }
}

template <int M, int NP>
__global__ void __launch_bounds__(256, 2) k_prior_grad_tc7(const TcArgs ta, const __grid_constant__ TcConst cc) {
    using G = Tc7Geom<M, NP>;
    using GB = TcGeom<M, NP, 64>;
    constexpr int C = G::C, KT = G::KT, L = G::LANES, RING = G::RING;
    extern __shared__ __align__(128) float sm[];
    float* bsm = sm + G::SM_B;
    float* us = sm + G::SM_U;                                   // ring [RING][UP]
    float* zs = sm + G::SM_Z;
    __shared__ uint32_t tbase_s;
    __shared__ __align__(8) uint64_t mbar_f, mbar_b;
    __shared__ double red[32];

    const K1Args& args = ta.k;
    const int R = args.tc_rows;                                 // output rows per tile (runtime)
    const int RR = R + 2 * C;                                   // response rows
    const int UYR = R + 4 * C;                                  // staged rows
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
    const int t = threadIdx.x, warp = __shfl_sync(0xffffffffu, t >> 5, 0);
    const int wg = warp >> 2;
    const int l = (warp & 3) * 32 + (t & 31);
    const int nbands = (H + R - 1) / R;
    const int nnorm = nbands * ta.tiles_x;
    const bool packed = tile >= nnorm;
    int y0, x0, sy0, ocol;
    bool svalid = true;
    const int SP = args.tc_rem + 4 * C;
    int band0 = 0;
    if (!packed) {
        const int ty = tile / ta.tiles_x, tx = tile - ty * ta.tiles_x;
        y0 = ty * R; x0 = tx * G::OW; sy0 = y0; ocol = l;
    } else {
        band0 = (tile - nnorm) * args.tc_spt;
        const int st = l / SP;
        ocol = l - st * SP;
        svalid = st < args.tc_spt && band0 + st < nbands;
        y0 = band0 * R; x0 = ta.tiles_x * G::OW; sy0 = (band0 + st) * R;
    }

    if (warp == 0) tc::tmem_alloc<GB::TCOLS>(&tbase_s);
    if (t == 0) {
        tc::mbar_init(&mbar_f, 1);
        tc::mbar_init(&mbar_b, 1);
        tc::mbar_fence_init();
    }
    {
        const float4* src = reinterpret_cast<const float4*>(ta.bimg);
        float4* dst = reinterpret_cast<float4*>(bsm);
#pragma unroll 4
        for (int i = t; i < GB::B_FLOATS / 4; i += 256) dst[i] = __ldg(src + i);
    }
    const int yc = min(y0 + min(R, H) / 2, H - 1), xc = min(x0 + (packed ? args.tc_rem : G::OW) / 2, W - 1);
    const bool udom = args.udom != 0;
    const double wc = w[(size_t)yc * W + xc];
    const float cst = (float)(udom ? wc : exp(wc));
    // this thread's staged column (t < UX): image column and unwrapped row origin of its strip
    const bool st_on = t < G::UX;
    bool st_ok = false;
    int st_gx = 0, st_yb = 0;
    if (st_on) {
        if (!packed) {
            st_ok = true;
            st_gx = wrap_idx(x0 - 2 * C + t, W);
            st_yb = y0 - 2 * C;
        } else {
            const int st = t / SP, band = band0 + st;
            st_ok = st < args.tc_spt && band < nbands;
            st_gx = wrap_idx(x0 - 2 * C + (t - st * SP), W);
            st_yb = band * R - 2 * C;
        }
    }
    auto stage_load = [&](int jj) -> double {
        return (st_ok && jj < UYR) ? w[(size_t)wrap_idx(st_yb + jj, H) * W + st_gx] : wc;
    };
    auto stage_store = [&](int jj, double v) {
        if (st_on && jj < UYR) us[(jj & (RING - 1)) * G::UP + t] = udom ? (float)(v - (double)cst) : cst * expm1f((float)(v - wc));
    };
    // prologue: staged rows 0 .. 2C, prefetch of row 2C + 1
    {
        double v[2 * C + 1];
#pragma unroll
        for (int jj = 0; jj <= 2 * C; ++jj) v[jj] = stage_load(jj);
#pragma unroll
        for (int jj = 0; jj <= 2 * C; ++jj) stage_store(jj, v[jj]);
    }
    double pf = stage_load(2 * C + 1);
    tc::fence_proxy_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tb = tbase_s;
    const uint32_t tl = tb + ((uint32_t)((warp & 3) * 32) << 16);
    const uint32_t idf = tc::idesc_tf32(128, NP);
    const uint32_t idb = tc::idesc_tf32(128, G::NB);
    const uint32_t b_base = tc::smem_u32(bsm);

    const int ow = packed ? args.tc_rem : G::OW;
    const bool col_own = svalid && (ocol >= C) && (ocol < C + ow) && (x0 - C + ocol < W);
    const bool out_col = svalid && (ocol < ow) && (x0 + ocol < W);

    double e_acc = 0.0;
    constexpr int NC8 = KT / 8, H8 = (NC8 + 1) / 2;
    constexpr int NZ8 = G::NB / 8, HZ8 = (NZ8 + 1) / 2;
    constexpr int NF8 = NP / 8, HF8 = NF8 / 2;
    constexpr int A0 = C + 1, A1 = M - A0;
    float acc[A0 > A1 ? A0 : A1];
#pragma unroll
    for (int k = 0; k < (A0 > A1 ? A0 : A1); ++k) acc[k] = 0.f;
    float* gout = args.g + (size_t)gslot * args.g_slot_stride + (size_t)b * HW;
    float* hand = sm + G::SM_HAND;
    float* zls = sm + G::SM_ZL;

#pragma unroll 1
    for (int j = 0; j <= RR; ++j) {
        float uq = 0.f;
        if (j < RR) {
            const float* rp[M];
#pragma unroll
            for (int a = 0; a < M; ++a) rp[a] = us + ((j + a) & (RING - 1)) * G::UP + l;
            const float vc = rp[C][C];
            uq = vc + cst;
            if (wg == 0) tc_im2col_ring<M, 0, H8>(rp, vc, tl + GB::COL_AHI, tl + GB::COL_ALO);
            else tc_im2col_ring<M, H8, NC8>(rp, vc, tl + GB::COL_AHI, tl + GB::COL_ALO);
        }
        if (j > 0) {
            tc::mbar_wait(&mbar_b, (uint32_t)((j - 1) & 1));
            tc::fence_after_sync();
            if (wg == 0) tc_z_to_smem<L, 0, HZ8>(tl + GB::COL_Z, zs, l);
            else tc_z_to_smem<L, HZ8, NZ8>(tl + GB::COL_Z, zs, l);
        }
        tc::wait_st();
        tc::fence_before_sync();
        __syncthreads();
        if (warp == 0 && j < RR) {
            tc::fence_after_sync();
#pragma unroll
            for (int s = 0; s < NC8; ++s) {
                const uint32_t off = (uint32_t)(s * 2 * NP * 16);
                const uint64_t bh = tc::sdesc_kmajor(b_base + off, NP * 16, 128);
                const uint64_t bl = tc::sdesc_kmajor(b_base + GB::BF_FLOATS * 4 + off, NP * 16, 128);
                tc::mma_tf32_ts_warp(tb + GB::COL_D, tb + GB::COL_AHI + s * 8, bl, idf, s > 0);
                tc::mma_tf32_ts_warp(tb + GB::COL_D, tb + GB::COL_ALO + s * 8, bh, idf, 1);
            }
#pragma unroll
            for (int s = 0; s < NC8; ++s) {
                const uint32_t off = (uint32_t)(s * 2 * NP * 16);
                const uint64_t bh = tc::sdesc_kmajor(b_base + off, NP * 16, 128);
                tc::mma_tf32_ts_warp(tb + GB::COL_D, tb + GB::COL_AHI + s * 8, bh, idf, 1);
            }
            tc::mma_commit_warp(&mbar_f);
        }
        if (j > 0) {
            const int jz = j - 1;
            if (wg == 0) {
#pragma unroll
                for (int a = 0; a < A0; ++a) {
                    float sa = 0.f;
#pragma unroll
                    for (int bb = 0; bb < M; ++bb) sa += zs[(a * M + bb) * L + l + bb];
                    acc[a] += sa;
                }
                const int o = jz - (A0 - 1);
                if (o >= 0) hand[(o & 7) * L + l] = acc[A0 - 1];
#pragma unroll
                for (int k = A0 - 1; k > 0; --k) acc[k] = acc[k - 1];
                acc[0] = 0.f;
            } else {
                const float* zl = zls + (jz & 1) * 2 * L;
#pragma unroll
                for (int k = 0; k < A1; ++k) {
                    const int a = A0 + k;
                    float sa = 0.f;
#pragma unroll
                    for (int bb = 0; bb < M; ++bb) {
                        const int tap = a * M + bb;
                        sa += tap < G::NB ? zs[tap * L + l + bb] : zl[l + bb] + zl[L + l + bb];
                    }
                    acc[k] += sa;
                }
                const int o = jz - 2 * C;
                if (o >= 0 && o < R && out_col && sy0 + o < H) {
                    const float s_tot = acc[A1 - 1] + hand[(o & 7) * L + l];
                    const float u = udom ? 1.0f : us[((o + 2 * C) & (RING - 1)) * G::UP + l + 2 * C] + cst;
                    gout[(size_t)(sy0 + o) * W + x0 + ocol] = u * s_tot;
                }
#pragma unroll
                for (int k = A1 - 1; k > 0; --k) acc[k] = acc[k - 1];
                acc[0] = 0.f;
            }
        }
        if (j < RR) {
            // stream the next staged row (needed by im2col(j + 1)), prefetch the one after
            stage_store(j + 2 * C + 1, pf);
            pf = stage_load(j + 2 * C + 2);
            tc::mbar_wait(&mbar_f, (uint32_t)(j & 1));
            tc::fence_after_sync();
            const bool own = col_own && (j >= C) && (j < C + R) && (sy0 - C + j < H);
            float zl;
            const float el = wg == 0
                ? tc_epilogue<0, HF8>(tl + GB::COL_D, tl + GB::COL_PHI, tl + GB::COL_PLO, uq, cc.sumk, cc.thl, cc.kbl, zl)
                : tc_epilogue<HF8, NF8>(tl + GB::COL_D, tl + GB::COL_PHI, tl + GB::COL_PLO, uq, cc.sumk, cc.thl, cc.kbl, zl);
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
                    const uint64_t bh = tc::sdesc_kmajor(b_base + 2 * GB::BF_FLOATS * 4 + off, G::NB * 16, 128);
                    const uint64_t bl = tc::sdesc_kmajor(b_base + (2 * GB::BF_FLOATS + GB::BB_FLOATS) * 4 + off,
                                                         G::NB * 16, 128);
                    tc::mma_tf32_ts_warp(tb + GB::COL_Z, tb + GB::COL_PHI + s * 8, bl, idb, s > 0);
                    tc::mma_tf32_ts_warp(tb + GB::COL_Z, tb + GB::COL_PLO + s * 8, bh, idb, 1);
                }
#pragma unroll
                for (int s = 0; s < NF8; ++s) {
                    const uint32_t off = (uint32_t)(s * 2 * G::NB * 16);
                    const uint64_t bh = tc::sdesc_kmajor(b_base + 2 * GB::BF_FLOATS * 4 + off, G::NB * 16, 128);
                    tc::mma_tf32_ts_warp(tb + GB::COL_Z, tb + GB::COL_PHI + s * 8, bh, idb, 1);
                }
                tc::mma_commit_warp(&mbar_b);
            }
        }
    }
    const double e = block_sum_d(e_acc, red);
    if (t == 0) args.epart[(size_t)b * args.ntiles * args.groups + blockIdx.x] = e;
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<GB::TCOLS>(tb);
}

}  // namespace foe
