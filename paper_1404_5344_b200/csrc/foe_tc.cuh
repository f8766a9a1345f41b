// foe_tc.cuh -- shared pieces of the tensor-core FoE stencil K8 (foe_th.cuh): its launch
// arguments, the fp64 -> fp32 staging of the u tile (a2) and the read-out of the backward
// accumulator Z into shared memory for the col2im.
#pragma once

#include "foe_kernels.cuh"
#include "tc_ptx.cuh"

// rows of the u tile a warp stages at a time (their loads all in flight before the exponentials)
#ifndef FOE_STAGE_ROWS
#define FOE_STAGE_ROWS 2
#endif


namespace foe {

struct TcArgs {
    K1Args k;                 // image geometry, slots, control, outputs (as K1)
    const void* bimg;         // B operand images (fp16 hi/lo), built at model creation
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
                                           int x0, int c2, bool udom, float cst, double wc, int warp, int lane,
                                           int uy_lo = 0, int uy_hi = UY) {
    constexpr int NX = (UX + 31) / 32;
    const double ec = udom ? 0.0 : exp(wc);
    int gx[NX];
#pragma unroll
    for (int k = 0; k < NX; ++k) gx[k] = wrap_idx(x0 - c2 + lane + 32 * k, W);
    // FOE_STAGE_ROWS rows per warp in flight (all their loads issued before any exponential)
    constexpr int NRB = FOE_STAGE_ROWS;
    for (int uy0 = uy_lo + warp * NRB; uy0 < uy_hi; uy0 += NWARPS * NRB) {
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
            for (int k = 0; k < NX; ++k) v[r][k] = (uy < uy_hi && lane + 32 * k < UX) ? src[gx[k]] : wc;
        }
#pragma unroll
        for (int r = 0; r < NRB; ++r) {
            const int uy = uy0 + r;
            if (uy >= uy_hi) break;
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
                                                  double wc, int warp, int lane, int uy_lo = 0, int uy_hi = UY) {
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
    for (int uy = uy_lo + warp; uy < uy_hi; uy += NWARPS) {
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

}  // namespace foe
