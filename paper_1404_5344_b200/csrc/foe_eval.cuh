// foe_eval.cuh -- evaluation and synthesis kernels of SURVEY.md 8(f) f4: PSNR and SSIM of a
// restored batch against the clean images (the paper's reporting, PAPER.md
// Sec. III), and counter-based speckle synthesis f = u sqrt(s), s ~ Gamma(L, 1/L) (reading
// R-14: the amplitude model pinned by Table II).
//
// The Gamma variate: Marsaglia-Tsang's method (shape L >= 1) driven by Philox4x32-10 (Salmon et
// al., SC'11) -- attempt k of pixel p uses the counter (p lo, p hi, k, 0) under the key (seed lo,
// seed hi), so every pixel's draw is independent of the launch geometry.  All of it in fp64.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "foe_kernels.cuh"

namespace foe {

// ---- Philox4x32-10 -----------------------------------------------------------------------------
__device__ __forceinline__ void philox4x32_10(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c[0], hi0 = __umulhi(0xD2511F53u, c[0]);
        const uint32_t lo1 = 0xCD9E8D57u * c[2], hi1 = __umulhi(0xCD9E8D57u, c[2]);
        const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}
__device__ __forceinline__ double u01(uint32_t w) { return ((double)w + 0.5) * (1.0 / 4294967296.0); }

// f = u sqrt(s) for B images of HW pixels; looks[b] >= 1; status[b] counts pixels that needed
// more than 64 attempts (then s of the last attempt is used; probability ~1e-40 per pixel)
__global__ void k_add_speckle(const float* u, const double* looks, int B, size_t HW, unsigned long long seed,
                              float* f, unsigned int* capped) {
    const uint32_t k0 = (uint32_t)(seed & 0xFFFFFFFFull), k1 = (uint32_t)(seed >> 32);
    const size_t n = (size_t)B * HW;
    for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (size_t)gridDim.x * blockDim.x) {
        const int b = (int)(p / HW);
        const double L = looks[b];
        const double d = L - 1.0 / 3.0, cc = 1.0 / sqrt(9.0 * d);
        double s = 1.0;
        bool done = false;
        for (int k = 0; k < 64 && !done; ++k) {
            uint32_t c[4] = {(uint32_t)(p & 0xFFFFFFFFull), (uint32_t)(p >> 32), (uint32_t)k, 0u};
            philox4x32_10(c, k0, k1);
            const double x = sqrt(-2.0 * log(u01(c[0]))) * cos(6.283185307179586 * u01(c[1]));
            const double t = 1.0 + cc * x;
            const double v = t * t * t;
            if (v > 0.0 && log(u01(c[2])) < 0.5 * x * x + d - d * v + d * log(v)) {
                s = d * v / L;
                done = true;
            } else if (v > 0.0) {
                s = d * v / L;
            }
        }
        if (!done) atomicAdd(capped, 1u);
        f[p] = (float)((double)u[p] * sqrt(s));
    }
}

// ---- PSNR: per-block fixed-order partials of sum (x - ref)^2 ------------------------------------
__global__ void __launch_bounds__(kThreads) k_sq_err_part(const float* x, const float* ref, size_t HW, int nblk,
                                                          double* part) {
    __shared__ double red[32];
    const int b = blockIdx.y;
    double acc = 0.0;
    for (size_t p = (size_t)blockIdx.x * kThreads + threadIdx.x; p < HW; p += (size_t)nblk * kThreads) {
        const double e = (double)x[(size_t)b * HW + p] - (double)ref[(size_t)b * HW + p];
        acc += e * e;
    }
    const double s = block_sum_d(acc, red);
    if (threadIdx.x == 0) part[(size_t)b * nblk + blockIdx.x] = s;
}

// ---- SSIM: one thread per valid-region pixel, explicit 11 x 11 Gaussian windowed moments -------
struct SsimParams {
    double w[11];   // normalised 1-D Gaussian (sigma 1.5); the 2-D window is w_a w_b
    double c1, c2;
};

__global__ void __launch_bounds__(kThreads) k_ssim_part(const float* x, const float* ref, int H, int W, int nblk,
                                                        const __grid_constant__ SsimParams sp, double* part) {
    __shared__ double red[32];
    const int b = blockIdx.y;
    const int oh = H - 10, ow = W - 10;
    const size_t on = (size_t)oh * ow;
    const float* xb = x + (size_t)b * H * W;
    const float* yb = ref + (size_t)b * H * W;
    double acc = 0.0;
    for (size_t q = (size_t)blockIdx.x * kThreads + threadIdx.x; q < on; q += (size_t)nblk * kThreads) {
        const int oy = (int)(q / ow), ox = (int)(q - (size_t)oy * ow);
        double mx = 0, my = 0, sxx = 0, syy = 0, sxy = 0;
        for (int a = 0; a < 11; ++a) {
            const float* xr = xb + (size_t)(oy + a) * W + ox;
            const float* yr = yb + (size_t)(oy + a) * W + ox;
            double rx = 0, ry = 0, rxx = 0, ryy = 0, rxy = 0;
#pragma unroll
            for (int c = 0; c < 11; ++c) {
                const double xv = xr[c], yv = yr[c], wc = sp.w[c];
                rx += wc * xv; ry += wc * yv;
                rxx += wc * xv * xv; ryy += wc * yv * yv; rxy += wc * xv * yv;
            }
            const double wa = sp.w[a];
            mx += wa * rx; my += wa * ry; sxx += wa * rxx; syy += wa * ryy; sxy += wa * rxy;
        }
        const double vx = sxx - mx * mx, vy = syy - my * my, cxy = sxy - mx * my;
        acc += (2 * mx * my + sp.c1) * (2 * cxy + sp.c2) / ((mx * mx + my * my + sp.c1) * (vx + vy + sp.c2));
    }
    const double s = block_sum_d(acc, red);
    if (threadIdx.x == 0) part[(size_t)b * nblk + blockIdx.x] = s;
}

}  // namespace foe
