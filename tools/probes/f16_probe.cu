// Probe: the kind::f16 (fp16 operands, fp32 accumulate) encodings planned for the next K8.
//  1. forward with A from shared memory as per-u-row im2col "entries" (core matrix rows =
//     8 pixels, K = 8 taps of one filter row) in a 7-slot ring with zero guards, filter-row
//     pairs per K = 16 MMA (a split pair at the ring wrap = two MMAs against the guards), the
//     last MMA pairing row 6 with a per-pixel correction block (different LBO), 3-pass hi/lo
//     split with power-of-two scales.  Checked against fp64.
//  2. backward with A = P (fp16 hi/lo packed two per TMEM column) from TMEM.
//  3. tensor-pipe cycles of a chain of K = 16, N = 48 SS MMAs with these descriptors.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_fp16.h>
#include "../../paper_1404_5344_b200/csrc/tc_ptx.cuh"
using namespace foe::tc;

constexpr int M = 7, NF = 48, L = 128, NG = L / 8, SLOT = NG * 128;   // bytes per ring slot (2 KB)
constexpr int NS = 7;                                                 // ring slots

__host__ __device__ constexpr uint32_t idesc_f16(int m, int n) {
    return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void mma_f16_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
                 "r"(a), "l"(b), "r"(id), "r"(acc));
}
// fp16 hi/lo split of a float pair: hi = rn(x), lo = rn(x - hi)
__device__ __forceinline__ void split_h2(float2 v, uint32_t& hi, uint32_t& lo) {
    const __half2 h = __float22half2_rn(v);
    const float2 hb = __half22float2(h);
    const __half2 l = __float22half2_rn(make_float2(v.x - hb.x, v.y - hb.y));
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = *reinterpret_cast<const uint32_t*>(&l);
}

struct Params {
    const float* u;      // [8 rows][L + 8] u values
    const float* kf;     // [M][M][NF] forward taps (already oriented)
    const float* p;      // [L][NF] backward A
    const float* kb;     // [NF][48] backward B
    float su, sf, sp, sb;
    int base;            // ring slot of row 0
    int pix;             // 1: per-pixel DC shift (c = u[a][q+3]) instead of per (row, group)
    float* R;            // [L][NF] forward result (unscaled, DC restored)
    float* Z;            // [L][48]
    long long* cyc;
};

__global__ void probe(Params pr) {
    extern __shared__ __align__(1024) unsigned char sm[];
    // layout: hi ring [guard][7 slots][guard] | lo ring (same) | A2 hi | A2 lo | Bf hi | Bf lo | Bb hi | Bb lo
    unsigned char* rh = sm;
    unsigned char* rl = rh + (NS + 2) * SLOT;
    unsigned char* a2h = rl + (NS + 2) * SLOT;
    unsigned char* a2l = a2h + SLOT;
    unsigned char* bfh = a2l + SLOT;                  // K = 64 x N = 48 fp16: 6 KB
    unsigned char* bfl = bfh + 64 * NF * 2;
    unsigned char* bbh = bfl + 64 * NF * 2;           // K = 48 x N = 48: 4.5 KB
    unsigned char* bbl = bbh + 48 * 48 * 2;
    __shared__ float cs[8][NG];                       // c_{y,G}
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t mbar;
    const int t = threadIdx.x, warp = t >> 5;
    for (int i = t; i < (NS + 2) * SLOT * 2 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    if (t < 8 * NG) cs[t / NG][t % NG] = pr.u[(t / NG) * (L + 8) + (t % NG) * 8 + 6];
    __syncthreads();
    // B forward: element (k, n), k = chunk*16 + h*8 + e; chunk c < 3: a = 2c + h, b = e; chunk 3:
    // h = 0 -> a = 6, b = e; h = 1 -> correction row a' = e (row sums); b = 7 / a' = 7 -> 0
    for (int i = t; i < 64 * NF; i += blockDim.x) {
        const int k = i / NF, n = i % NF, c = k / 16, h = (k % 16) / 8, e = k % 8;
        float v = 0.f;
        if (c < 3 || h == 0) {
            const int a = c < 3 ? 2 * c + h : 6;
            if (e < M) v = pr.kf[(a * M + e) * NF + n];
        } else if (e < M) {
            for (int b = 0; b < M; ++b) v += pr.kf[(e * M + b) * NF + n];
        }
        v *= pr.sf;
        const __half hh = __float2half_rn(v), hl = __float2half_rn(v - __half2float(hh));
        const int off = c * (2 * NF * 16) + h * (NF * 16) + n * 16 + e * 2;
        *reinterpret_cast<__half*>(bfh + off) = hh;
        *reinterpret_cast<__half*>(bfl + off) = hl;
    }
    for (int i = t; i < 48 * 48; i += blockDim.x) {
        const int k = i / 48, n = i % 48, c = k / 16, h = (k % 16) / 8, e = k % 8;
        const float v = pr.kb[k * 48 + n] * pr.sb;
        const __half hh = __float2half_rn(v), hl = __float2half_rn(v - __half2float(hh));
        const int off = c * (2 * 48 * 16) + h * (48 * 16) + n * 16 + e * 2;
        *reinterpret_cast<__half*>(bbh + off) = hh;
        *reinterpret_cast<__half*>(bbl + off) = hl;
    }
    // ring entries: row a at slot (base + a) % NS; entry of pixel q = 8 halves of
    // (u[a][q + b] - c_{a,G}) * su, b < M, else 0
    if (t < L) {
        const int q = t, G = q / 8, r = q % 8;
        for (int a = 0; a < M; ++a) {
            const int s = (pr.base + a) % NS;
            uint32_t hi[4], lo[4];
            for (int b = 0; b < 8; b += 2) {
                const float ca = pr.pix ? pr.u[a * (L + 8) + q + 3] : cs[a][G];
                const float v0 = b < M ? (pr.u[a * (L + 8) + q + b] - ca) * pr.su : 0.f;
                const float v1 = b + 1 < M ? (pr.u[a * (L + 8) + q + b + 1] - ca) * pr.su : 0.f;
                split_h2(make_float2(v0, v1), hi[b / 2], lo[b / 2]);
            }
            const int off = SLOT * (1 + s) + G * 128 + r * 16;
            *reinterpret_cast<uint4*>(rh + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
            *reinterpret_cast<uint4*>(rl + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        }
        // correction block: (c_{a,G} - c_{3,G}) * su for a < M
        uint32_t hi[4], lo[4];
        for (int a = 0; a < 8; a += 2) {
            auto cc = [&](int aa) { return pr.pix ? pr.u[aa * (L + 8) + q + 3] : cs[aa][G]; };
            const float v0 = a < M ? (cc(a) - cc(3)) * pr.su : 0.f;
            const float v1 = a + 1 < M ? (cc(a + 1) - cc(3)) * pr.su : 0.f;
            split_h2(make_float2(v0, v1), hi[a / 2], lo[a / 2]);
        }
        *reinterpret_cast<uint4*>(a2h + G * 128 + r * 16) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(a2l + G * 128 + r * 16) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
    if (warp == 0) tmem_alloc<256>(&tbase);
    if (t == 0) { mbar_init(&mbar, 1); mbar_fence_init(); }
    fence_proxy_async_smem();
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tb = tbase;
    const uint32_t tl = tb + ((uint32_t)((warp & 3) * 32) << 16);
    // P (backward A) into TMEM columns [128, 152) hi, [152, 176) lo: column c holds halves 2c, 2c+1
    if (t < L) {
        for (int c8 = 0; c8 < 3; ++c8) {
            float h8[8], l8[8];
            for (int e = 0; e < 8; ++e) {
                const int i = (c8 * 8 + e) * 2;
                uint32_t hi, lo;
                split_h2(make_float2(pr.p[t * NF + i] * pr.sp, pr.p[t * NF + i + 1] * pr.sp), hi, lo);
                h8[e] = __uint_as_float(hi);
                l8[e] = __uint_as_float(lo);
            }
            tmem_st8(tl + 128 + c8 * 8, h8);
            tmem_st8(tl + 152 + c8 * 8, l8);
        }
    }
    wait_st();
    fence_before_sync();
    __syncthreads();
    const uint32_t idf = idesc_f16(128, NF), idb = idesc_f16(128, 48);
    const uint32_t srh = smem_u32(rh), srl = smem_u32(rl);
    if (t == 0) {
        fence_after_sync();
        // forward: 3 passes (A_hi B_lo, A_lo B_hi, A_hi B_hi) into D = columns [0, 48)
        int n = 0;
        for (int pass = 0; pass < 3; ++pass) {
            const uint32_t ra = pass == 1 ? srl : srh;
            const uint32_t a2 = smem_u32(pass == 1 ? a2l : a2h);
            const uint32_t bsel = smem_u32(pass == 0 ? bfl : bfh);
            for (int c = 0; c < 4; ++c) {
                const uint64_t bd = sdesc_kmajor(bsel + c * 2 * NF * 16, NF * 16, 128);
                const int a = 2 * c;
                const int s = (pr.base + a) % NS;
                const uint32_t sa = ra + SLOT * (1 + s);
                if (c == 3) {
                    mma_f16_ss(tb, sdesc_kmajor(sa, a2 - sa, 128), bd, idf, n++ > 0);
                } else if (s == NS - 1) {
                    mma_f16_ss(tb, sdesc_kmajor(sa, SLOT, 128), bd, idf, n++ > 0);   // row a | guard
                    mma_f16_ss(tb, sdesc_kmajor(ra, SLOT, 128), bd, idf, n++ > 0);   // guard | row a+1
                } else {
                    mma_f16_ss(tb, sdesc_kmajor(sa, SLOT, 128), bd, idf, n++ > 0);
                }
            }
        }
        // backward: Z = P Kb, columns [64, 112), A from TMEM
        for (int pass = 0; pass < 3; ++pass) {
            const uint32_t acol = pass == 1 ? 152 : 128;
            const uint32_t bsel = smem_u32(pass == 0 ? bbl : bbh);
            for (int c = 0; c < 3; ++c)
                mma_f16_ts(tb + 64, tb + acol + c * 8, sdesc_kmajor(bsel + c * 2 * 48 * 16, 48 * 16, 128), idb,
                           pass > 0 || c > 0);
        }
        mma_commit(&mbar);
    }
    __syncwarp();
    mbar_wait(&mbar, 0);
    fence_after_sync();
    if (t < L) {
        const int G = t / 8;
        float ksum[NF];
        for (int i = 0; i < NF; ++i) {
            double s = 0.0;
            for (int k = 0; k < M * M; ++k) s += pr.kf[k * NF + i];
            ksum[i] = (float)s;
        }
        const float inv = 1.f / (pr.su * pr.sf);
        for (int c = 0; c < NF; c += 8) {
            float v[8];
            tmem_ld8(tl + c, v);
            wait_ld();
            for (int j = 0; j < 8; ++j) pr.R[t * NF + c + j] = v[j] * inv + (pr.pix ? pr.u[3 * (L + 8) + t + 3] : cs[3][G]) * ksum[c + j];
        }
        const float invz = 1.f / (pr.sp * pr.sb);
        for (int c = 0; c < 48; c += 8) {
            float v[8];
            tmem_ld8(tl + 64 + c, v);
            wait_ld();
            for (int j = 0; j < 8; ++j) pr.Z[t * 48 + c + j] = v[j] * invz;
        }
    }
    // 3. rate: chains of 12 SS MMAs (K = 16, N = 48) with a commit + wait per chain
    __syncthreads();
    if (warp == 0) {
        const uint64_t ad = sdesc_kmajor(srh + SLOT, SLOT, 128);
        const uint64_t bd = sdesc_kmajor(smem_u32(bfh), NF * 16, 128);
        const long long c0 = clock64();
        for (int it = 0; it < 200; ++it) {
            for (int k = 0; k < 12; ++k) {
                asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tb + 192),
                             "l"(ad), "l"(bd), "r"(idf), "r"(1u));
            }
            mma_commit_warp(&mbar);
            mbar_wait(&mbar, (uint32_t)((it + 1) & 1));
        }
        const long long c1 = clock64();
        for (int it = 0; it < 200; ++it) {
            for (int k = 0; k < 12; ++k) {
                asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tb + 192),
                             "r"(tb + 128 + (k & 1) * 8), "l"(bd), "r"(idf), "r"(1u));
            }
            mma_commit_warp(&mbar);
            mbar_wait(&mbar, (uint32_t)((it + 201) & 1));
        }
        if (t == 0) { pr.cyc[0] = c1 - c0; pr.cyc[1] = clock64() - c1; }
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 0) tmem_dealloc<256>(tb);
}

int main() {
    srand(7);
    auto U = [] { return (double)rand() / RAND_MAX; };
    std::vector<float> u(8 * (L + 8)), kf(M * M * NF), p(L * NF), kb(NF * 48), R(L * NF), Z(L * 48);
    // u: smooth ramp around 120 + an edge + noise (a piecewise-smooth patch)
    for (int y = 0; y < 8; ++y)
        for (int x = 0; x < L + 8; ++x)
            u[y * (L + 8) + x] = (float)(120.0 + 0.3 * x - 0.7 * y + (x > 70 ? 90.0 : 0.0) + 4.0 * (U() - 0.5));
    for (int i = 0; i < NF; ++i) {
        double s = 0, s2 = 0;
        std::vector<double> k(M * M);
        for (auto& v : k) { v = U() - 0.5; s += v; }
        for (auto& v : k) { v -= s / (M * M); s2 += v * v; }
        for (int j = 0; j < M * M; ++j) kf[j * NF + i] = (float)(k[j] / sqrt(s2));
    }
    for (auto& v : p) v = (float)(U() - 0.5);
    for (auto& v : kb) v = (float)(2.0 * (U() - 0.5));
    float *du, *dkf, *dp, *dkb, *dR, *dZ;
    long long* dc;
    cudaMalloc(&du, u.size() * 4); cudaMalloc(&dkf, kf.size() * 4); cudaMalloc(&dp, p.size() * 4);
    cudaMalloc(&dkb, kb.size() * 4); cudaMalloc(&dR, R.size() * 4); cudaMalloc(&dZ, Z.size() * 4);
    cudaMalloc(&dc, 16);
    cudaMemcpy(du, u.data(), u.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dkf, kf.data(), kf.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dp, p.data(), p.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dkb, kb.data(), kb.size() * 4, cudaMemcpyHostToDevice);
    const int smem = (NS + 2) * SLOT * 2 + 2 * SLOT + 2 * 64 * NF * 2 + 2 * 48 * 48 * 2;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int rc = 0;
    for (int run = 0; run < 2 * NS; ++run) {
        const int base = run % NS, pix = run / NS;
        Params pr{du, dkf, dp, dkb, 64.f, 8192.f, 16384.f, 8192.f, base, pix, dR, dZ, dc};
        probe<<<1, 128, smem>>>(pr);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("kernel: %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(R.data(), dR, R.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(Z.data(), dZ, Z.size() * 4, cudaMemcpyDeviceToHost);
        long long cyc[2];
        cudaMemcpy(cyc, dc, 16, cudaMemcpyDeviceToHost);
        double er = 0, nr = 0, ez = 0, nz = 0, mr = 0, ee = 0, ne = 0;
        for (int q = 0; q < 122; ++q)
            for (int i = 0; i < NF; ++i) {
                double r = 0;
                for (int a = 0; a < M; ++a)
                    for (int b = 0; b < M; ++b) r += (double)kf[(a * M + b) * NF + i] * u[a * (L + 8) + q + b];
                er += (R[q * NF + i] - r) * (R[q * NF + i] - r);
                nr += r * r;
                if (q / 8 * 8 + 13 >= 70 && q / 8 * 8 <= 70) { ee += (R[q * NF + i] - r) * (R[q * NF + i] - r); ne += r * r; }
                mr = fmax(mr, fabs(R[q * NF + i] - r));
            }
        for (int q = 0; q < L; ++q)
            for (int n = 0; n < 48; ++n) {
                double z = 0;
                for (int i = 0; i < NF; ++i) z += (double)p[q * NF + i] * kb[i * 48 + n];
                ez += (Z[q * 48 + n] - z) * (Z[q * 48 + n] - z);
                nz += z * z;
            }
        printf("pix %d base %d: forward rel L2 %.3e (max abs %.3e, edge groups %.3e)  backward rel L2 %.3e  "
               "SS %.1f TS %.1f cycles/MMA\n", pix, base, sqrt(er / nr), mr, sqrt(ee / ne), sqrt(ez / nz),
               cyc[0] / (200.0 * 12), cyc[1] / (200.0 * 12));
        if (!(sqrt(er / nr) < 1e-6 && sqrt(ez / nz) < 1e-6)) rc = 2;
    }
    return rc;
}
