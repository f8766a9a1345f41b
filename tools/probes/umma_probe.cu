// Probe: validate the tcgen05 TF32 MMA encodings of tc_ptx.cuh on a B200.
// D[128 x N] = A[128 x K] . B[K x N], A in TMEM (tcgen05.st), B in smem (K-major, no swizzle),
// single pass (tf32-rounded operands, compared exactly against fp64 on the rounded values)
// and 3xTF32 (hi/lo split, compared against fp64 on the fp32 values).
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../../paper_1404_5344_b200/csrc/tc_ptx.cuh"
using namespace foe::tc;

constexpr int M = 128, K = 16, N = 48;

__global__ void probe(const float* A, const float* B, float* D1, float* D3) {
    __shared__ __align__(128) float bs_hi[K * N];
    __shared__ __align__(128) float bs_lo[K * N];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t mbar;
    const int t = threadIdx.x, warp = t >> 5;
    for (int i = t; i < K * N; i += blockDim.x) {
        const int k = i / N, n = i % N;           // B[k][n]
        const float v = B[i];
        const float hi = to_tf32(v), lo = to_tf32(v - hi);
        const int off = (k / 4) * (N * 4) + n * 4 + (k % 4);   // [kc][n][4]
        bs_hi[off] = hi; bs_lo[off] = lo;
    }
    if (warp == 0) tmem_alloc<256>(&tbase);
    if (t == 0) { mbar_init(&mbar, 1); mbar_fence_init(); }
    fence_proxy_async_smem();
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tb = tbase;
    const uint32_t lane_addr = tb + ((uint32_t)(warp * 32) << 16);
    // A row t: cols [0,K) hi, [K,2K) lo
    for (int c = 0; c < K; c += 8) {
        float h[8], l[8];
        for (int j = 0; j < 8; ++j) {
            const float v = A[t * K + c + j];
            h[j] = to_tf32(v); l[j] = to_tf32(v - h[j]);
        }
        tmem_st8(lane_addr + c, h);
        tmem_st8(lane_addr + K + c, l);
    }
    wait_st();
    fence_before_sync();
    __syncthreads();
    const uint32_t id = idesc_tf32(M, N);
    const uint32_t D1c = 64, D3c = 128;
    if (t == 0) {
        fence_after_sync();
        for (int s = 0; s < K / 8; ++s) {
            const uint64_t bh = sdesc_kmajor(smem_u32(bs_hi) + s * 2 * N * 16, N * 16, 128);
            const uint64_t bl = sdesc_kmajor(smem_u32(bs_lo) + s * 2 * N * 16, N * 16, 128);
            mma_tf32_ts(tb + D1c, tb + s * 8, bh, id, s > 0);
            mma_tf32_ts(tb + D3c, tb + s * 8, bh, id, s > 0);          // hi.hi
            mma_tf32_ts(tb + D3c, tb + s * 8, bl, id, 1);              // hi.lo
            mma_tf32_ts(tb + D3c, tb + K + s * 8, bh, id, 1);          // lo.hi
        }
        mma_commit(&mbar);
    }
    __syncwarp();
    mbar_wait(&mbar, 0);
    fence_after_sync();
    for (int c = 0; c < N; c += 8) {
        float v[8];
        tmem_ld8(lane_addr + D1c + c, v);
        wait_ld();
        for (int j = 0; j < 8; ++j) D1[t * N + c + j] = v[j];
        tmem_ld8(lane_addr + D3c + c, v);
        wait_ld();
        for (int j = 0; j < 8; ++j) D3[t * N + c + j] = v[j];
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 0) tmem_dealloc<256>(tb);
}

static float tf32h(float x) {  // host emulation of cvt.rna.tf32
    uint32_t u; memcpy(&u, &x, 4);
    u = (u + 0x1000u) & 0xFFFFE000u;
    float r; memcpy(&r, &u, 4); return r;
}

int main() {
    std::vector<float> A(M * K), B(K * N), D1(M * N), D3(M * N);
    srand(1);
    for (auto& x : A) x = (float)rand() / RAND_MAX * 2 - 1;
    for (auto& x : B) x = (float)rand() / RAND_MAX * 2 - 1;
    float *dA, *dB, *dD1, *dD3;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD1, D1.size() * 4); cudaMalloc(&dD3, D3.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    probe<<<1, 128>>>(dA, dB, dD1, dD3);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    cudaMemcpy(D1.data(), dD1, D1.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(D3.data(), dD3, D3.size() * 4, cudaMemcpyDeviceToHost);
    double e1 = 0, e3 = 0, n2 = 0, e1x = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double r = 0, r1 = 0;
            for (int k = 0; k < K; ++k) {
                r += (double)A[m * K + k] * B[k * N + n];
                r1 += (double)tf32h(A[m * K + k]) * tf32h(B[k * N + n]);
            }
            e1 += (D1[m * N + n] - r1) * (D1[m * N + n] - r1);
            e1x = fmax(e1x, fabs(D1[m * N + n] - r1));
            e3 += (D3[m * N + n] - r) * (D3[m * N + n] - r);
            n2 += r * r;
        }
    printf("1xTF32 vs fp64(tf32 operands): rel L2 %.3e (max abs %.3e)\n", sqrt(e1 / n2), e1x);
    printf("3xTF32 vs fp64: rel L2 %.3e\n", sqrt(e3 / n2));
    printf("D1[0..3] %f %f %f %f\n", D1[0], D1[1], D1[2], D1[3]);
    return (sqrt(e1 / n2) < 1e-6 && sqrt(e3 / n2) < 1e-6) ? 0 : 2;
}
