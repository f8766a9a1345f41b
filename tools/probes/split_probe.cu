// Probe: tf32_split2 (paired Veltkamp) on the GPU against the integer-rounding split.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../../paper_1404_5344_b200/csrc/tc_ptx.cuh"
using namespace foe::tc;
__global__ void k(const float* x, float* hi, float* lo, float* hi2, float* lo2, int n) {
    int i = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (i + 1 >= n) return;
    float2 h, l;
    tf32_split2(make_float2(x[i], x[i + 1]), h, l);
    hi[i] = h.x; hi[i + 1] = h.y; lo[i] = l.x; lo[i + 1] = l.y;
    for (int j = 0; j < 2; ++j) {
        float a = tf32_hi(x[i + j]);
        hi2[i + j] = a; lo2[i + j] = tf32_hi(x[i + j] - a);
    }
}
int main() {
    const int n = 1 << 16;
    std::vector<float> x(n), hi(n), lo(n), hi2(n), lo2(n);
    srand(3);
    for (auto& v : x) v = ((float)rand() / RAND_MAX - 0.5f) * powf(10.f, (float)(rand() % 7 - 3));
    float *dx, *dh, *dl, *dh2, *dl2;
    cudaMalloc(&dx, n * 4); cudaMalloc(&dh, n * 4); cudaMalloc(&dl, n * 4); cudaMalloc(&dh2, n * 4); cudaMalloc(&dl2, n * 4);
    cudaMemcpy(dx, x.data(), n * 4, cudaMemcpyHostToDevice);
    k<<<n / 512, 256>>>(dx, dh, dl, dh2, dl2, n);
    cudaDeviceSynchronize();
    cudaMemcpy(hi.data(), dh, n * 4, cudaMemcpyDeviceToHost); cudaMemcpy(lo.data(), dl, n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hi2.data(), dh2, n * 4, cudaMemcpyDeviceToHost); cudaMemcpy(lo2.data(), dl2, n * 4, cudaMemcpyDeviceToHost);
    double e1 = 0, e2 = 0; int bad = 0;
    for (int i = 0; i < n; ++i) {
        double r1 = fabs(((double)hi[i] + lo[i]) - x[i]) / fabs(x[i]);
        double r2 = fabs(((double)hi2[i] + lo2[i]) - x[i]) / fabs(x[i]);
        e1 = fmax(e1, r1); e2 = fmax(e2, r2);
        unsigned hb; memcpy(&hb, &hi[i], 4);
        if (hb & 0x1FFF) ++bad;
        if (i < 4) printf("x %g hi %g lo %g | hi2 %g lo2 %g\n", x[i], hi[i], lo[i], hi2[i], lo2[i]);
    }
    printf("veltkamp2 max rel %.3e (hi with low bits: %d) ; integer max rel %.3e\n", e1, bad, e2);
    return 0;
}
