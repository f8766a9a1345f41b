// foe_api.cu -- C ABI of libfoe (include/foe.h): model, energy/gradient, Lipschitz
// estimate and the device-controlled iPiano solver loop.  Host code only orchestrates
// launches of the kernels in foe_kernels.cuh; every step of the method runs on the GPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "foe.h"
#include "foe_kernels.cuh"
#include "foe_tc.cuh"
#include "foe_th.cuh"
#include <cuda_fp16.h>
#include "foe_eval.cuh"
#include "foe_persist.cuh"

using foe::ImgCtl;
using foe::K1Args;
using foe::kThreads;
using foe::kTile;
using foe::TapParams;

namespace {

thread_local std::string g_err;
std::atomic<long long> g_launches{0};  // kernels launched by this library (process-wide)
thread_local bool t_capturing = false;   // graph capture: replays are counted instead
thread_local bool t_slab_member = false; // ipiano_slabs_create is creating its member states
thread_local int t_force_ncp = 0;        // ... with the whole scene's K1 chunk size
thread_local int t_force_pxt = 0;        // ... and the group's K2 pixels per thread
inline void count_launch(long long n) {
    if (!t_capturing) g_launches.fetch_add(n, std::memory_order_relaxed);
}

foe_status fail(foe_status s, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

foe_status cuda_fail(cudaError_t e, const char* what, int line) {
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? FOE_ERR_OUT_OF_MEMORY : FOE_ERR_CUDA,
                "%s failed: %s (foe_api.cu:%d)", what, cudaGetErrorString(e), line);
}

#define CK(call)                                                        \
    do {                                                                \
        cudaError_t e_ = (call);                                        \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call, __LINE__);   \
    } while (0)
#define CKL(what)                                                       \
    do {                                                                \
        cudaError_t e_ = cudaGetLastError();                            \
        if (e_ != cudaSuccess) return cuda_fail(e_, what, __LINE__);    \
    } while (0)

// Kernel configuration per filter size: NC filters per shared-memory chunk, SF forward
// rows per thread item (K1), SFH for the HVP variant.
template <int M> struct Tr;
template <> struct Tr<7> { static constexpr int NC = 4, SF = 7, SFH = 5; };
template <> struct Tr<5> { static constexpr int NC = 4, SF = 4, SFH = 4; };
template <> struct Tr<3> { static constexpr int NC = 4, SF = 6, SFH = 6; };

template <int M, bool HVP>
constexpr int smem_bytes() {
    using G = foe::K1Geom<M, Tr<M>::NC, HVP ? Tr<M>::SFH : Tr<M>::SF>;
    return (HVP ? G::SMEM_FLOATS_HVP : G::SMEM_FLOATS) * 4;
}

template <int M, bool HVP>
cudaError_t k1_set_attr() {
    constexpr int SF = HVP ? Tr<M>::SFH : Tr<M>::SF;
    return cudaFuncSetAttribute(foe::k_prior_grad<M, Tr<M>::NC, SF, HVP>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<M, HVP>());
}

template <int M, bool HVP>
void k1_launch(const K1Args& a, const TapParams& tp, dim3 grid, cudaStream_t s) {
    constexpr int SF = HVP ? Tr<M>::SFH : Tr<M>::SF;
    foe::k_prior_grad<M, Tr<M>::NC, SF, HVP><<<grid, kThreads, smem_bytes<M, HVP>(), s>>>(a, tp);
}

// K1 v2 (paired FFMA2): NCP filter pairs per shared-memory chunk, SF forward rows per item
// (chunks of 1 pair for images too small to fill the GPU with 2-pair chunks: plan_stencil)
constexpr int kNCP = 2, kSF2 = 5;
template <int M, int NCP = kNCP>
constexpr int smem2_bytes() { return foe::G2<M, NCP, kSF2>::SMEM_BYTES; }
template <int M>
cudaError_t k2g_set_attr() {
    cudaError_t e = cudaFuncSetAttribute(foe::k_prior_grad2<M, kNCP, kSF2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         smem2_bytes<M>());
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(foe::k_prior_grad2<M, 1, kSF2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem2_bytes<M, 1>());
}
template <int M>
void k2g_launch(const K1Args& a, const foe::TapParams2& tp, dim3 grid, cudaStream_t s) {
    if (a.ncp == 1) foe::k_prior_grad2<M, 1, kSF2><<<grid, kThreads, smem2_bytes<M, 1>(), s>>>(a, tp);
    else foe::k_prior_grad2<M, kNCP, kSF2><<<grid, kThreads, smem2_bytes<M>(), s>>>(a, tp);
}

// hvp: the v1 stencil (setup only); gradient/energy: the v2 paired-FMA stencil
void k1_dispatch(int m, bool hvp, const K1Args& a, const TapParams& tp, const foe::TapParams2& tp2, dim3 grid,
                 cudaStream_t s) {
    count_launch(1);
    switch (m) {
        case 7: hvp ? k1_launch<7, true>(a, tp, grid, s) : k2g_launch<7>(a, tp2, grid, s); break;
        case 5: hvp ? k1_launch<5, true>(a, tp, grid, s) : k2g_launch<5>(a, tp2, grid, s); break;
        default: hvp ? k1_launch<3, true>(a, tp, grid, s) : k2g_launch<3>(a, tp2, grid, s); break;
    }
}

// K8 (tensor-core stencil): output tile rows -- 64 (the bands of the slab path, and the batch
// path when the launch fills the GPU), or 32 / 16 for single images that cannot fill 148 SMs with
// 64-row tiles (plan_stencil)
constexpr int kTcR = 64;
// 1: the Lipschitz estimate's HVPs after the first read S_i = rho''(K_i u)/2 stored by the first
// (k_hvp_s); 0: every HVP recomputes it (A/B knob)
#ifndef FOE_HVP_STORE_S
#define FOE_HVP_STORE_S 1
#endif
// 1: the batch path's K8 tiles compute their own rows' responses only (no row halos; the partial
// sums of the rows near band edges meet in K2); 0: tiles with row halos (A/B knob)
#ifndef FOE_K8_NH
#define FOE_K8_NH 1
#endif
// 1: ... and without column halos when 128-column tiles tile W (A/B knob)
#ifndef FOE_K8_NHC
#define FOE_K8_NHC 1
#endif
template <int M, int NP, int R>
constexpr int th_smem() { return foe::ThGeom<M, NP, R>::SMEM_BYTES; }
template <int M, int NP, int R, int MODE>
cudaError_t th_attr() {
    return cudaFuncSetAttribute(foe::k_prior_grad_th<M, NP, R, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                th_smem<M, NP, R>());
}
template <int M, int NP>
cudaError_t tc_set_attr() {
    cudaError_t e = cudaFuncSetAttribute(foe::k_hvp_th<M, NP, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         foe::ThHGeom<M, NP, 64>::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(foe::k_hvp_s<M, NP, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, th_smem<M, NP, 64>());
    if (e != cudaSuccess) return e;
    const cudaError_t es[] = {th_attr<M, NP, 64, 0>(), th_attr<M, NP, 32, 0>(), th_attr<M, NP, 16, 0>(),
                              th_attr<M, NP, 8, 0>(),  th_attr<M, NP, 4, 0>(),  th_attr<M, NP, 64, 1>(),
                              th_attr<M, NP, 32, 1>(), th_attr<M, NP, 16, 1>(), th_attr<M, NP, 8, 1>(),
                              th_attr<M, NP, 4, 1>(),  th_attr<M, NP, 64, 2>(), th_attr<M, NP, 32, 2>(),
                              th_attr<M, NP, 16, 2>(), th_attr<M, NP, 8, 2>(),  th_attr<M, NP, 4, 2>()};
    for (cudaError_t x : es)
        if (x != cudaSuccess) return x;
    return cudaSuccess;
}
// the banks K8 has an instantiation for: (m, padded N_f)
int tc_np(int m, int nf) {
    if (m == 7 && nf <= 48) return 48;
    if (m == 5 && nf <= 32) return 32;
    return 0;
}

constexpr int kPxt2 = 8;  // pixels per thread of the pointwise kernels

// Launch with programmatic stream serialization (PDL): the kernel may be scheduled while its
// predecessor on the stream drains; it calls pdl_wait() before touching the predecessor's output
// (foe_kernels.cuh).  Used for the graph driver's trial rounds K2 -> K8 -> K3.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    cudaLaunchConfig_t c = {};
    c.gridDim = grid;
    c.blockDim = block;
    c.dynamicSmemBytes = smem;
    c.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    c.attrs = at;
    c.numAttrs = 1;
    return cudaLaunchKernelEx(&c, kern, std::forward<Args>(args)...);
}

int div_up(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace

// ------------------------------------------------------------------------------- model

struct foe_model {
    int dev = 0, nf = 0, m = 0, nsm = 148;
    foe_data_term term = FOE_DATA_COMBINED;
    double lam[2] = {0, 0};
    TapParams* tp = nullptr;        // host copy, passed by value to the HVP stencil launches
    foe::TapParams2* tp2 = nullptr; // pair-interleaved taps of the paired-FMA stencil
    // K8 (fp16 tensor cores, foe_th.cuh): fp16 hi/lo B images and the epilogue constants
    int tc_np = 0;                  // padded N_f of the K8 instantiation (0: no K8 for this bank)
    unsigned char* th_bimg = nullptr;
    foe::ThConst* th_const = nullptr;
    int stencil = FOE_STENCIL_AUTO; // foe_energy_grad's choice
    bool persist_phases = false;
    cudaMemPool_t pool = nullptr;   // private stream-ordered pool of the per-call scratch    // FOE_PERSIST_PHASES=1 (read once here): persistent-driver phase timings
    // ipiano_run's reusable workspace (one solver state + host-I/O staging buffers), kept for
    // repeated calls of the same shape and configuration; guarded by run_mu (a concurrent call
    // falls back to a private workspace)
    mutable std::mutex run_mu;
    mutable ipiano_state* run_state = nullptr;
    mutable float* io_buf = nullptr;   // [2][n] device staging of host f and u
    mutable size_t io_n = 0;
    // foe_estimate_lipschitz's S_i = rho''(K_i u)/2 buffer ([B][NP][H][W] fp32, grown on demand),
    // guarded by s_mu (a concurrent estimate recomputes K u in every HVP instead)
    mutable std::mutex s_mu;
    mutable float* s_buf = nullptr;
    mutable size_t s_n = 0;
};

struct ipiano_state {
    const foe_model* model = nullptr;
    int B = 0, H = 0, W = 0;
    size_t HW = 0;
    ipiano_config cfg{};
    ipiano_config cfg_in{};   // the configuration as the caller passed it (ipiano_run's cache key)
    foe::SolverParams sp{};
    int tiles_x = 0, ntiles = 0, groups = 1, nchunks = 0, nblk2 = 0;
    int ncp = 2;                  // K1: filter pairs per chunk (plan_stencil)
    int pxt2 = 8;                 // pixels per thread of K2 (nblk2 = HW / (kThreads pxt2) blocks)
    int kind = FOE_STENCIL_FFMA;  // resolved stencil of this state (K1 or K8)
    int tc_rem = 0, tc_spt = 0;   // K8 column packing of this state's plan
    int tc_rows = 64;             // K8 output rows per tile
    int nblk3 = 0;                // test partials per image K3 sums (= the K2 blocks)
    int solver = FOE_SOLVER_GRAPH;  // resolved trial-loop driver
    int pgrid = 0;                // persistent driver: co-resident CTAs
    unsigned int* bar = nullptr;  // persistent driver: grid barrier counter
    unsigned long long* phase_ns = nullptr;  // FOE_PERSIST_PHASES=1: CTA 0's phase timestamps
    double* w = nullptr;      // [3][B][HW]
    float* g = nullptr;       // [2][groups][B][HW]
    float* gedge = nullptr;   // K8 without row halos: [2][B][H / tc_rows][2C][W] band-boundary shares
    unsigned int* tcnt = nullptr;   // ... and their arrival counters [3][B][H / tc_rows][tiles_x + 1]
    float* gright = nullptr;        // K8 without column halos: [2][B][W / 128][H][2C]
    float* gcorner = nullptr;       // ... [2][B][H / tc_rows][W / 128][2C][2C]
    int tc_mode = 0;                // K8: 0 halos, 1 no row halos, 2 no row / column halos
    float* ft = nullptr;      // [B][HW]
    double* epart = nullptr;  // [B][ntiles*groups]
    double* ppart = nullptr;  // [2][B][nblk2][8] (buffer 1: the persistent driver's odd rounds)
    double* trace = nullptr;  // [B][max_iters+1][8]
    ImgCtl* ctl = nullptr;    // [B] ([pgrid][B] with the persistent driver: per-CTA copies)
    ImgCtl* hctl = nullptr;   // pinned mirror
    std::vector<double> lam;  // [B][2]
    cudaStream_t s = nullptr;
    cudaEvent_t sync_ev = nullptr;
    cudaGraphExec_t graph = nullptr;
    int graph_rounds = 0;
    bool profile = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_live, ev_live_k2;
    double k1_ms = 0.0, k2_ms = 0.0;
    long long k1_launches = 0, total_launches = 0, k2_launches = 0;
};

namespace {

// K8 fp16 operand images (foe_th.cuh), element (k, n) of a K-major B matrix at half offset
// chunk(k/16) * 2 N 8 + ((k % 16) / 8) N 8 + n 8 + k % 8, hi image then lo image:
//   forward  Kf[k][i], k = 16 c + 8 h + e: ring slot 2c + h of the response row's window; slot 0
//            (A2) carries the row sums ks[e][i] = sum_b fwd_i[e][b], slot 1 + a the taps fwd_i[a][e]
//            (e < m; fwd = the flipped taps); x s_f
//   backward Kb[i][t] = 2 theta_i k_i[t] for t < NB (N padded to NBP), x s_b
// hi = fp16(v), lo = fp16(v - hi) (from the fp64 value); s_f, s_b = 2^(13 - e) with 2^e <= max|v|.
foe_status build_th_images(foe_model* md) {
    const int m = md->m, nf = md->nf, NP = md->tc_np, TAPS = m * m;
    const int NCH = (m + 1) / 2, NB = foe::th_nb(m), NBP = ((NB + 15) / 16) * 16, NKB = NP / 16;
    const size_t BF = (size_t)NCH * 16 * NP, BB = (size_t)NKB * 16 * NBP;   // halves per image
    std::vector<double> kf((size_t)NCH * 16 * NP, 0.0), kb((size_t)NP * NBP, 0.0);
    for (int i = 0; i < nf; ++i) {
        const float* fw = md->tp->fwd + (size_t)i * TAPS;
        for (int k = 0; k < NCH * 16; ++k) {
            const int slot = k / 8, e = k % 8;
            double v = 0.0;
            if (slot == 0) {
                if (e < m) for (int b2 = 0; b2 < m; ++b2) v += (double)fw[e * m + b2];
            } else if (slot - 1 < m && e < m) {
                v = (double)fw[(slot - 1) * m + e];
            }
            kf[(size_t)k * NP + i] = v;
        }
        for (int t = 0; t < NB; ++t)   // column = the tap's Z column (foe::th_zcol: col2im read order)
            kb[(size_t)i * NBP + foe::th_zcol(m, t / m, t % m)] = (double)md->tp->bwd[(size_t)i * TAPS + t];
    }
    auto scale_of = [](const std::vector<double>& v) {
        double mx = 0.0;
        for (double x : v) mx = std::max(mx, std::fabs(x));
        if (!(mx > 0.0)) return 1.0;
        return std::ldexp(1.0, 13 - std::ilogb(mx));
    };
    const double sf = scale_of(kf), sb = scale_of(kb);
    std::vector<__half> img(2 * BF + 2 * BB, __float2half_rn(0.0f));
    auto put = [&](size_t base, size_t nimg, int N, int k, int n, double v) {
        const size_t off = (size_t)(k / 16) * 2 * N * 8 + (size_t)((k % 16) / 8) * N * 8 + (size_t)n * 8 + k % 8;
        const __half h = __float2half_rn((float)v);
        img[base + off] = h;
        img[base + nimg + off] = __float2half_rn((float)(v - (double)__half2float(h)));
    };
    for (int k = 0; k < NCH * 16; ++k)
        for (int i = 0; i < NP; ++i) put(0, BF, NP, k, i, kf[(size_t)k * NP + i] * sf);
    for (int i = 0; i < NP; ++i)
        for (int t = 0; t < NBP; ++t) put(2 * BF, BB, NBP, i, t, kb[(size_t)i * NBP + t] * sb);
    md->th_const = new (std::nothrow) foe::ThConst();
    if (!md->th_const) return fail(FOE_ERR_OUT_OF_MEMORY, "host allocation");
    std::memset(md->th_const, 0, sizeof(foe::ThConst));
    for (int i = 0; i < nf; ++i) {
        md->th_const->sumk[i] = md->tp->sumk[i];
        md->th_const->thl[i] = (float)md->tp->theta_ln2[i];
        md->th_const->kbl[i] = (float)((double)md->tp->bwd[(size_t)i * TAPS + TAPS - 1] * sb);   // x P's 2^14 = Z units
    }
    md->th_const->inv_sf = (float)(1.0 / sf);
    md->th_const->inv_z = (float)(1.0 / (sb * (double)foe::kThPScale));
    double kabs = 0.0;
    for (int i = 0; i < nf; ++i) {
        double t = 0.0;
        for (int k = 0; k < TAPS; ++k) t += std::fabs((double)md->tp->fwd[(size_t)i * TAPS + k]);
        kabs = std::max(kabs, t);
    }
    md->th_const->kabs = (float)kabs;
    CK(cudaMalloc((void**)&md->th_bimg, img.size() * sizeof(__half)));
    CK(cudaMemcpy(md->th_bimg, img.data(), img.size() * sizeof(__half), cudaMemcpyHostToDevice));
    return FOE_OK;
}

}  // namespace

extern "C" {

const char* foe_last_error(void) { return g_err.c_str(); }

const char* foe_status_string(foe_status s) {
    switch (s) {
        case FOE_OK: return "FOE_OK";
        case FOE_ERR_INVALID_ARGUMENT: return "FOE_ERR_INVALID_ARGUMENT";
        case FOE_ERR_CUDA: return "FOE_ERR_CUDA";
        case FOE_ERR_OUT_OF_MEMORY: return "FOE_ERR_OUT_OF_MEMORY";
        case FOE_ERR_NONFINITE: return "FOE_ERR_NONFINITE";
        case FOE_ERR_BACKTRACK_LIMIT: return "FOE_ERR_BACKTRACK_LIMIT";
        case FOE_ERR_PROX_NO_CONVERGENCE: return "FOE_ERR_PROX_NO_CONVERGENCE";
        case FOE_ERR_DOMAIN: return "FOE_ERR_DOMAIN";
        case FOE_ERR_COMM: return "FOE_ERR_COMM";
        case FOE_ERR_UNSUPPORTED: return "FOE_ERR_UNSUPPORTED";
    }
    return "FOE_ERR_UNKNOWN";
}

const char* foe_version(void) { return "libfoe 0.1.0 sm_100a"; }

long long foe_kernel_launches(void) { return g_launches.load(); }

foe_status foe_model_create(const float* filters, int n_filters, int m, const float* alphas,
                            const double* lambda, double looks_L, foe_data_term term,
                            int cuda_device, foe_model** out) {
    if (!out) return fail(FOE_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (!filters) return fail(FOE_ERR_INVALID_ARGUMENT, "filters is NULL");
    if (!alphas) return fail(FOE_ERR_INVALID_ARGUMENT, "alphas is NULL");
    if (m < 3 || m % 2 == 0) return fail(FOE_ERR_INVALID_ARGUMENT, "filter side m=%d must be odd and >= 3", m);
    if (m != 3 && m != 5 && m != 7) return fail(FOE_ERR_UNSUPPORTED, "filter side m=%d: this build has kernels for m in {3,5,7}", m);
    if (n_filters < 1 || n_filters > foe::kMaxFilters)
        return fail(FOE_ERR_INVALID_ARGUMENT, "n_filters=%d outside [1,%d]", n_filters, foe::kMaxFilters);
    if ((long long)n_filters * m * m > foe::kMaxTaps)
        return fail(FOE_ERR_INVALID_ARGUMENT, "n_filters*m*m=%d exceeds %d", n_filters * m * m, foe::kMaxTaps);
    if (term != FOE_DATA_COMBINED && term != FOE_DATA_NAKAGAMI && term != FOE_DATA_IDIV)
        return fail(FOE_ERR_INVALID_ARGUMENT, "unknown data term %d", (int)term);
    if (term == FOE_DATA_IDIV && !lambda)
        return fail(FOE_ERR_INVALID_ARGUMENT, "FOE_DATA_IDIV needs an explicit lambda (PAPER.md:231 prints none)");
    for (int i = 0; i < n_filters; ++i) {
        if (!(alphas[i] > 0.0f) || !std::isfinite(alphas[i]))
            return fail(FOE_ERR_INVALID_ARGUMENT, "non-positive weight at filter %d (theta=%g)", i, (double)alphas[i]);
        for (int t = 0; t < m * m; ++t)
            if (!std::isfinite(filters[i * m * m + t]))
                return fail(FOE_ERR_INVALID_ARGUMENT, "non-finite tap at filter %d", i);
    }
    double lam[2];
    if (lambda) {
        lam[0] = lambda[0];
        lam[1] = lambda[1];
    } else {
        // PAPER.md:272-274 (Sec. III-B) and :389 (Sec. III-C)
        if (looks_L == 8) { lam[0] = 550; lam[1] = 0.02; }
        else if (looks_L == 3) { lam[0] = 310; lam[1] = 0.008; }
        else if (looks_L == 1) { lam[0] = 160; lam[1] = 0.004; }
        else if (looks_L == 5) { lam[0] = 50; lam[1] = 0.15; }
        else return fail(FOE_ERR_INVALID_ARGUMENT, "lambda is NULL and looks_L=%g has no preset (1,3,5,8)", looks_L);
    }
    if (term == FOE_DATA_NAKAGAMI || term == FOE_DATA_IDIV) lam[1] = 0.0;
    if (!(lam[0] >= 0) || !(lam[1] >= 0) || !std::isfinite(lam[0]) || !std::isfinite(lam[1]) ||
        (lam[0] == 0 && lam[1] == 0))
        return fail(FOE_ERR_INVALID_ARGUMENT, "lambda=(%g,%g) must be finite, >= 0 and not both 0", lam[0], lam[1]);

    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (cuda_device < 0 || cuda_device >= ndev)
        return fail(FOE_ERR_INVALID_ARGUMENT, "cuda_device=%d outside [0,%d)", cuda_device, ndev);
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, cuda_device));
    if (prop.major != 10 || prop.minor != 0)
        return fail(FOE_ERR_CUDA, "libfoe is built for sm_100a (B200); device %d is sm_%d%d", cuda_device,
                    prop.major, prop.minor);
    CK(cudaSetDevice(cuda_device));
    if (tc_np(m, n_filters) == 48) CK((tc_set_attr<7, 48>()));
    if (tc_np(m, n_filters) == 32) CK((tc_set_attr<5, 32>()));
    switch (m) {
        case 7: CK((k2g_set_attr<7>())); CK((k1_set_attr<7, true>())); break;
        case 5: CK((k2g_set_attr<5>())); CK((k1_set_attr<5, true>())); break;
        default: CK((k2g_set_attr<3>())); CK((k1_set_attr<3, true>())); break;
    }

    foe_model* md = new (std::nothrow) foe_model();
    if (!md) return fail(FOE_ERR_OUT_OF_MEMORY, "host allocation");
    md->tp = new (std::nothrow) TapParams();
    md->tp2 = new (std::nothrow) foe::TapParams2();
    if (!md->tp || !md->tp2) { delete md->tp; delete md->tp2; delete md; return fail(FOE_ERR_OUT_OF_MEMORY, "host allocation"); }
    std::memset(md->tp, 0, sizeof(TapParams));
    std::memset(md->tp2, 0, sizeof(foe::TapParams2));
    md->dev = cuda_device;
    {   // the per-call scratch of foe_energy_grad / foe_hvp / foe_estimate_lipschitz / ipiano_run comes
        // from a stream-ordered pool private to the model (the device's default pool and its release
        // threshold are left alone): up to 256 MB stay mapped between calls instead of going back to
        // the driver at every synchronisation (remapping cost ~0.2-1 ms per call)
        cudaMemPoolProps pp{};
        pp.allocType = cudaMemAllocationTypePinned;
        pp.location.type = cudaMemLocationTypeDevice;
        pp.location.id = cuda_device;
        if (cudaMemPoolCreate(&md->pool, &pp) != cudaSuccess) {
            delete md->tp; delete md->tp2; delete md;
            return fail(FOE_ERR_CUDA, "cudaMemPoolCreate failed");
        }
        // the pool keeps up to 4 GiB mapped between calls (a c4 Lipschitz estimate's scratch is
        // 0.4 GB: released and re-mapped on every call at a 256 MB threshold, tens of ms); the
        // pool is private to the model and released with it
        uint64_t keep = 4ull << 30;
        cudaMemPoolSetAttribute(md->pool, cudaMemPoolAttrReleaseThreshold, &keep);
        cudaGetLastError();
    }
    md->nf = n_filters;
    md->m = m;
    md->nsm = prop.multiProcessorCount;
    md->term = term;
    {
        const char* ph = std::getenv("FOE_PERSIST_PHASES");   // diagnostics only, read once
        md->persist_phases = ph != nullptr && ph[0] == '1';
    }
    md->lam[0] = lam[0];
    md->lam[1] = lam[1];
    for (int i = 0; i < n_filters; ++i) {
        const float* k = filters + (size_t)i * m * m;
        double s = 0.0;
        for (int a = 0; a < m; ++a)
            for (int b = 0; b < m; ++b) {
                // forward: K_i u (true convolution) = correlation with the flipped kernel
                md->tp->fwd[i * m * m + a * m + b] = k[(m - 1 - a) * m + (m - 1 - b)];
                // backward: theta_i K_i^T = correlation with theta_i k_i; x2 of rho'(x)=2x/(1+x^2)
                md->tp->bwd[i * m * m + a * m + b] = (float)(2.0 * (double)alphas[i] * (double)k[a * m + b]);
                s += (double)k[a * m + b];
            }
        md->tp->sumk[i] = (float)s;
        md->tp->theta_ln2[i] = (double)alphas[i] * 0.69314718055994530942;
        // pair layout: filter i is lane (i & 1) of pair i/2; an odd N_f leaves a zero partner
        const int pr = i / 2, ln = i & 1;
        for (int t = 0; t < m * m; ++t) {
            float* f2 = reinterpret_cast<float*>(&md->tp2->fwd[pr * m * m + t]);
            float* b2 = reinterpret_cast<float*>(&md->tp2->bwd[pr * m * m + t]);
            f2[ln] = md->tp->fwd[i * m * m + t];
            b2[ln] = md->tp->bwd[i * m * m + t];
        }
        md->tp2->sumk[i] = md->tp->sumk[i];
        md->tp2->theta_ln2[i] = md->tp->theta_ln2[i];
    }
    md->tc_np = tc_np(m, n_filters);
    if (md->tc_np) {
        foe_status r = build_th_images(md);
        if (r != FOE_OK) { foe_model_destroy(md); return r; }
    }
    *out = md;
    return FOE_OK;
}

foe_status foe_model_set_stencil(foe_model* model, int stencil) {
    if (!model) return fail(FOE_ERR_INVALID_ARGUMENT, "model is NULL");
    if (stencil < FOE_STENCIL_AUTO || stencil > FOE_STENCIL_TENSOR)
        return fail(FOE_ERR_INVALID_ARGUMENT, "unknown stencil %d", stencil);
    if (stencil == FOE_STENCIL_TENSOR && !model->tc_np)
        return fail(FOE_ERR_UNSUPPORTED, "no tensor-core stencil for %d filters of %dx%d (m=7: N_f<=48, m=5: N_f<=32)",
                    model->nf, model->m, model->m);
    model->stencil = stencil;
    return FOE_OK;
}

void foe_model_destroy(foe_model* model) {
    if (!model) return;
    if (model->run_state) ipiano_state_destroy(model->run_state);
    if (model->io_buf) cudaFree(model->io_buf);
    if (model->s_buf) cudaFree(model->s_buf);
    if (model->th_bimg) cudaFree(model->th_bimg);
    delete model->th_const;
    // outstanding stream-ordered frees are honoured: the pool is released once they land
    if (model->pool) cudaMemPoolDestroy(model->pool);
    delete model->tp;
    delete model->tp2;
    delete model;
    cudaGetLastError();   // destroy reports nothing: leave no stale error for the next launch check
}

}  // extern "C"

// ------------------------------------------------------------------------ helpers

namespace {

// Choose the number of filter groups (split-N_f) so that a launch fills the machine.
int choose_groups(const foe_model* md, int ntiles, int B, int requested, int nchunks) {
    if (requested > 0) return std::min(requested, nchunks);
    const long long slots = 2LL * md->nsm;  // 2 CTAs / SM
    double best = 1e30;
    int bg = 1;
    for (int g = 1; g <= nchunks; ++g) {
        const long long ctas = (long long)ntiles * B * g;
        const double waves = std::ceil((double)ctas / (double)slots);
        const double per = std::ceil((double)nchunks / g) + 0.15;  // chunk work + staging/epilogue
        const double cost = waves * per;
        if (cost < best - 1e-9) { best = cost; bg = g; }
    }
    return bg;
}

// Stencil plan of one evaluation over B images of H x W: kernel, tiling and energy partials.
// H_grid: rows that decide whether a K8 launch fills the GPU (the whole scene for slabs).
struct Plan {
    int kind = FOE_STENCIL_FFMA;
    int tiles_x = 0, ntiles = 0, groups = 1;
    int tc_rem = 0, tc_spt = 0;   // K8 column packing (K1Args::tc_rem / tc_spt)
    int tc_rows = 64;             // K8 output rows per tile (v7: chosen per problem)
    int tc_mode = 0;              // K8: 0 halos, 1 no row halos, 2 no row / column halos (foe_th.cuh)
    int ncp = kNCP, nchunks = 0;  // K1: filter pairs per chunk, chunks
};
Plan plan_stencil(const foe_model* md, int B, int H, int W, int H_grid, int pref, int req_groups,
                  bool allow_pack = true, int req_rows = 0, bool allow_nh = false) {
    Plan p;
    const int ow = 128 - (md->m - 1);
    const bool pack_ok = allow_pack && H_grid == H;
    // K8 tiling with R output rows: full tiles of ow columns per band of R rows; the remainder
    // columns of several bands share one packed tile (not for row slabs, whose energy partials are
    // per 64-row band)
    auto tiling = [&](int R, Plan& q) {
        // the batch path's tiles without row halos (bands of R that tile H, R >= 2C), and without
        // column halos when 128-column tiles tile W (foe_th.cuh MODE 1 / 2)
        q.tc_mode = FOE_K8_NH && allow_nh && pack_ok && H % R == 0 && R >= md->m - 1 ? 1 : 0;
        if (q.tc_mode == 1 && FOE_K8_NHC && W % 128 == 0) {
            q.tc_mode = 2;
            q.tiles_x = W / 128;
            q.ntiles = (H / R) * q.tiles_x;
            q.tc_rem = 0;
            q.tc_spt = 0;
            q.tc_rows = R;
            return;
        }
        int nfull = W / ow, rem = W - nfull * ow, spt = 0;
        if (rem > 0 && pack_ok) {
            spt = 128 / ((rem + 2 * (md->m - 1) + 7) & ~7);   // strips of a multiple of 8 lanes
            if (spt < 2) spt = 0;
        }
        if (rem > 0 && spt == 0) { nfull += 1; rem = 0; }
        const int nbands = div_up(H, R);
        q.tiles_x = nfull;
        q.ntiles = nbands * nfull + (rem > 0 ? div_up(nbands, spt) : 0);
        q.tc_rem = rem;
        q.tc_spt = spt;
        q.tc_rows = R;
    };
    // R: 64 unless a single small image cannot fill the GPU with 64-row tiles; then the R with the
    // fewest (waves of 2 CTAs per SM) x (response rows + ~8 rows of prologue) -- c3 (512^2): R = 8,
    // 278 CTAs instead of 35.  Row slabs keep R = 64 (their bands).
    int bestR = kTcR;
    if (pack_ok && req_rows > 0) {
        bestR = req_rows;
    } else if (pack_ok) {
        double best = 1e30;
        for (int R : {64, 32, 16, 8, 4}) {
            Plan q;
            tiling(R, q);
            const double waves = std::ceil((double)q.ntiles * B / (2.0 * md->nsm));
            const double cost = waves * (R + (md->m - 1) + 8);
            if (cost < best - 1e-9) { best = cost; bestR = R; }
        }
    }
    bool tc = md->tc_np != 0 && pref != FOE_STENCIL_FFMA;
    if (tc && pref == FOE_STENCIL_AUTO) {
        if (!pack_ok) {   // row slabs: the whole scene's 64-row tiles fill two CTAs per SM
            tc = (long long)div_up(W, ow) * div_up(H_grid, kTcR) * B >= 2LL * md->nsm;
        } else {
            Plan q;
            tiling(bestR, q);
            tc = (long long)q.ntiles * B >= (3LL * md->nsm) / 4;
        }
    }
    if (tc) {
        p.kind = FOE_STENCIL_TENSOR;
        tiling(bestR, p);
        p.groups = 1;
    } else {
        p.kind = FOE_STENCIL_FFMA;
        p.tiles_x = div_up(W, kTile);
        p.ntiles = p.tiles_x * div_up(H, kTile);
        // one filter pair per chunk for latency-bound launches (fewer than 8 two-pair work items per
        // SM: single small images; measured on the persistent driver: c2 9.23 -> 8.62 ms, c3 26.76 ->
        // 26.39 ms per solve), two pairs when the launch is throughput-bound (less staging per flop)
        const int npairs = (md->nf + 1) / 2;
        const long long tiles_grid = (long long)p.tiles_x * div_up(H_grid, kTile) * B;
        p.ncp = t_force_ncp > 0 ? t_force_ncp : tiles_grid * div_up(npairs, kNCP) < 8LL * md->nsm ? 1 : kNCP;
        p.nchunks = div_up(npairs, p.ncp);
        p.groups = choose_groups(md, p.tiles_x * div_up(H_grid, kTile), B, req_groups, p.nchunks);
    }
    return p;
}

// K8 launch of tile height R (4 .. 64), with or without row halos (NH), as a programmatic
// dependent launch (the graph trial rounds) or a plain one
template <int M, int NP, int MODE, int RR>
cudaError_t launch_th_r(dim3 grid, cudaStream_t s, const foe::TcArgs& ta, const foe::ThConst& cc, bool pdl) {
    if (pdl) return launch_pdl(foe::k_prior_grad_th<M, NP, RR, MODE>, grid, dim3(256), th_smem<M, NP, RR>(), s, ta, cc);
    foe::k_prior_grad_th<M, NP, RR, MODE><<<grid, 256, th_smem<M, NP, RR>(), s>>>(ta, cc);
    return cudaGetLastError();
}
template <int M, int NP, int MODE>
cudaError_t launch_th(int R, dim3 grid, cudaStream_t s, const foe::TcArgs& ta, const foe::ThConst& cc, bool pdl) {
    switch (R) {
        case 4: return launch_th_r<M, NP, MODE, 4>(grid, s, ta, cc, pdl);
        case 8: return launch_th_r<M, NP, MODE, 8>(grid, s, ta, cc, pdl);
        case 16: return launch_th_r<M, NP, MODE, 16>(grid, s, ta, cc, pdl);
        case 32: return launch_th_r<M, NP, MODE, 32>(grid, s, ta, cc, pdl);
        default: return launch_th_r<M, NP, MODE, 64>(grid, s, ta, cc, pdl);
    }
}
template <int M, int NP>
cudaError_t launch_th_mode(int mode, int R, dim3 grid, cudaStream_t s, const foe::TcArgs& ta, const foe::ThConst& cc,
                           bool pdl) {
    if (mode == 2) return launch_th<M, NP, 2>(R, grid, s, ta, cc, pdl);
    if (mode == 1) return launch_th<M, NP, 1>(R, grid, s, ta, cc, pdl);
    return launch_th<M, NP, 0>(R, grid, s, ta, cc, pdl);
}

// Launch the prior energy+gradient evaluation `a` (tiling fields taken from the plan).
foe_status launch_prior(const foe_model* md, int kind, K1Args a, int B, cudaStream_t s, int ntiles_grid = -1,
                        bool pdl = false) {
    if (kind == FOE_STENCIL_FFMA) {
        k1_dispatch(md->m, false, a, *md->tp, *md->tp2, dim3(a.ntiles * a.groups, B), s);
        CKL("k_prior_grad2");
        return FOE_OK;
    }
    foe::TcArgs ta;
    ta.k = a;
    ta.k.groups = 1;
    ta.bimg = md->th_bimg;
    ta.tiles_x = a.tiles_x;
    count_launch(1);
    const dim3 grid(ntiles_grid >= 0 ? ntiles_grid : a.ntiles - a.tile_off, B);
    if (grid.x == 0) return FOE_OK;
    const int R = a.tc_rows;
    const int mode = a.gedge == nullptr ? 0 : (a.gright == nullptr ? 1 : 2);
    const cudaError_t e = md->tc_np == 48 ? launch_th_mode<7, 48>(mode, R, grid, s, ta, *md->th_const, pdl)
                                          : launch_th_mode<5, 32>(mode, R, grid, s, ta, *md->th_const, pdl);
    CK(e);
    CKL("k_prior_grad_th");
    return FOE_OK;
}

foe_status check_dims(const foe_model* md, int B, int H, int W) {
    if (!md) return fail(FOE_ERR_INVALID_ARGUMENT, "model is NULL");
    if (B < 1) return fail(FOE_ERR_INVALID_ARGUMENT, "B=%d must be >= 1", B);
    if (H < md->m || W < md->m)
        return fail(FOE_ERR_INVALID_ARGUMENT, "image %dx%d smaller than the %dx%d filters (SPEC.md:92)", H, W,
                    md->m, md->m);
    if ((long long)B * H * W > (1LL << 40)) return fail(FOE_ERR_INVALID_ARGUMENT, "B*H*W too large");
    if (B > 65535) return fail(FOE_ERR_INVALID_ARGUMENT, "B=%d exceeds 65535 images per call (one grid row per image)", B);
    return FOE_OK;
}

struct StreamJoin {  // run work on `inner` ordered after `outer`, and `outer` after the work
    cudaStream_t outer, inner;
    cudaEvent_t ev;
};

bool is_device_ptr(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Evaluate K1 at device w[B][HW] (no control block); fills epart[B][ntiles*groups] and
// the gradient planes gparts[groups][B][HW].
foe_status run_k1_plain(const foe_model* md, const double* w, int B, int H, int W, int groups,
                        double* epart, float* gparts, bool hvp, const double* v, const float* gw,
                        cudaStream_t s, int kind = FOE_STENCIL_FFMA, int tiles_x_tc = 0, int ntiles_tc = 0,
                        int tc_rem = 0, int tc_spt = 0, int tc_rows = kTcR, int ncp = kNCP, int nchunks2 = 0,
                        float* sbuf = nullptr, bool s_stored = false) {
    K1Args a{};
    a.w = w;
    a.w_slot_stride = 0;
    a.g = gparts;
    a.g_slot_stride = 0;
    a.g_group_stride = (size_t)B * H * W;
    a.epart = epart;
    a.ctl = nullptr;
    a.which_cur = 1;
    a.H = H;
    a.W = W;
    a.tiles_x = div_up(W, kTile);
    a.ntiles = a.tiles_x * div_up(H, kTile);
    a.groups = groups;
    a.nf = md->nf;
    a.nchunks = div_up(md->nf, Tr<7>::NC);   // (4 filters = 2 pairs per chunk; the v1 HVP stencil too)
    if (!hvp && kind == FOE_STENCIL_FFMA && nchunks2 > 0) {
        a.ncp = ncp;
        a.nchunks = nchunks2;
    }
    a.v = v;
    a.gw = gw;
    a.udom = md->term == FOE_DATA_IDIV;
    if (!hvp) {
        if (kind == FOE_STENCIL_TENSOR) {
            a.tiles_x = tiles_x_tc;
            a.ntiles = ntiles_tc;
            a.groups = 1;
            a.tc_rem = tc_rem;
            a.tc_spt = tc_spt;
            a.tc_rows = tc_rows;
        }
        return launch_prior(md, kind, a, B, s);
    }
    if (md->tc_np) {
        // K8h: the HVP on the tensor cores (whole images, 64-row tiles of 128 - 2C columns, no
        // packing; one CTA per SM)
        foe::TcArgs ta;
        ta.k = a;
        ta.k.groups = 1;
        ta.k.tiles_x = div_up(W, 128 - (md->m - 1));
        ta.k.ntiles = ta.k.tiles_x * div_up(H, kTcR);
        ta.k.tile_off = 0;
        ta.bimg = md->th_bimg;
        ta.tiles_x = ta.k.tiles_x;
        count_launch(1);
        const dim3 grid(ta.k.ntiles, B);
        // sbuf (the Lipschitz estimate): the first HVP stores S_i = rho''(K_i u)/2 of every pixel,
        // the later ones (same w) read it (k_hvp_s: one GEMM fewer, two CTAs per SM)
        ta.k.sbuf = sbuf;
        if (sbuf != nullptr && s_stored) {
            if (md->tc_np == 48)
                foe::k_hvp_s<7, 48, kTcR><<<grid, 256, th_smem<7, 48, kTcR>(), s>>>(ta, *md->th_const);
            else
                foe::k_hvp_s<5, 32, kTcR><<<grid, 256, th_smem<5, 32, kTcR>(), s>>>(ta, *md->th_const);
            CKL("k_hvp_s");
            return FOE_OK;
        }
        if (md->tc_np == 48)
            foe::k_hvp_th<7, 48, kTcR><<<grid, 256, foe::ThHGeom<7, 48, kTcR>::SMEM_BYTES, s>>>(ta, *md->th_const);
        else
            foe::k_hvp_th<5, 32, kTcR><<<grid, 256, foe::ThHGeom<5, 32, kTcR>::SMEM_BYTES, s>>>(ta, *md->th_const);
        CKL("k_hvp_th");
        return FOE_OK;
    }
    dim3 grid(a.ntiles * groups, B);
    k1_dispatch(md->m, hvp, a, *md->tp, *md->tp2, grid, s);
    CKL("k_prior_grad launch");
    return FOE_OK;
}

// grad_w F at device w into g [B][H][W] (one plane: groups = 1), on the stencil the model's AUTO
// plan picks (K8 for the banks it has, so the Lipschitz setup's gradient is a tensor-core one too)
foe_status grad_direct(const foe_model* md, const double* w, int B, int H, int W, float* g, cudaStream_t s) {
    const Plan pl = plan_stencil(md, B, H, W, H, FOE_STENCIL_AUTO, 1);
    double* epart = nullptr;
    CK(cudaMallocFromPoolAsync((void**)&epart, sizeof(double) * B * (size_t)std::max(pl.ntiles * pl.groups, 1),
                               md->pool, s));
    foe_status st = run_k1_plain(md, w, B, H, W, 1, epart, g, false, nullptr, nullptr, s, pl.kind, pl.tiles_x,
                                 pl.ntiles, pl.tc_rem, pl.tc_spt, pl.tc_rows, pl.ncp, pl.nchunks);
    CK(cudaFreeAsync(epart, s));
    return st;
}

}  // namespace

extern "C" {

foe_status foe_energy_grad(const foe_model* md, const double* w, const float* f, int B, int H, int W,
                           const double* lambda_per_image, double* prior_energy, double* data_energy,
                           float* grad, void* stream) {
    foe_status st = check_dims(md, B, H, W);
    if (st != FOE_OK) return st;
    if (!w) return fail(FOE_ERR_INVALID_ARGUMENT, "w is NULL");
    if (data_energy && !f) return fail(FOE_ERR_INVALID_ARGUMENT, "f is NULL but data_energy requested");
    CK(cudaSetDevice(md->dev));
    cudaStream_t s = (cudaStream_t)stream;
    const size_t HW = (size_t)H * W;
    const Plan pl = plan_stencil(md, B, H, W, H, md->stencil, 0);
    const int groups = pl.groups;
    const int ne = pl.ntiles * pl.groups;
    double* epart = nullptr;
    float* gparts = nullptr;
    double* dred = nullptr;
    double* dpart = nullptr;
    double* dlam = nullptr;
    const int nblk = div_up((long long)HW, (long long)kThreads * kPxt2);
    CK(cudaMallocFromPoolAsync((void**)&epart, sizeof(double) * B * ne, md->pool, s));
    const bool direct = (groups == 1 && grad != nullptr);
    if (!direct) CK(cudaMallocFromPoolAsync((void**)&gparts, sizeof(float) * groups * B * HW, md->pool, s));
    CK(cudaMallocFromPoolAsync((void**)&dred, sizeof(double) * B * 2, md->pool, s));
    st = run_k1_plain(md, w, B, H, W, groups, epart, direct ? grad : gparts, false, nullptr, nullptr, s, pl.kind,
                      pl.tiles_x, pl.ntiles, pl.tc_rem, pl.tc_spt, pl.tc_rows, pl.ncp, pl.nchunks);
    if (st != FOE_OK) return st;
    if (grad && !direct) {
        const size_t n = (size_t)B * HW;
        foe::k_sum_groups<<<div_up((long long)n, 256), 256, 0, s>>>(gparts, n, groups, grad, n);
        count_launch(1);
        CKL("k_sum_groups");
    }
    foe::k_reduce_rows<<<B, kThreads, 0, s>>>(epart, ne, 1, 1, dred);
    count_launch(1);
    CKL("k_reduce_rows");
    if (data_energy) {
        std::vector<double> lam(2 * (size_t)B);
        for (int b = 0; b < B; ++b) {
            lam[2 * b] = lambda_per_image ? lambda_per_image[2 * b] : md->lam[0];
            lam[2 * b + 1] = md->term != FOE_DATA_COMBINED ? 0.0 : (lambda_per_image ? lambda_per_image[2 * b + 1] : md->lam[1]);
        }
        CK(cudaMallocFromPoolAsync((void**)&dlam, sizeof(double) * 2 * B, md->pool, s));
        CK(cudaMallocFromPoolAsync((void**)&dpart, sizeof(double) * B * nblk, md->pool, s));
        CK(cudaMemcpyAsync(dlam, lam.data(), sizeof(double) * 2 * B, cudaMemcpyHostToDevice, s));
        foe::k_data_energy<<<dim3(nblk, B), kThreads, 0, s>>>(w, f, dlam, dpart, nblk, HW, kPxt2,
                                                               md->term == FOE_DATA_IDIV);
        count_launch(1);
        CKL("k_data_energy");
        foe::k_reduce_rows<<<B, kThreads, 0, s>>>(dpart, nblk, 1, 1, dred + B);
        count_launch(1);
        CKL("k_reduce_rows");
    }
    std::vector<double> hred(2 * (size_t)B);
    if (prior_energy || data_energy) {
        CK(cudaMemcpyAsync(hred.data(), dred, sizeof(double) * 2 * B, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaFreeAsync(epart, s));
    if (gparts) CK(cudaFreeAsync(gparts, s));
    if (dpart) CK(cudaFreeAsync(dpart, s));
    if (dlam) CK(cudaFreeAsync(dlam, s));
    CK(cudaFreeAsync(dred, s));
    if (prior_energy || data_energy) {
        CK(cudaStreamSynchronize(s));
        for (int b = 0; b < B; ++b) {
            if (prior_energy) prior_energy[b] = hred[b];
            if (data_energy) data_energy[b] = hred[B + b];
        }
    }
    return FOE_OK;
}

foe_status foe_hvp(const foe_model* md, const double* w, const double* v, int B, int H, int W, float* hv,
                   void* stream) {
    foe_status st = check_dims(md, B, H, W);
    if (st != FOE_OK) return st;
    if (!w || !v || !hv) return fail(FOE_ERR_INVALID_ARGUMENT, "w, v and hv must be non-NULL");
    CK(cudaSetDevice(md->dev));
    cudaStream_t s = (cudaStream_t)stream;
    const size_t n = (size_t)B * H * W;
    const int tiles = div_up(W, kTile) * div_up(H, kTile);
    double* epart = nullptr;
    float* gw = nullptr;
    CK(cudaMallocFromPoolAsync((void**)&epart, sizeof(double) * B * tiles, md->pool, s));
    CK(cudaMallocFromPoolAsync((void**)&gw, sizeof(float) * n, md->pool, s));
    st = grad_direct(md, w, B, H, W, gw, s);
    if (st == FOE_OK) st = run_k1_plain(md, w, B, H, W, 1, epart, hv, true, v, gw, s);
    CK(cudaFreeAsync(epart, s));
    CK(cudaFreeAsync(gw, s));
    return st;
}

foe_status foe_estimate_lipschitz(const foe_model* md, const float* f, int B, int H, int W, const double* v0,
                                  int power_iters, double* rho_out, double* L_out, void* stream) {
    foe_status st = check_dims(md, B, H, W);
    if (st != FOE_OK) return st;
    if (!f || !v0 || !L_out) return fail(FOE_ERR_INVALID_ARGUMENT, "f, v0 and L_out must be non-NULL");
    if (power_iters < 1) return fail(FOE_ERR_INVALID_ARGUMENT, "power_iters=%d must be >= 1", power_iters);
    CK(cudaSetDevice(md->dev));
    cudaStream_t s = (cudaStream_t)stream;
    const size_t HW = (size_t)H * W, n = (size_t)B * HW;
    const int tiles = div_up(W, kTile) * div_up(H, kTile);
    const int nblk = div_up((long long)HW, (long long)kThreads * kPxt2);
    double *w0 = nullptr, *v = nullptr, *epart = nullptr, *part = nullptr, *sums = nullptr;
    float *gw = nullptr, *h = nullptr;
    CK(cudaMallocFromPoolAsync((void**)&w0, sizeof(double) * n, md->pool, s));
    CK(cudaMallocFromPoolAsync((void**)&v, sizeof(double) * n, md->pool, s));
    CK(cudaMallocFromPoolAsync((void**)&gw, sizeof(float) * n, md->pool, s));
    CK(cudaMallocFromPoolAsync((void**)&h, sizeof(float) * n, md->pool, s));
    CK(cudaMallocFromPoolAsync((void**)&epart, sizeof(double) * B * tiles, md->pool, s));
    CK(cudaMallocFromPoolAsync((void**)&part, sizeof(double) * B * nblk * 3, md->pool, s));
    CK(cudaMallocFromPoolAsync((void**)&sums, sizeof(double) * B * 3, md->pool, s));
    const int eb = div_up((long long)n, 256);
    foe::k_log_ftilde<<<eb, 256, 0, s>>>(f, w0, n, md->term == FOE_DATA_IDIV);
    count_launch(1);
    CKL("k_log_ftilde");
    // v <- v0 / ||v0||
    foe::k_dot3<<<dim3(nblk, B), kThreads, 0, s>>>(v0, nullptr, part, nblk, HW, kPxt2);
    count_launch(1);
    foe::k_reduce_rows<<<B, kThreads, 0, s>>>(part, nblk, 3, 3, sums);
    count_launch(1);
    const dim3 nb_grid((unsigned)div_up((long long)HW, 1024), B);   // ~4 pixels per thread
    foe::k_normalize<double><<<nb_grid, 256, 0, s>>>(v0, v, sums, 3, 2, HW, B);
    count_launch(1);
    CKL("power-iteration init");
    st = grad_direct(md, w0, B, H, W, gw, s);
    // S_i = rho''(K_i u)/2 at w0 for the tensor-core HVPs after the first (k_hvp_s); without the
    // memory for it every HVP recomputes K u
    float* sbuf = nullptr;
    std::unique_lock<std::mutex> slk(md->s_mu, std::try_to_lock);
    if (md->tc_np && FOE_HVP_STORE_S && slk.owns_lock()) {
        const size_t need = (size_t)md->tc_np * n;
        if (md->s_n < need) {
            if (md->s_buf) {
                CK(cudaStreamSynchronize(s));   // (an earlier estimate's kernels may still read it)
                cudaFree(md->s_buf);
                md->s_buf = nullptr;
                md->s_n = 0;
            }
            if (cudaMalloc((void**)&md->s_buf, sizeof(float) * need) == cudaSuccess) md->s_n = need;
            else { cudaGetLastError(); md->s_buf = nullptr; }
        }
        sbuf = md->s_buf;
    }
    for (int it = 0; it < power_iters && st == FOE_OK; ++it) {
        st = run_k1_plain(md, w0, B, H, W, 1, epart, h, true, v, gw, s, FOE_STENCIL_FFMA, 0, 0, 0, 0, kTcR, kNCP, 0,
                          sbuf, it > 0);   // h = Hess v
        // <h,h> every step, <v,h> (the Rayleigh quotient) at the last one
        foe::k_dot3<<<dim3(nblk, B), kThreads, 0, s>>>(it + 1 < power_iters ? nullptr : v, h, part, nblk, HW, kPxt2);
        count_launch(1);
        foe::k_reduce_rows<<<B, kThreads, 0, s>>>(part, nblk, 3, 3, sums);  // <v,h>, <h,h>
        foe::k_normalize<float><<<nb_grid, 256, 0, s>>>(h, v, sums, 3, 1, HW, B);
        count_launch(1);
        CKL("power iteration");
    }
    std::vector<double> hs(3 * (size_t)B);
    CK(cudaMemcpyAsync(hs.data(), sums, sizeof(double) * 3 * B, cudaMemcpyDeviceToHost, s));
    CK(cudaFreeAsync(w0, s)); CK(cudaFreeAsync(v, s)); CK(cudaFreeAsync(gw, s)); CK(cudaFreeAsync(h, s));
    CK(cudaFreeAsync(epart, s)); CK(cudaFreeAsync(part, s)); CK(cudaFreeAsync(sums, s));
    CK(cudaStreamSynchronize(s));
    if (st != FOE_OK) return st;
    for (int b = 0; b < B; ++b) {
        const double rho = std::fabs(hs[3 * b]);
        if (!(rho > 0) || !std::isfinite(rho))
            return fail(FOE_ERR_NONFINITE, "Lipschitz estimate of image %d is %g", b, rho);
        if (rho_out) rho_out[b] = rho;
        L_out[b] = std::ldexp(1.0, (int)std::ceil(std::log2(rho)));
    }
    return FOE_OK;
}

void ipiano_config_default(ipiano_config* c) {
    if (!c) return;
    c->beta = 0.4;
    c->step_safety = 0.95;
    c->backtrack_factor = 2.0;
    c->shrink = 1.0;
    c->max_iters = 300;
    c->max_backtracks = 60;
    c->newton_max_iters = 30;
    c->newton_tol = 1e-12;
    c->rel_change_tol = 0.0;
    c->w_guard = 40.0;
    c->record_trace = 1;
    c->filter_groups = 0;
    c->stencil = FOE_STENCIL_AUTO;
    c->solver = FOE_SOLVER_AUTO;
    c->tile_rows = 0;
}

}  // extern "C"

// --------------------------------------------------------------------------- solver

namespace {

foe_status join_begin(ipiano_state* st, cudaStream_t user) {
    CK(cudaEventRecord(st->sync_ev, user));
    CK(cudaStreamWaitEvent(st->s, st->sync_ev, 0));
    return FOE_OK;
}
foe_status join_end(ipiano_state* st, cudaStream_t user) {
    CK(cudaEventRecord(st->sync_ev, st->s));
    CK(cudaStreamWaitEvent(user, st->sync_ev, 0));
    return FOE_OK;
}

K1Args state_k1_args(const ipiano_state* st, int which_cur) {
    K1Args a{};
    a.w = st->w;
    a.w_slot_stride = (size_t)st->B * st->HW;
    a.g = st->g;
    a.g_group_stride = (size_t)st->B * st->HW;
    a.g_slot_stride = a.g_group_stride * st->groups;
    a.epart = st->epart;
    a.ctl = st->ctl;
    a.which_cur = which_cur;
    a.H = st->H;
    a.W = st->W;
    a.tiles_x = st->tiles_x;
    a.ntiles = st->ntiles;
    a.groups = st->groups;
    a.nf = st->model->nf;
    a.nchunks = st->nchunks;
    a.ncp = st->ncp;
    a.udom = st->model->term == FOE_DATA_IDIV;
    a.tc_rem = st->tc_rem;
    a.tc_spt = st->tc_spt;
    a.tc_rows = st->tc_rows;
    a.gedge = st->gedge;
    a.gedge_slot_stride = st->gedge ? (size_t)st->B * (st->H / st->tc_rows) * (st->model->m - 1) * st->W : 0;
    a.tcnt = st->tcnt;
    a.gright = st->gright;
    a.gcorner = st->gcorner;
    a.gright_slot_stride = st->gright ? (size_t)st->B * st->tiles_x * st->H * (st->model->m - 1) : 0;
    a.gcorner_slot_stride =
        st->gcorner ? (size_t)st->B * (st->H / st->tc_rows) * st->tiles_x * (st->model->m - 1) * (st->model->m - 1) : 0;
    return a;
}

cudaEvent_t pool_event(ipiano_state* st) {
    if (!st->ev_pool.empty()) {
        cudaEvent_t e = st->ev_pool.back();
        st->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

foe::K2Args state_k2_args(const ipiano_state* st) {
    foe::K2Args a2{};
    a2.w = st->w;
    a2.w_slot_stride = (size_t)st->B * st->HW;
    a2.g = st->g;
    a2.g_group_stride = (size_t)st->B * st->HW;
    a2.g_slot_stride = a2.g_group_stride * st->groups;
    a2.ft = st->ft;
    a2.ppart = st->ppart;
    a2.ctl = st->ctl;
    a2.sp = st->sp;
    a2.groups = st->groups;
    a2.nblk = st->nblk2;
    a2.HW = st->HW;
    a2.idiv = st->model->term == FOE_DATA_IDIV;
    a2.pairs = FOE_K2_PAIRS && st->HW % 4 == 0;
    return a2;
}

foe::K3Args state_k3_args(const ipiano_state* st) {
    foe::K3Args a3{};
    a3.ctl = st->ctl;
    a3.epart = st->epart;
    a3.ppart = st->ppart;
    a3.trace = st->trace;
    a3.ne = st->ntiles * st->groups;
    a3.nblk = st->nblk3;
    a3.estride = 1;
    a3.sp = st->sp;
    return a3;
}

// One trial round for every active image: K2 -> K1 (candidate) -> K3, as programmatic dependent
// launches (each kernel's launch and independent prologue overlap its predecessor's drain).
foe_status launch_round(ipiano_state* st, cudaStream_t s, bool timed) {
    cudaEvent_t k0 = nullptr;
    if (timed) {
        k0 = pool_event(st);
        CK(cudaEventRecord(k0, s));
    }
    {
        const foe::K2Args a2 = state_k2_args(st);
        const dim3 g2(st->nblk2, st->B), tb(kThreads);
        if (st->pxt2 == 1) CK(launch_pdl(foe::k_inertial_prox<1>, g2, tb, 0, s, a2));
        else if (st->pxt2 == 4) CK(launch_pdl(foe::k_inertial_prox<4>, g2, tb, 0, s, a2));
        else if (st->pxt2 == 16) CK(launch_pdl(foe::k_inertial_prox<16>, g2, tb, 0, s, a2));
        else if (st->pxt2 == 32) CK(launch_pdl(foe::k_inertial_prox<32>, g2, tb, 0, s, a2));
        else CK(launch_pdl(foe::k_inertial_prox<kPxt2>, g2, tb, 0, s, a2));
        count_launch(1);
        CKL("k_inertial_prox");
    }
    const K1Args a1 = state_k1_args(st, 0);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timed) {
        e0 = pool_event(st);
        e1 = pool_event(st);
        CK(cudaEventRecord(e0, s));
        st->ev_live_k2.emplace_back(k0, e0);
        st->k2_launches += 1;
    }
    foe_status rl = launch_prior(st->model, st->kind, a1, st->B, s, -1, !timed);
    if (rl != FOE_OK) return rl;
    if (timed) {
        CK(cudaEventRecord(e1, s));
        st->ev_live.emplace_back(e0, e1);
        st->k1_launches += 1;
    }
    const foe::K3Args a3 = state_k3_args(st);
    CK(launch_pdl(foe::k_decide, dim3(st->B), dim3(kThreads), 0, s, a3));
    count_launch(1);
    CKL("k_decide");
    st->total_launches += 3;
    return FOE_OK;
}

// ---- persistent driver (foe_persist.cuh) ----
template <int M, int PXT, int NCP>
const void* persist_kernel() { return (const void*)foe::k_ipiano_persistent<M, NCP, kSF2, PXT>; }
const void* persist_kernel_for(int m, int pxt, int ncp) {
    if (m == 7) return pxt == 1 ? (ncp == 1 ? persist_kernel<7, 1, 1>() : persist_kernel<7, 1, 2>())
                                : (ncp == 1 ? persist_kernel<7, 4, 1>() : persist_kernel<7, 4, 2>());
    if (m == 5) return pxt == 1 ? (ncp == 1 ? persist_kernel<5, 1, 1>() : persist_kernel<5, 1, 2>())
                                : (ncp == 1 ? persist_kernel<5, 4, 1>() : persist_kernel<5, 4, 2>());
    return pxt == 1 ? (ncp == 1 ? persist_kernel<3, 1, 1>() : persist_kernel<3, 1, 2>())
                    : (ncp == 1 ? persist_kernel<3, 4, 1>() : persist_kernel<3, 4, 2>());
}
int smem2_for(int m, int ncp) {
    if (ncp == 1) return m == 7 ? smem2_bytes<7, 1>() : m == 5 ? smem2_bytes<5, 1>() : smem2_bytes<3, 1>();
    return m == 7 ? smem2_bytes<7>() : m == 5 ? smem2_bytes<5>() : smem2_bytes<3>();
}

// co-resident CTAs of the persistent kernel on this device (0 if cooperative launch is unsupported)
int persist_capacity(const foe_model* md, int pxt, int ncp) {
    int coop = 0;
    if (cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, md->dev) != cudaSuccess || !coop) {
        cudaGetLastError();
        return 0;
    }
    const void* k = persist_kernel_for(md->m, pxt, ncp);
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2_for(md->m, ncp)) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreads, smem2_for(md->m, ncp)) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return per_sm * md->nsm;
}

// up to max_rounds trial rounds (fewer once no image is active) in one cooperative launch
foe_status launch_persistent(ipiano_state* st, long long max_rounds) {
    foe::PersistArgs pa{};
    pa.a1 = state_k1_args(st, 0);
    pa.a2 = state_k2_args(st);
    pa.a3 = state_k3_args(st);
    pa.ctl = st->ctl;
    pa.bar = st->bar;
    pa.ppart_stride = (size_t)st->B * st->nblk2 * foe::kNumPart;
    pa.B = st->B;
    pa.max_rounds = (int)std::min<long long>(max_rounds, 1LL << 30);
    pa.k1_items = st->ntiles * st->groups;
    pa.k2_items = st->nblk2;
    pa.rounds_out = nullptr;
    pa.phase_ns = st->phase_ns;
    CK(cudaMemsetAsync(st->bar, 0, sizeof(unsigned int), st->s));
    void* args[] = {(void*)&pa, (void*)st->model->tp2};
    CK(cudaLaunchCooperativeKernel(persist_kernel_for(st->model->m, st->pxt2, st->ncp), dim3(st->pgrid), dim3(kThreads),
                                   args, (size_t)smem2_for(st->model->m, st->ncp), st->s));
    count_launch(1);
    st->total_launches += 1;
    return FOE_OK;
}

constexpr int kGraphRounds = 10;

foe_status ensure_graph(ipiano_state* st) {
    if (st->graph) return FOE_OK;
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(st->s, cudaStreamCaptureModeThreadLocal));
    foe_status r = FOE_OK;
    const long long tl = st->total_launches;
    t_capturing = true;
    for (int i = 0; i < kGraphRounds && r == FOE_OK; ++i) r = launch_round(st, st->s, false);
    t_capturing = false;
    st->total_launches = tl;
    cudaError_t e = cudaStreamEndCapture(st->s, &g);
    if (r != FOE_OK) { if (g) cudaGraphDestroy(g); return r; }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture", __LINE__);
    e = cudaGraphInstantiate(&st->graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate", __LINE__);
    st->graph_rounds = kGraphRounds;
    return FOE_OK;
}

foe_status launch_rounds(ipiano_state* st, long long rounds) {
    if (st->solver == FOE_SOLVER_PERSISTENT && !st->profile) return launch_persistent(st, rounds);
    if (st->profile) {
        for (int i = 0; i < rounds; ++i) {
            foe_status r = launch_round(st, st->s, true);
            if (r != FOE_OK) return r;
        }
        return FOE_OK;
    }
    foe_status r = ensure_graph(st);
    if (r != FOE_OK) return r;
    const int reps = div_up(rounds, st->graph_rounds);
    for (int i = 0; i < reps; ++i) {
        CK(cudaGraphLaunch(st->graph, st->s));
        const long long per = 3;
        st->total_launches += per * st->graph_rounds;
        count_launch(per * st->graph_rounds);
    }
    return FOE_OK;
}

foe_status sync_ctl(ipiano_state* st) {
    CK(cudaMemcpyAsync(st->hctl, st->ctl, sizeof(ImgCtl) * st->B, cudaMemcpyDeviceToHost, st->s));
    CK(cudaStreamSynchronize(st->s));
    for (auto& pr : st->ev_live) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) st->k1_ms += ms;
        st->ev_pool.push_back(pr.first);
        st->ev_pool.push_back(pr.second);
    }
    st->ev_live.clear();
    for (auto& pr : st->ev_live_k2) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) st->k2_ms += ms;
        st->ev_pool.push_back(pr.first);   // (pr.second is also an ev_live start event)
    }
    st->ev_live_k2.clear();
    return FOE_OK;
}

foe_status first_image_error(const ipiano_state* st) {
    for (int b = 0; b < st->B; ++b) {
        const ImgCtl& c = st->hctl[b];
        if (c.status != 0) {
            const char* what = c.status == foe::ST_PROX        ? "prox Newton cap exceeded (SPEC.md:198)"
                               : c.status == foe::ST_BACKTRACK ? "more than max_backtracks doublings (SPEC.md:288)"
                               : c.status == foe::ST_DOMAIN    ? "accepted |w| above w_guard (R-11)"
                                                               : "non-finite accepted energy or iterate (SPEC.md:288)";
            return fail((foe_status)c.status, "image %d, iteration %d: %s", b, c.n + 1, what);
        }
    }
    return FOE_OK;
}


// a1: f~ = max(f,1), w^0 = log f~, w^{-1} = w^0, F(w^0) and grad F(w^0), trace row 0.
foe_status state_init(ipiano_state* st, const float* f, const double* lipschitz_init, cudaStream_t user) {
    const int B = st->B;
    const size_t n = (size_t)B * st->HW;
    for (int b = 0; b < B; ++b) {
        ImgCtl& c = st->hctl[b];
        std::memset(&c, 0, sizeof(c));
        c.L = lipschitz_init[b];
        c.lam1 = st->lam[2 * b];
        c.lam2 = st->lam[2 * b + 1];
        c.cur = 0; c.prev = 1; c.cand = 2;
        c.gcur = 0; c.gcand = 1;
        c.active = 1;  // for the initial evaluation
        c.target = 0;
    }
    foe_status r = join_begin(st, user);
    if (r != FOE_OK) return r;
    CK(cudaMemcpyAsync(st->ctl, st->hctl, sizeof(ImgCtl) * B, cudaMemcpyHostToDevice, st->s));
    if (st->cfg.record_trace)
        CK(cudaMemsetAsync(st->trace, 0, sizeof(double) * B * (st->cfg.max_iters + 1) * 8, st->s));
    foe::k_init<<<dim3(st->nblk2, B), kThreads, 0, st->s>>>(f, st->ft, st->w, n, st->ppart, st->nblk2, st->ctl,
                                                             st->HW, st->pxt2, nullptr, nullptr, 0,
                                                             st->model->term == FOE_DATA_IDIV);
    count_launch(1);
    CKL("k_init");
    const K1Args a1 = state_k1_args(st, 1);
    foe_status rl = launch_prior(st->model, st->kind, a1, B, st->s);
    if (rl != FOE_OK) return rl;
    foe::k_init_finalize<<<B, kThreads, 0, st->s>>>(st->ctl, st->epart, st->ntiles * st->groups, 1, st->ppart,
                                                    st->nblk2, st->trace, st->cfg.max_iters, st->cfg.record_trace);
    count_launch(1);
    CKL("k_init_finalize");
    foe::k_set_target<<<div_up(B, 128), 128, 0, st->s>>>(st->ctl, B, 0);
    count_launch(1);
    CKL("k_set_target");
    return join_end(st, user);
}

}  // namespace

extern "C" {

int ipiano_state_stencil(const ipiano_state* st) { return st ? st->kind : -1; }
foe_status ipiano_state_tiling(const ipiano_state* st, int* tile_rows, int* tile_cols, int* halo_mode) {
    if (!st || !tile_rows || !tile_cols || !halo_mode) return fail(FOE_ERR_INVALID_ARGUMENT, "NULL state or output");
    const bool tc = st->kind == FOE_STENCIL_TENSOR;
    *tile_rows = tc ? st->tc_rows : 0;
    *tile_cols = tc ? (st->tc_mode == 2 ? 128 : 128 - (st->model->m - 1)) : 0;
    *halo_mode = tc ? st->tc_mode : 0;
    return FOE_OK;
}
int ipiano_state_solver(const ipiano_state* st) { return st ? st->solver : -1; }

void ipiano_state_destroy(ipiano_state* st) {
    if (!st) return;
    cudaSetDevice(st->model->dev);
    if (st->s) cudaStreamSynchronize(st->s);
    if (st->graph) cudaGraphExecDestroy(st->graph);
    cudaFree(st->w); cudaFree(st->g); cudaFree(st->gedge); cudaFree(st->tcnt); cudaFree(st->gright); cudaFree(st->gcorner); cudaFree(st->ft); cudaFree(st->epart); cudaFree(st->ppart);
    if (st->phase_ns) {   // FOE_PERSIST_PHASES diagnostics: mean phase durations of the last launch
        std::vector<unsigned long long> h(4 * foe::kPhaseRounds, 0);
        cudaMemcpy(h.data(), st->phase_ns, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost);
        double t[3] = {0, 0, 0};
        int n = 0;
        for (int r = 1; r < foe::kPhaseRounds && h[4 * r + 3] > h[4 * r]; ++r, ++n)
            for (int k = 0; k < 3; ++k) t[k] += (double)(h[4 * r + k + 1] - h[4 * r + k]);
        if (n > 0)
            std::fprintf(stderr, "[foe persistent] grid %d, %d rounds: K2+barrier %.2f us, K1+barrier %.2f us, K3 %.2f us\n",
                         st->pgrid, n, 1e-3 * t[0] / n, 1e-3 * t[1] / n, 1e-3 * t[2] / n);
        cudaFree(st->phase_ns);
    }
    cudaFree(st->trace); cudaFree(st->ctl); cudaFree(st->bar);
    if (st->hctl) cudaFreeHost(st->hctl);
    for (auto e : st->ev_pool) cudaEventDestroy(e);
    for (auto& pr : st->ev_live) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
    for (auto& pr : st->ev_live_k2) cudaEventDestroy(pr.first);
    if (st->sync_ev) cudaEventDestroy(st->sync_ev);
    if (st->s) cudaStreamDestroy(st->s);
    delete st;
    cudaGetLastError();   // (as ipiano_slabs_destroy)
}

foe_status ipiano_state_create(const foe_model* md, const float* f, int B, int H, int W,
                               const double* lambda_per_image, const double* lipschitz_init,
                               const ipiano_config* cfg_in, void* stream, ipiano_state** out) {
    if (!out) return fail(FOE_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    foe_status rs = check_dims(md, B, H, W);
    if (rs != FOE_OK) return rs;
    if (!f) return fail(FOE_ERR_INVALID_ARGUMENT, "f is NULL");
    if (!lipschitz_init) return fail(FOE_ERR_INVALID_ARGUMENT, "lipschitz_init is NULL");
    ipiano_config cfg;
    if (cfg_in) cfg = *cfg_in; else ipiano_config_default(&cfg);
    if (!(cfg.beta >= 0.0 && cfg.beta < 1.0)) return fail(FOE_ERR_INVALID_ARGUMENT, "beta=%g outside [0,1)", cfg.beta);
    if (cfg.max_iters < 1) return fail(FOE_ERR_INVALID_ARGUMENT, "max_iters=%d must be >= 1", cfg.max_iters);
    if (!(cfg.step_safety > 0.0 && cfg.step_safety <= 1.0))
        return fail(FOE_ERR_INVALID_ARGUMENT, "step_safety=%g outside (0,1]", cfg.step_safety);
    if (!(cfg.backtrack_factor > 1.0)) return fail(FOE_ERR_INVALID_ARGUMENT, "backtrack_factor=%g must be > 1", cfg.backtrack_factor);
    if (!(cfg.shrink > 0.0 && cfg.shrink <= 1.0)) return fail(FOE_ERR_INVALID_ARGUMENT, "shrink=%g outside (0,1]", cfg.shrink);
    if (cfg.max_backtracks < 0 || cfg.newton_max_iters < 1 || !(cfg.newton_tol > 0.0) || !(cfg.w_guard > 0.0) ||
        !(cfg.rel_change_tol >= 0.0))
        return fail(FOE_ERR_INVALID_ARGUMENT, "invalid solver limits (max_backtracks, newton_max_iters, newton_tol, w_guard, rel_change_tol)");
    for (int b = 0; b < B; ++b) {
        if (!(lipschitz_init[b] > 0.0) || !std::isfinite(lipschitz_init[b]))
            return fail(FOE_ERR_INVALID_ARGUMENT, "lipschitz_init[%d]=%g must be > 0", b, lipschitz_init[b]);
        if (lambda_per_image) {
            const double l1 = lambda_per_image[2 * b], l2 = lambda_per_image[2 * b + 1];
            if (!(l1 >= 0) || !(l2 >= 0) || !std::isfinite(l1) || !std::isfinite(l2) || (l1 == 0 && l2 == 0))
                return fail(FOE_ERR_INVALID_ARGUMENT, "lambda of image %d = (%g,%g) invalid", b, l1, l2);
        }
    }
    CK(cudaSetDevice(md->dev));
    ipiano_state* st = new (std::nothrow) ipiano_state();
    if (!st) return fail(FOE_ERR_OUT_OF_MEMORY, "host allocation");
    st->model = md;
    st->B = B; st->H = H; st->W = W;
    st->HW = (size_t)H * W;
    st->cfg = cfg;
    st->sp.beta = cfg.beta;
    st->sp.safety = cfg.step_safety;
    st->sp.eta = cfg.backtrack_factor;
    st->sp.shrink = cfg.shrink;
    st->sp.newton_tol = cfg.newton_tol;
    st->sp.rel_tol = cfg.rel_change_tol;
    st->sp.w_guard = cfg.w_guard;
    st->sp.max_backtracks = cfg.max_backtracks;
    st->sp.newton_cap = cfg.newton_max_iters;
    st->sp.record_trace = cfg.record_trace;
    st->sp.max_iters = cfg.max_iters;
    if (cfg.stencil < FOE_STENCIL_AUTO || cfg.stencil > FOE_STENCIL_TENSOR) {
        delete st;
        return fail(FOE_ERR_INVALID_ARGUMENT, "unknown stencil %d", cfg.stencil);
    }
    if (cfg.stencil == FOE_STENCIL_TENSOR && !md->tc_np) {
        delete st;
        return fail(FOE_ERR_UNSUPPORTED, "no tensor-core stencil for %d filters of %dx%d", md->nf, md->m, md->m);
    }
    if (cfg.solver < FOE_SOLVER_AUTO || cfg.solver > FOE_SOLVER_PERSISTENT) {
        delete st;
        return fail(FOE_ERR_INVALID_ARGUMENT, "unknown solver %d", cfg.solver);
    }
    if (cfg.solver == FOE_SOLVER_PERSISTENT && cfg.stencil == FOE_STENCIL_TENSOR) {
        delete st;
        return fail(FOE_ERR_UNSUPPORTED, "the persistent solver runs the FFMA stencil only");
    }
    if (cfg.tile_rows != 0 && cfg.tile_rows != 4 && cfg.tile_rows != 8 && cfg.tile_rows != 16 && cfg.tile_rows != 32 &&
        cfg.tile_rows != 64) {
        delete st;
        return fail(FOE_ERR_INVALID_ARGUMENT, "tile_rows %d is not 0, 4, 8, 16, 32 or 64", cfg.tile_rows);
    }
    // trial-loop driver (f4): persistent for problems that cannot fill the GPU
    const long long npx = (long long)B * H * W;
    const bool want_persist = cfg.solver == FOE_SOLVER_PERSISTENT ||
                              (cfg.solver == FOE_SOLVER_AUTO && cfg.stencil != FOE_STENCIL_TENSOR &&
                               (npx < (1LL << 16) || (md->tc_np == 0 && npx <= (1LL << 18))));
    const int pref = want_persist ? FOE_STENCIL_FFMA : cfg.stencil;
    const Plan pl = plan_stencil(md, B, H, W, H, pref, cfg.filter_groups, !t_slab_member, cfg.tile_rows, true);
    st->kind = pl.kind;
    st->tiles_x = pl.tiles_x;
    st->tc_rem = pl.tc_rem;
    st->tc_spt = pl.tc_spt;
    st->tc_rows = pl.tc_rows;
    st->tc_mode = pl.kind == FOE_STENCIL_TENSOR ? pl.tc_mode : 0;
    st->ntiles = pl.ntiles;
    st->ncp = pl.kind == FOE_STENCIL_FFMA ? pl.ncp : kNCP;
    st->nchunks = pl.kind == FOE_STENCIL_FFMA ? pl.nchunks : div_up(md->nf, Tr<7>::NC);
    st->groups = pl.groups;
    st->pxt2 = kPxt2;
    // 16 pixels per thread halve the per-pixel share of K2's block reduction (c4: 223 -> 213 us)
    // when the launch still has >= 4 blocks per SM; slab members keep kPxt2 (whole K2 blocks per
    // 64-row band for W % 32 == 0)
#ifndef FOE_K2_PXT_LARGE
#define FOE_K2_PXT_LARGE 16
#endif
    if (!t_slab_member && (long long)B * H * W >= 4LL * md->nsm * kThreads * 16) st->pxt2 = 16;
    if (!t_slab_member && (long long)B * H * W >= 4LL * md->nsm * kThreads * FOE_K2_PXT_LARGE) st->pxt2 = FOE_K2_PXT_LARGE;
#ifndef FOE_K2_PXT_SMALL
#define FOE_K2_PXT_SMALL 4
#endif
    // a launch of fewer than ~4 blocks per SM at 8 px/thread (one 512^2 image: 128 blocks) is
    // fp64-latency bound: more, smaller blocks
    if (!t_slab_member && (long long)B * H * W < 4LL * md->nsm * kThreads * kPxt2) st->pxt2 = FOE_K2_PXT_SMALL;
#ifndef FOE_K2_PXT_TINY
#define FOE_K2_PXT_TINY 1
#endif
    // below one block per SM at 4 px/thread (c2: 256^2 = 64 blocks): one pixel per thread
    if (!t_slab_member && (long long)B * H * W < (long long)md->nsm * kThreads * FOE_K2_PXT_SMALL) st->pxt2 = FOE_K2_PXT_TINY;
    if (t_slab_member && t_force_pxt > 0) st->pxt2 = t_force_pxt;
    if (want_persist && pl.kind == FOE_STENCIL_FFMA) {
        // K2 items: one pixel per thread while the grid can hold them all, else four
        const int pxt = npx <= 2LL * md->nsm * kThreads ? 1 : 4;
        const int cap = persist_capacity(md, pxt, pl.ncp);
        if (cap > 0) {
            const long long items = std::max((long long)pl.ntiles * pl.groups * B,
                                             (long long)div_up((long long)st->HW, (long long)kThreads * pxt) * B);
            st->solver = FOE_SOLVER_PERSISTENT;
            st->pxt2 = pxt;
            st->pgrid = (int)std::max(1LL, std::min<long long>(cap, items));
        } else if (cfg.solver == FOE_SOLVER_PERSISTENT) {
            delete st;
            return fail(FOE_ERR_UNSUPPORTED, "cooperative launch of the persistent solver is not available");
        }
    }
    st->nblk2 = div_up((long long)st->HW, (long long)kThreads * st->pxt2);
    st->nblk3 = st->nblk2;
    auto cleanup = [&](foe_status s) { ipiano_state_destroy(st); return s; };
#define CKS(call)                                                                    \
    do {                                                                             \
        cudaError_t e_ = (call);                                                     \
        if (e_ != cudaSuccess) return cleanup(cuda_fail(e_, #call, __LINE__));       \
    } while (0)
    CKS(cudaStreamCreateWithFlags(&st->s, cudaStreamNonBlocking));
    CKS(cudaEventCreateWithFlags(&st->sync_ev, cudaEventDisableTiming));
    const size_t n = (size_t)B * st->HW;
    CKS(cudaMalloc((void**)&st->w, sizeof(double) * 3 * n));
    CKS(cudaMalloc((void**)&st->g, sizeof(float) * 2 * st->groups * n));
    // K8 without row halos (foe_th.cuh): the batch path's tensor-core stencil when the bands tile H
    // and are at least 2C rows tall (a row near a band edge then takes contributions from two bands)
    if (st->tc_mode >= 1) {   // (plan_stencil: bands of R that tile H, R >= 2C; mode 2: W % 128 == 0)
        const size_t nb = H / st->tc_rows, c2 = md->m - 1;
        CKS(cudaMalloc((void**)&st->gedge, sizeof(float) * 2 * (size_t)B * nb * c2 * W));
        if (st->tc_mode == 2) {
            CKS(cudaMalloc((void**)&st->gright, sizeof(float) * 2 * (size_t)B * st->tiles_x * H * c2));
            CKS(cudaMalloc((void**)&st->gcorner, sizeof(float) * 2 * (size_t)B * nb * st->tiles_x * c2 * c2));
        }
        const size_t nc = 3 * (size_t)B * nb * (st->tiles_x + 1);
        CKS(cudaMalloc((void**)&st->tcnt, sizeof(unsigned int) * nc));
        CKS(cudaMemset(st->tcnt, 0, sizeof(unsigned int) * nc));
    }
    CKS(cudaMalloc((void**)&st->ft, sizeof(float) * n));
    CKS(cudaMalloc((void**)&st->epart, sizeof(double) * B * st->ntiles * st->groups));
    CKS(cudaMalloc((void**)&st->ppart, sizeof(double) * 2 * B * st->nblk2 * foe::kNumPart));
    CKS(cudaMalloc((void**)&st->trace, sizeof(double) * B * (cfg.max_iters + 1) * 8));
    CKS(cudaMemset(st->trace, 0, sizeof(double) * B * (cfg.max_iters + 1) * 8));
    CKS(cudaMalloc((void**)&st->ctl, sizeof(ImgCtl) * B * std::max(1, st->pgrid)));
    if (st->solver == FOE_SOLVER_PERSISTENT) {
        CKS(cudaMalloc((void**)&st->bar, sizeof(unsigned int)));
        if (md->persist_phases) {
            CKS(cudaMalloc((void**)&st->phase_ns, sizeof(unsigned long long) * 4 * foe::kPhaseRounds));
            CKS(cudaMemset(st->phase_ns, 0, sizeof(unsigned long long) * 4 * foe::kPhaseRounds));
        }
    }
    CKS(cudaMallocHost((void**)&st->hctl, sizeof(ImgCtl) * B));
    st->lam.resize(2 * (size_t)B);
    for (int b = 0; b < B; ++b) {
        st->lam[2 * b] = lambda_per_image ? lambda_per_image[2 * b] : md->lam[0];
        st->lam[2 * b + 1] = md->term != FOE_DATA_COMBINED ? 0.0 : (lambda_per_image ? lambda_per_image[2 * b + 1] : md->lam[1]);
    }
    rs = state_init(st, f, lipschitz_init, (cudaStream_t)stream);
    if (rs != FOE_OK) return cleanup(rs);
#undef CKS
    *out = st;
    return FOE_OK;
}

// replace the per-image lambdas of an existing state (validated like ipiano_state_create)
static foe_status set_state_lambdas(ipiano_state* st, const double* lambda_per_image) {
    const foe_model* md = st->model;
    for (int b = 0; b < st->B; ++b) {
        const double l1 = lambda_per_image ? lambda_per_image[2 * b] : md->lam[0];
        const double l2 = md->term != FOE_DATA_COMBINED ? 0.0 : (lambda_per_image ? lambda_per_image[2 * b + 1] : md->lam[1]);
        if (!(l1 >= 0) || !(l2 >= 0) || !std::isfinite(l1) || !std::isfinite(l2) || (l1 == 0 && l2 == 0))
            return fail(FOE_ERR_INVALID_ARGUMENT, "lambda of image %d = (%g,%g) invalid", b, l1, l2);
        st->lam[2 * b] = l1;
        st->lam[2 * b + 1] = l2;
    }
    return FOE_OK;
}

foe_status ipiano_state_reset(ipiano_state* st, const float* f, const double* lipschitz_init, void* stream) {
    if (!st) return fail(FOE_ERR_INVALID_ARGUMENT, "state is NULL");
    if (!f || !lipschitz_init) return fail(FOE_ERR_INVALID_ARGUMENT, "f and lipschitz_init must be non-NULL");
    for (int b = 0; b < st->B; ++b)
        if (!(lipschitz_init[b] > 0.0) || !std::isfinite(lipschitz_init[b]))
            return fail(FOE_ERR_INVALID_ARGUMENT, "lipschitz_init[%d]=%g must be > 0", b, lipschitz_init[b]);
    CK(cudaSetDevice(st->model->dev));
    return state_init(st, f, lipschitz_init, (cudaStream_t)stream);
}

foe_status ipiano_solve(ipiano_state* st, void* stream) {
    if (!st) return fail(FOE_ERR_INVALID_ARGUMENT, "state is NULL");
    CK(cudaSetDevice(st->model->dev));
    cudaStream_t user = (cudaStream_t)stream;
    foe_status r = join_begin(st, user);
    if (r != FOE_OK) return r;
    foe::k_set_target<<<div_up(st->B, 128), 128, 0, st->s>>>(st->ctl, st->B, st->cfg.max_iters);
    count_launch(1);
    CKL("k_set_target");
    r = sync_ctl(st);
    if (r != FOE_OK) return r;
    const long long max_rounds = (long long)st->cfg.max_iters * (st->cfg.max_backtracks + 2) + 8;
    long long done_rounds = 0;
    for (;;) {
        int min_n = st->cfg.max_iters;
        bool any = false;
        for (int b = 0; b < st->B; ++b)
            if (st->hctl[b].active) { any = true; min_n = std::min(min_n, st->hctl[b].n); }
        if (!any || done_rounds > max_rounds) break;
        const long long rounds = st->solver == FOE_SOLVER_PERSISTENT && !st->profile
                                     ? max_rounds - done_rounds + 1
                                     : std::max(1, st->cfg.max_iters - min_n);
        r = launch_rounds(st, rounds);
        if (r != FOE_OK) return r;
        done_rounds += rounds;
        r = sync_ctl(st);
        if (r != FOE_OK) return r;
    }
    r = join_end(st, user);
    if (r != FOE_OK) return r;
    return first_image_error(st);
}

foe_status ipiano_step(ipiano_state* st, void* stream, int* accepted_iters_out) {
    if (!st) return fail(FOE_ERR_INVALID_ARGUMENT, "state is NULL");
    CK(cudaSetDevice(st->model->dev));
    cudaStream_t user = (cudaStream_t)stream;
    foe_status r = join_begin(st, user);
    if (r != FOE_OK) return r;
    r = sync_ctl(st);
    if (r != FOE_OK) return r;
    // per-image target n_b + 1 (capped at max_iters)
    for (int b = 0; b < st->B; ++b) {
        ImgCtl& c = st->hctl[b];
        c.target = std::min(c.n + 1, st->cfg.max_iters);
        c.active = (c.status == 0 && !c.done && c.n < c.target) ? 1 : 0;
    }
    CK(cudaMemcpyAsync(st->ctl, st->hctl, sizeof(ImgCtl) * st->B, cudaMemcpyHostToDevice, st->s));
    const int max_rounds = st->cfg.max_backtracks + 2;
    for (int i = 0; i < max_rounds; ++i) {
        bool any = false;
        for (int b = 0; b < st->B; ++b) any |= st->hctl[b].active != 0;
        if (!any) break;
        r = launch_rounds(st, st->solver == FOE_SOLVER_PERSISTENT ? max_rounds - i : 1);
        if (r != FOE_OK) return r;
        r = sync_ctl(st);
        if (r != FOE_OK) return r;
    }
    if (accepted_iters_out)
        for (int b = 0; b < st->B; ++b) accepted_iters_out[b] = st->hctl[b].n;
    r = join_end(st, user);
    if (r != FOE_OK) return r;
    return first_image_error(st);
}

foe_status ipiano_get_iterate(const ipiano_state* st, double* w_out, float* u_out, void* stream) {
    if (!st) return fail(FOE_ERR_INVALID_ARGUMENT, "state is NULL");
    CK(cudaSetDevice(st->model->dev));
    ipiano_state* s = const_cast<ipiano_state*>(st);
    cudaStream_t user = (cudaStream_t)stream;
    foe_status r = join_begin(s, user);
    if (r != FOE_OK) return r;
    if (w_out || u_out) {
        const int gx = std::max(1, std::min(div_up((long long)st->HW, 256), 4 * st->model->nsm));
        foe::k_iterate_out<<<dim3(gx, st->B), 256, 0, s->s>>>(st->ctl, st->w, (size_t)st->B * st->HW, w_out,
                                                              u_out, st->HW, st->model->term == FOE_DATA_IDIV);
        CKL("k_iterate_out");
        count_launch(1);
    }
    return join_end(s, user);
}

foe_status ipiano_get_counters(const ipiano_state* st, int* iters, int* trials, int* status, double* lipschitz) {
    if (!st) return fail(FOE_ERR_INVALID_ARGUMENT, "state is NULL");
    CK(cudaSetDevice(st->model->dev));
    ipiano_state* s = const_cast<ipiano_state*>(st);
    foe_status r = sync_ctl(s);
    if (r != FOE_OK) return r;
    for (int b = 0; b < st->B; ++b) {
        if (iters) iters[b] = st->hctl[b].n;
        if (trials) trials[b] = st->hctl[b].total_trials;
        if (status) status[b] = st->hctl[b].status;
        if (lipschitz) lipschitz[b] = st->hctl[b].L;
    }
    return FOE_OK;
}

foe_status ipiano_get_trace(const ipiano_state* st, void* host_trace, size_t bytes) {
    if (!st || !host_trace) return fail(FOE_ERR_INVALID_ARGUMENT, "state or host_trace is NULL");
    const size_t need = sizeof(double) * 8 * st->B * (size_t)(st->cfg.max_iters + 1);
    if (bytes < need) return fail(FOE_ERR_INVALID_ARGUMENT, "trace buffer %zu bytes < %zu", bytes, need);
    CK(cudaSetDevice(st->model->dev));
    CK(cudaMemcpyAsync(host_trace, st->trace, need, cudaMemcpyDeviceToHost, st->s));
    CK(cudaStreamSynchronize(st->s));
    return FOE_OK;
}

foe_status ipiano_profile(ipiano_state* st, int enable) {
    if (!st) return fail(FOE_ERR_INVALID_ARGUMENT, "state is NULL");
    st->profile = enable != 0;
    return FOE_OK;
}

foe_status ipiano_profile_read(ipiano_state* st, double* k1_ms, long long* k1_launches, long long* total_launches) {
    if (!st) return fail(FOE_ERR_INVALID_ARGUMENT, "state is NULL");
    CK(cudaSetDevice(st->model->dev));
    foe_status r = sync_ctl(st);
    if (r != FOE_OK) return r;
    if (k1_ms) *k1_ms = st->k1_ms;
    if (k1_launches) *k1_launches = st->k1_launches;
    if (total_launches) *total_launches = st->total_launches;
    st->k1_ms = 0.0;
    st->k1_launches = 0;
    st->total_launches = 0;
    return FOE_OK;
}

foe_status ipiano_profile_read_k2(ipiano_state* st, double* k2_ms, long long* k2_launches) {
    if (!st) return fail(FOE_ERR_INVALID_ARGUMENT, "state is NULL");
    CK(cudaSetDevice(st->model->dev));
    foe_status r = sync_ctl(st);
    if (r != FOE_OK) return r;
    if (k2_ms) *k2_ms = st->k2_ms;
    if (k2_launches) *k2_launches = st->k2_launches;
    st->k2_ms = 0.0;
    st->k2_launches = 0;
    return FOE_OK;
}

foe_status ipiano_run(const foe_model* md, const float* f, int B, int H, int W, const double* lambda_per_image,
                      const double* lipschitz_init, const ipiano_config* cfg, float* u_out, void* trace,
                      size_t trace_bytes, void* stream) {
    foe_status r = check_dims(md, B, H, W);
    if (r != FOE_OK) return r;
    if (!f || !u_out) return fail(FOE_ERR_INVALID_ARGUMENT, "f and u_out must be non-NULL");
    if (!lipschitz_init) return fail(FOE_ERR_INVALID_ARGUMENT, "lipschitz_init is NULL");
    CK(cudaSetDevice(md->dev));
    cudaStream_t s = (cudaStream_t)stream;
    const size_t n = (size_t)B * H * W;
    const bool f_dev = is_device_ptr(f), u_dev = is_device_ptr(u_out);
    ipiano_config c;
    if (cfg) c = *cfg; else ipiano_config_default(&c);
    std::unique_lock<std::mutex> lk(md->run_mu, std::try_to_lock);
    const bool cached = lk.owns_lock();
    // staging buffers for host I/O
    float* df = nullptr;
    float* du = nullptr;
    if (!f_dev || !u_dev) {
        if (cached) {
            if (md->io_n < n) {
                if (md->io_buf) cudaFree(md->io_buf);
                md->io_buf = nullptr;
                md->io_n = 0;
                CK(cudaMalloc((void**)&md->io_buf, sizeof(float) * 2 * n));
                md->io_n = n;
            }
            df = md->io_buf;
            du = md->io_buf + md->io_n;
        } else {
            CK(cudaMallocFromPoolAsync((void**)&df, sizeof(float) * 2 * n, md->pool, s));
            du = df + n;
        }
    }
    if (!f_dev) CK(cudaMemcpyAsync(df, f, sizeof(float) * n, cudaMemcpyHostToDevice, s));
    const float* fd = f_dev ? f : df;
    // the solver state: reuse the cached one when shape and configuration match
    ipiano_state* st = nullptr;
    bool own = true;
    if (cached && md->run_state && md->run_state->B == B && md->run_state->H == H && md->run_state->W == W &&
        std::memcmp(&md->run_state->cfg_in, &c, sizeof(c)) == 0) {
        st = md->run_state;
        own = false;
        r = set_state_lambdas(st, lambda_per_image);
        if (r == FOE_OK) r = ipiano_state_reset(st, fd, lipschitz_init, stream);
    } else {
        r = ipiano_state_create(md, fd, B, H, W, lambda_per_image, lipschitz_init, &c, stream, &st);
        if (r == FOE_OK) st->cfg_in = c;
        if (r == FOE_OK && cached) {
            if (md->run_state) ipiano_state_destroy(md->run_state);
            md->run_state = st;
            own = false;
        }
    }
    if (r == FOE_OK) r = ipiano_solve(st, stream);
    foe_status r2 = FOE_OK;
    if (st) {
        const std::string keep = g_err;
        r2 = ipiano_get_iterate(st, nullptr, u_dev ? u_out : du, stream);
        if (r2 == FOE_OK && trace) r2 = ipiano_get_trace(st, trace, trace_bytes);
        if (own) ipiano_state_destroy(st);
        if (r != FOE_OK) g_err = keep;
    }
    if (!u_dev && r2 == FOE_OK) CK(cudaMemcpyAsync(u_out, du, sizeof(float) * n, cudaMemcpyDeviceToHost, s));
    if (df && !cached) CK(cudaFreeAsync(df, s));
    CK(cudaStreamSynchronize(s));
    return r != FOE_OK ? r : r2;
}

}  // extern "C"

// ============================================================================ row slabs
//
// One periodic scene cut into `nslabs` equal row slabs (BASELINE.json
// configs[4]).  Per trial round every slab runs
//   A  K2 on its rows; w+ of its first/last kHalo rows is stored by K2 itself straight into the
//      neighbours' ghost rows (in-process slabs, or peer GPUs through CUDA IPC mappings), or
//      into a send buffer for NCCL
//   X  halo exchange: top ghost rows <- the slab above's last kHalo rows, bottom ghost rows
//      <- the slab below's first kHalo rows (ring: slab 0's top comes from slab G-1) -- nothing
//      to do in-process; a 1-element NCCL all-reduce (ordering) with peers; else ncclSend/Recv
//   B  K1 on its rows, reading the ghost rows (energy over owned responses, g+ on owned px)
//   R  per-band (64-row) partials of K1 and K2 into its part of the global band array
//   Y  gather of the band arrays (NCCL all-gather; in-process slabs share the array)
//   C  K3 on the global band array: every slab takes the identical decision.
// Bands are a fixed partition of the scene and every reduction has a fixed order, so the
// iterate and the trace are bitwise identical for any number of slabs.

#include <dlfcn.h>
#include <nccl.h>

namespace {

struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// NCCL is resolved at run time (the copy torch already loaded, else the system one), so that
// libfoe itself loads without it; only the multi-process slab path needs it.
const NcclApi& nccl_api() {
    static NcclApi api;
    static bool tried = false;
    static std::atomic<int> lock{0};
    while (lock.exchange(1)) {}
    if (!tried) {
        tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
            api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
            api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
            api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
            api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
            api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
            api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
            api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
            api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
            api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
            api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.GroupStart && api.GroupEnd &&
                     api.Send && api.Recv && api.AllGather && api.AllReduce && api.GetErrorString;
        }
    }
    lock.store(0);
    return api;
}

foe_status nccl_fail(ncclResult_t r, const char* what, int line) {
    const NcclApi& api = nccl_api();
    return fail(FOE_ERR_COMM, "%s failed: %s (foe_api.cu:%d)", what,
                api.GetErrorString ? api.GetErrorString(r) : "?", line);
}
#define CKN(call)                                                         \
    do {                                                                  \
        ncclResult_t r_ = (call);                                         \
        if (r_ != ncclSuccess) return nccl_fail(r_, #call, __LINE__);     \
    } while (0)

}  // namespace

struct foe_comm {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0, dev = 0;
};

struct ipiano_slabs {
    const foe_model* model = nullptr;
    const foe_comm* comm = nullptr;        // nullptr: all slabs in this process
    int nslabs = 1, first = 0;             // global slab index of members[0]
    int Hs = 0, W = 0, Hg = 0;             // slab rows, columns, scene rows
    int nb_local = 0, nb_global = 0, e_per_band = 0, bpb = 0, pxt = 8;
    std::vector<ipiano_state*> members;    // slabs owned by this process, in ring order
    double* band_all = nullptr;            // [nb_global][kNumPart]
    double* halo = nullptr;                // [members][2][kHalo][W] received ghost rows
    double* halo_send = nullptr;           // [members][2][kHalo][W] own boundary rows (NCCL send path)
    // fused exchange: K2 stores its boundary rows straight into the neighbours' ghost rows
    // (in-process slabs always; across processes after ipiano_slabs_connect_peers, through
    // CUDA IPC mappings of the neighbours' ghost buffers over NVLink)
    bool p2p = false;
    double* peer_up = nullptr;             // the slab above's ghost buffer (mapped), or own (1 rank)
    double* peer_dn = nullptr;             // the slab below's ghost buffer
    bool up_opened = false, dn_opened = false;
    int* barrier_buf = nullptr;            // 1 int: the NCCL all-reduce that orders peer stores before K1
    cudaStream_t s = nullptr;
    cudaStream_t sx = nullptr;             // the ghost-row exchange, overlapped with interior K8 bands
    cudaEvent_t sync_ev = nullptr;
    cudaEvent_t ev_k2 = nullptr, ev_x = nullptr;
    cudaGraphExec_t graph = nullptr;
    bool use_graph = true;
};

namespace {

size_t halo_elems(const ipiano_slabs* g) { return (size_t)2 * foe::kHalo * g->W; }

// Where member j's boundary rows go: top rows -> the slab above's bottom ghost rows, bottom rows
// -> the slab below's top ghost rows (or this slab's send buffer on the NCCL send/recv path).
void halo_dst(ipiano_slabs* g, int j, double*& up_dst, double*& dn_dst) {
    const size_t he = halo_elems(g), hp = (size_t)foe::kHalo * g->W;
    if (g->comm == nullptr) {
        const int n = (int)g->members.size();
        up_dst = g->halo + (size_t)((j + n - 1) % n) * he + hp;
        dn_dst = g->halo + (size_t)((j + 1) % n) * he;
    } else if (g->p2p) {
        up_dst = g->peer_up + hp;
        dn_dst = g->peer_dn;
    } else {
        up_dst = g->halo_send;
        dn_dst = g->halo_send + hp;
    }
}

// A (K2 + pack) for member j
foe_status slab_k2(ipiano_slabs* g, int j) {
    ipiano_state* st = g->members[j];
    foe::K2Args a2{};
    a2.w = st->w;
    a2.w_slot_stride = st->HW;
    a2.g = st->g;
    a2.g_group_stride = st->HW;
    a2.g_slot_stride = a2.g_group_stride * st->groups;
    a2.ft = st->ft;
    a2.ppart = st->ppart;
    a2.ctl = st->ctl;
    a2.sp = st->sp;
    a2.groups = st->groups;
    a2.nblk = st->nblk2;
    a2.HW = st->HW;
    halo_dst(g, j, a2.halo_up, a2.halo_dn);
    a2.halo_sys_fence = g->p2p && g->comm && g->comm->nranks > 1;
    a2.halo_px = (size_t)foe::kHalo * g->W;
    a2.idiv = st->model->term == FOE_DATA_IDIV;
    a2.pairs = FOE_K2_PAIRS && st->HW % 4 == 0;
    if (st->pxt2 == 16) foe::k_inertial_prox<16><<<dim3(st->nblk2, 1), kThreads, 0, g->s>>>(a2);
    else foe::k_inertial_prox<kPxt2><<<dim3(st->nblk2, 1), kThreads, 0, g->s>>>(a2);
    count_launch(1);
    CKL("k_inertial_prox (slab)");
    return FOE_OK;
}

// X: ghost rows.  Top ghost of slab i = last kHalo rows of slab i-1; bottom ghost = first
// kHalo rows of slab i+1 (periodic ring).
foe_status slab_exchange(ipiano_slabs* g, cudaStream_t xs) {
    const size_t hp = (size_t)foe::kHalo * g->W;
    if (g->comm == nullptr) return FOE_OK;   // K2 stored the rows into the neighbours' ghost buffers
    const NcclApi& api = nccl_api();
    if (g->p2p) {
        // the peers' K2 stored straight into our ghost rows; a 1-element all-reduce orders every
        // rank's K2 (and its system-scope fence) before any rank's K1
        if (g->comm->nranks > 1)
            CKN(api.AllReduce(g->barrier_buf, g->barrier_buf, 1, ncclInt32, ncclSum, g->comm->comm, xs));
        return FOE_OK;
    }
    // One fixed posting order on every rank (foe_slab_exchange_plan, which tests/test_dist.py
    // replays with gloo), so that two messages between the same pair of ranks (G = 2, or G = 1
    // to itself) match: send up, recv down, send down, recv up.
    int plan[4][3];
    foe_slab_exchange_plan(g->comm->nranks, g->comm->rank, &plan[0][0]);
    double* buf[4] = {g->halo_send, g->halo + hp, g->halo_send + hp, g->halo};   // FOE_HALO_* ids
    CKN(api.GroupStart());
    for (int k = 0; k < 4; ++k) {
        if (plan[k][0] == FOE_HALO_SEND) CKN(api.Send(buf[plan[k][2]], hp, ncclFloat64, plan[k][1], g->comm->comm, xs));
        else CKN(api.Recv(buf[plan[k][2]], hp, ncclFloat64, plan[k][1], g->comm->comm, xs));
    }
    CKN(api.GroupEnd());
    return FOE_OK;
}

K1Args slab_k1_args(ipiano_slabs* g, int j, int which_cur) {
    ipiano_state* st = g->members[j];
    K1Args a = state_k1_args(st, which_cur);
    a.w_slot_stride = st->HW;
    a.g_group_stride = st->HW;
    a.g_slot_stride = a.g_group_stride * st->groups;
    a.halo = g->halo + j * halo_elems(g);
    return a;
}

// R + Y: band partials of every member into the global array, then the all-gather.
foe_status slab_bands(ipiano_slabs* g) {
    for (size_t j = 0; j < g->members.size(); ++j) {
        ipiano_state* st = g->members[j];
        double* out = g->band_all + (size_t)(g->first + (int)j) * g->nb_local * foe::kNumPart;
        foe::k_band_reduce<<<g->nb_local, kThreads, 0, g->s>>>(st->epart, g->e_per_band, st->ppart, g->bpb, out);
        count_launch(1);
        CKL("k_band_reduce");
    }
    if (g->comm != nullptr && g->comm->nranks > 1) {
        const NcclApi& api = nccl_api();
        const size_t cnt = (size_t)g->nb_local * foe::kNumPart;
        CKN(api.AllGather(g->band_all + (size_t)g->comm->rank * cnt, g->band_all, cnt, ncclFloat64, g->comm->comm,
                          g->s));
    }
    return FOE_OK;
}

foe_status slab_round(ipiano_slabs* g, bool timed) {
    foe_status r;
    for (size_t j = 0; j < g->members.size(); ++j)
        if ((r = slab_k2(g, (int)j)) != FOE_OK) return r;
    // K8 in two parts: the interior bands need no ghost rows and run while
    // the exchange (NCCL on the side stream sx) moves them; the two boundary bands follow it.  The
    // same tiles with the same arithmetic either way, so the result does not depend on the split.
    const ipiano_state* s0 = g->members[0];
    const bool split = s0->kind == FOE_STENCIL_TENSOR && g->nb_local >= 3 && s0->tc_rows == kTcR;
    const int tx = s0->tiles_x, nb = g->nb_local;
    auto k8 = [&](int j, int tile_off, int ntiles) -> foe_status {
        ipiano_state* st = g->members[j];
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (timed) {
            e0 = pool_event(st);
            e1 = pool_event(st);
            CK(cudaEventRecord(e0, g->s));
        }
        K1Args a = slab_k1_args(g, j, 0);
        a.tile_off = tile_off;
        foe_status rl = launch_prior(st->model, st->kind, a, 1, g->s, ntiles);
        if (rl != FOE_OK) return rl;
        if (timed) {
            CK(cudaEventRecord(e1, g->s));
            st->ev_live.emplace_back(e0, e1);
            st->k1_launches += 1;
        }
        return FOE_OK;
    };
    if (split) {
        CK(cudaEventRecord(g->ev_k2, g->s));
        CK(cudaStreamWaitEvent(g->sx, g->ev_k2, 0));
        if ((r = slab_exchange(g, g->sx)) != FOE_OK) return r;
        CK(cudaEventRecord(g->ev_x, g->sx));
        for (size_t j = 0; j < g->members.size(); ++j)
            if ((r = k8((int)j, tx, (nb - 2) * tx)) != FOE_OK) return r;                 // interior bands
        CK(cudaStreamWaitEvent(g->s, g->ev_x, 0));
        for (size_t j = 0; j < g->members.size(); ++j) {
            if ((r = k8((int)j, 0, tx)) != FOE_OK) return r;                             // band 0
            if ((r = k8((int)j, (nb - 1) * tx, s0->ntiles - (nb - 1) * tx)) != FOE_OK) return r;   // last band
        }
    } else {
        if ((r = slab_exchange(g, g->s)) != FOE_OK) return r;
        for (size_t j = 0; j < g->members.size(); ++j)
            if ((r = k8((int)j, 0, -1)) != FOE_OK) return r;
    }
    if ((r = slab_bands(g)) != FOE_OK) return r;
    for (size_t j = 0; j < g->members.size(); ++j) {
        ipiano_state* st = g->members[j];
        foe::K3Args a3{};
        a3.ctl = st->ctl;
        a3.epart = g->band_all + 7;
        a3.estride = foe::kNumPart;
        a3.ppart = g->band_all;
        a3.trace = st->trace;
        a3.ne = g->nb_global;
        a3.nblk = g->nb_global;
        a3.sp = st->sp;
        foe::k_decide<<<1, kThreads, 0, g->s>>>(a3);
        count_launch(1);
        CKL("k_decide (slab)");
        st->total_launches += 4;
    }
    return FOE_OK;
}

foe_status slab_init(ipiano_slabs* g, const float* f, double L_init, cudaStream_t user) {
    CK(cudaEventRecord(g->sync_ev, user));
    CK(cudaStreamWaitEvent(g->s, g->sync_ev, 0));
    const size_t HWs = (size_t)g->Hs * g->W;
    for (size_t j = 0; j < g->members.size(); ++j) {
        ipiano_state* st = g->members[j];
        ImgCtl& c = st->hctl[0];
        std::memset(&c, 0, sizeof(c));
        c.L = L_init;
        c.lam1 = st->lam[0];
        c.lam2 = st->lam[1];
        c.cur = 0; c.prev = 1; c.cand = 2;
        c.gcur = 0; c.gcand = 1;
        c.active = 1;
        CK(cudaMemcpyAsync(st->ctl, st->hctl, sizeof(ImgCtl), cudaMemcpyHostToDevice, g->s));
        if (st->cfg.record_trace)
            CK(cudaMemsetAsync(st->trace, 0, sizeof(double) * (st->cfg.max_iters + 1) * 8, g->s));
        double *up_dst, *dn_dst;
        halo_dst(g, (int)j, up_dst, dn_dst);
        foe::k_init<<<dim3(st->nblk2, 1), kThreads, 0, g->s>>>(f + j * HWs, st->ft, st->w, HWs, st->ppart, st->nblk2,
                                                                st->ctl, HWs, st->pxt2, up_dst, dn_dst,
                                                                (size_t)foe::kHalo * g->W, st->model->term == FOE_DATA_IDIV);
        count_launch(1);
        CKL("k_init (slab)");
    }
    foe_status r = slab_exchange(g, g->s);
    if (r != FOE_OK) return r;
    for (size_t j = 0; j < g->members.size(); ++j) {
        ipiano_state* st = g->members[j];
        foe_status rl = launch_prior(st->model, st->kind, slab_k1_args(g, (int)j, 1), 1, g->s);
        if (rl != FOE_OK) return rl;
    }
    if ((r = slab_bands(g)) != FOE_OK) return r;
    for (size_t j = 0; j < g->members.size(); ++j) {
        ipiano_state* st = g->members[j];
        foe::k_init_finalize<<<1, kThreads, 0, g->s>>>(st->ctl, g->band_all + 7, g->nb_global, foe::kNumPart,
                                                        g->band_all, g->nb_global, st->trace, st->cfg.max_iters,
                                                        st->cfg.record_trace);
        count_launch(1);
        CKL("k_init_finalize (slab)");
        foe::k_set_target<<<1, 128, 0, g->s>>>(st->ctl, 1, 0);
        count_launch(1);
        CKL("k_set_target (slab)");
    }
    CK(cudaEventRecord(g->sync_ev, g->s));
    CK(cudaStreamWaitEvent(user, g->sync_ev, 0));
    return FOE_OK;
}

foe_status slab_sync(ipiano_slabs* g) {
    for (ipiano_state* st : g->members)
        CK(cudaMemcpyAsync(st->hctl, st->ctl, sizeof(ImgCtl), cudaMemcpyDeviceToHost, g->s));
    CK(cudaStreamSynchronize(g->s));
    for (ipiano_state* st : g->members) {
        for (auto& pr : st->ev_live) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) st->k1_ms += ms;
            st->ev_pool.push_back(pr.first);
            st->ev_pool.push_back(pr.second);
        }
        st->ev_live.clear();
    }
    return FOE_OK;
}

foe_status slab_ensure_graph(ipiano_slabs* g) {
    if (g->graph) return FOE_OK;
    cudaGraph_t gr = nullptr;
    CK(cudaStreamBeginCapture(g->s, cudaStreamCaptureModeThreadLocal));
    foe_status r = FOE_OK;
    t_capturing = true;
    std::vector<long long> tl;
    for (ipiano_state* st : g->members) tl.push_back(st->total_launches);
    for (int i = 0; i < kGraphRounds && r == FOE_OK; ++i) r = slab_round(g, false);
    t_capturing = false;
    for (size_t j = 0; j < g->members.size(); ++j) g->members[j]->total_launches = tl[j];
    cudaError_t e = cudaStreamEndCapture(g->s, &gr);
    if (r != FOE_OK) { if (gr) cudaGraphDestroy(gr); return r; }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture (slabs)", __LINE__);
    e = cudaGraphInstantiate(&g->graph, gr, 0);
    cudaGraphDestroy(gr);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate (slabs)", __LINE__);
    return FOE_OK;
}

}  // namespace

extern "C" {

foe_status foe_slab_exchange_plan(int nranks, int rank, int* plan_out) {
    if (nranks < 1 || rank < 0 || rank >= nranks || !plan_out)
        return fail(FOE_ERR_INVALID_ARGUMENT, "nranks=%d rank=%d plan_out=%p", nranks, rank, (void*)plan_out);
    const int up = (rank + nranks - 1) % nranks, dn = (rank + 1) % nranks;
    const int plan[4][3] = {{FOE_HALO_SEND, up, FOE_HALO_TOP_ROWS},        // my first kHalo rows -> above
                            {FOE_HALO_RECV, dn, FOE_HALO_BOTTOM_GHOST},    // below's first rows
                            {FOE_HALO_SEND, dn, FOE_HALO_BOTTOM_ROWS},     // my last rows -> below
                            {FOE_HALO_RECV, up, FOE_HALO_TOP_GHOST}};      // above's last rows
    std::memcpy(plan_out, plan, sizeof(plan));
    return FOE_OK;
}

foe_status foe_comm_unique_id(void* id_out) {
    if (!id_out) return fail(FOE_ERR_INVALID_ARGUMENT, "id_out is NULL");
    const NcclApi& api = nccl_api();
    if (!api.ok) return fail(FOE_ERR_COMM, "libnccl.so.2 could not be loaded");
    ncclUniqueId id;
    CKN(api.GetUniqueId(&id));
    std::memcpy(id_out, &id, sizeof(id));
    return FOE_OK;
}

foe_status foe_comm_init(const void* nccl_unique_id, int nranks, int rank, foe_comm** out) {
    int dev = 0;
    const cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice", __LINE__);
    return foe_comm_create(nccl_unique_id, nranks, rank, dev, out);
}

foe_status foe_comm_create(const void* id, int nranks, int rank, int cuda_device, foe_comm** out) {
    if (!out) return fail(FOE_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (!id) return fail(FOE_ERR_INVALID_ARGUMENT, "id is NULL");
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return fail(FOE_ERR_INVALID_ARGUMENT, "rank=%d outside [0, nranks=%d)", rank, nranks);
    const NcclApi& api = nccl_api();
    if (!api.ok) return fail(FOE_ERR_COMM, "libnccl.so.2 could not be loaded");
    CK(cudaSetDevice(cuda_device));
    foe_comm* c = new (std::nothrow) foe_comm();
    if (!c) return fail(FOE_ERR_OUT_OF_MEMORY, "host allocation");
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclResult_t r = api.CommInitRank(&c->comm, nranks, uid, rank);
    cudaGetLastError();   // NCCL's own runtime probes may leave a stale error in this thread
    if (r != ncclSuccess) { delete c; return nccl_fail(r, "ncclCommInitRank", __LINE__); }
    c->nranks = nranks;
    c->rank = rank;
    c->dev = cuda_device;
    *out = c;
    return FOE_OK;
}

void foe_comm_destroy(foe_comm* c) {
    if (!c) return;
    const NcclApi& api = nccl_api();
    if (c->comm && api.ok) api.CommDestroy(c->comm);
    delete c;
    cudaGetLastError();   // NCCL's own runtime calls may leave a stale error in this thread
}

void ipiano_slabs_destroy(ipiano_slabs* g) {
    if (!g) return;
    cudaSetDevice(g->model->dev);
    if (g->s) cudaStreamSynchronize(g->s);
    for (ipiano_state* st : g->members) {
        st->s = nullptr;  // the group's stream
        ipiano_state_destroy(st);
    }
    if (g->graph) cudaGraphExecDestroy(g->graph);
    cudaFree(g->band_all);
    cudaFree(g->halo);
    cudaFree(g->halo_send);
    if (g->up_opened) cudaIpcCloseMemHandle(g->peer_up);
    if (g->dn_opened && g->peer_dn != g->peer_up) cudaIpcCloseMemHandle(g->peer_dn);
    if (g->barrier_buf) cudaFree(g->barrier_buf);
    if (g->sync_ev) cudaEventDestroy(g->sync_ev);
    if (g->ev_k2) cudaEventDestroy(g->ev_k2);
    if (g->ev_x) cudaEventDestroy(g->ev_x);
    if (g->sx) cudaStreamSynchronize(g->sx);
    if (g->s) cudaStreamDestroy(g->s);
    if (g->sx) cudaStreamDestroy(g->sx);
    delete g;
    cudaGetLastError();   // destroy reports nothing: leave no stale error for the next launch check
}

foe_status ipiano_slabs_create(const foe_model* md, const float* f, int H_global, int W, int nslabs,
                               const double* lambda, double lipschitz_init, const ipiano_config* cfg_in,
                               const foe_comm* comm, void* stream, ipiano_slabs** out) {
    if (!out) return fail(FOE_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (!md) return fail(FOE_ERR_INVALID_ARGUMENT, "model is NULL");
    if (!f) return fail(FOE_ERR_INVALID_ARGUMENT, "f is NULL");
    if (comm) nslabs = comm->nranks;
    if (comm && comm->dev != md->dev)
        return fail(FOE_ERR_INVALID_ARGUMENT, "comm is on cuda:%d, the model on cuda:%d", comm->dev, md->dev);
    if (nslabs < 1) return fail(FOE_ERR_INVALID_ARGUMENT, "nslabs=%d must be >= 1", nslabs);
    if (H_global % (nslabs * foe::kBandRows) != 0)
        return fail(FOE_ERR_INVALID_ARGUMENT, "H_global=%d must be a multiple of %d x nslabs=%d (64-row bands per slab)",
                    H_global, foe::kBandRows, nslabs);
    if (W % 32 != 0 || W < md->m)
        return fail(FOE_ERR_INVALID_ARGUMENT, "W=%d must be a multiple of 32 and >= m", W);
    if (!(lipschitz_init > 0.0) || !std::isfinite(lipschitz_init))
        return fail(FOE_ERR_INVALID_ARGUMENT, "lipschitz_init=%g must be > 0", lipschitz_init);
    CK(cudaSetDevice(md->dev));
    ipiano_slabs* g = new (std::nothrow) ipiano_slabs();
    if (!g) return fail(FOE_ERR_OUT_OF_MEMORY, "host allocation");
    auto cleanup = [&](foe_status s) { ipiano_slabs_destroy(g); return s; };
    g->model = md;
    g->comm = comm;
    g->nslabs = nslabs;
    g->first = comm ? comm->rank : 0;
    g->Hs = H_global / nslabs;
    g->W = W;
    g->Hg = H_global;
    const int nmem = comm ? 1 : nslabs;
    const int pref = cfg_in ? cfg_in->stencil : FOE_STENCIL_AUTO;
    if (pref == FOE_STENCIL_TENSOR && !md->tc_np) {
        delete g;
        return fail(FOE_ERR_UNSUPPORTED, "no tensor-core stencil for %d filters of %dx%d", md->nf, md->m, md->m);
    }
    // one plan for the whole scene, so that every slab (and every slab count) runs the same kernel
    const Plan pl = plan_stencil(md, 1, H_global / nslabs, W, H_global, pref, cfg_in ? cfg_in->filter_groups : 0,
                                 /*allow_pack=*/false);
    const int groups = pl.groups;
    g->nb_local = g->Hs / foe::kBandRows;
    g->nb_global = H_global / foe::kBandRows;
    g->e_per_band = pl.tiles_x * groups;   // K1 and K8 tiles are both 64 rows high: one tile row per band
    // K2 blocks never straddle a 64-row band: 16 pixels per thread when W % 64 == 0 (c5: 8192),
    // else kPxt2 = 8 (W % 32 == 0 is required)
    g->pxt = W % 64 == 0 ? 16 : kPxt2;
    g->bpb = foe::kBandRows * W / (kThreads * g->pxt);
    CK(cudaStreamCreateWithFlags(&g->s, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&g->sx, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&g->sync_ev, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&g->ev_k2, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&g->ev_x, cudaEventDisableTiming));
    const size_t he = halo_elems(g);
    if (cudaMalloc((void**)&g->band_all, sizeof(double) * g->nb_global * foe::kNumPart) != cudaSuccess ||
        cudaMalloc((void**)&g->halo, sizeof(double) * he * nmem) != cudaSuccess ||
        cudaMalloc((void**)&g->halo_send, sizeof(double) * he * nmem) != cudaSuccess)
        return cleanup(cuda_fail(cudaErrorMemoryAllocation, "cudaMalloc (slabs)", __LINE__));
    cudaMemset(g->band_all, 0, sizeof(double) * g->nb_global * foe::kNumPart);
    ipiano_config cfg;
    if (cfg_in) cfg = *cfg_in; else ipiano_config_default(&cfg);
    cfg.filter_groups = groups;
    cfg.stencil = pl.kind;
    cfg.solver = FOE_SOLVER_GRAPH;   // the slab rounds are driven by ipiano_slabs_* (kPxt2 K2 blocks)
    // members: per-slab iPiano states of one image (B = 1) sharing the group's stream.
    // ipiano_state_create evaluates w^0 with periodic wrap; slab_init below redoes it with halos.
    const size_t HWs = (size_t)g->Hs * W;
    for (int j = 0; j < nmem; ++j) {
        ipiano_state* st = nullptr;
        t_slab_member = true;   // per-band energy partials: no K8 column packing
        t_force_ncp = pl.ncp;   // and the whole scene's K1 chunking, so slabs are G-invariant
        t_force_pxt = g->pxt;   // and its K2 block size
        foe_status r = ipiano_state_create(md, f + (size_t)j * HWs, 1, g->Hs, W, lambda, &lipschitz_init, &cfg,
                                           stream, &st);
        t_slab_member = false;
        t_force_ncp = 0;
        t_force_pxt = 0;
        if (r != FOE_OK) return cleanup(r);
        cudaStreamSynchronize(st->s);
        cudaStreamDestroy(st->s);
        st->s = g->s;
        g->members.push_back(st);
    }
    foe_status r = slab_init(g, f, lipschitz_init, (cudaStream_t)stream);
    if (r != FOE_OK) return cleanup(r);
    *out = g;
    return FOE_OK;
}

foe_status ipiano_slabs_reset(ipiano_slabs* g, const float* f, double lipschitz_init, void* stream) {
    if (!g || !f) return fail(FOE_ERR_INVALID_ARGUMENT, "slabs or f is NULL");
    if (!(lipschitz_init > 0.0) || !std::isfinite(lipschitz_init))
        return fail(FOE_ERR_INVALID_ARGUMENT, "lipschitz_init=%g must be > 0", lipschitz_init);
    CK(cudaSetDevice(g->model->dev));
    return slab_init(g, f, lipschitz_init, (cudaStream_t)stream);
}

foe_status ipiano_slabs_solve(ipiano_slabs* g, void* stream) {
    if (!g) return fail(FOE_ERR_INVALID_ARGUMENT, "slabs is NULL");
    return ipiano_slabs_advance(g, g->members[0]->cfg.max_iters, stream);
}

foe_status ipiano_slabs_advance(ipiano_slabs* g, int target_iters, void* stream) {
    if (!g) return fail(FOE_ERR_INVALID_ARGUMENT, "slabs is NULL");
    if (target_iters < 0) return fail(FOE_ERR_INVALID_ARGUMENT, "target_iters=%d must be >= 0", target_iters);
    CK(cudaSetDevice(g->model->dev));
    cudaStream_t user = (cudaStream_t)stream;
    CK(cudaEventRecord(g->sync_ev, user));
    CK(cudaStreamWaitEvent(g->s, g->sync_ev, 0));
    const int max_iters = std::min(target_iters, g->members[0]->cfg.max_iters);
    for (ipiano_state* st : g->members) {
        foe::k_set_target<<<1, 128, 0, g->s>>>(st->ctl, 1, max_iters);
        count_launch(1);
    }
    CKL("k_set_target (slabs)");
    foe_status r = slab_sync(g);
    if (r != FOE_OK) return r;
    const bool timed = g->members[0]->profile;
    const long long max_rounds = (long long)max_iters * (g->members[0]->cfg.max_backtracks + 2) + 8;
    long long done = 0;
    for (;;) {
        const ImgCtl& c = g->members[0]->hctl[0];   // identical on every slab
        if (!c.active || done > max_rounds) break;
        const int rounds = std::max(1, max_iters - c.n);
        if (timed || !g->use_graph) {
            for (int i = 0; i < rounds; ++i)
                if ((r = slab_round(g, timed)) != FOE_OK) return r;
            done += rounds;
        } else {
            if ((r = slab_ensure_graph(g)) != FOE_OK) return r;
            const int reps = div_up(rounds, kGraphRounds);
            for (int i = 0; i < reps; ++i) {
                CK(cudaGraphLaunch(g->graph, g->s));
                count_launch(4LL * kGraphRounds * (long long)g->members.size());
                for (ipiano_state* st : g->members) st->total_launches += 4LL * kGraphRounds;
            }
            done += (long long)reps * kGraphRounds;
        }
        if ((r = slab_sync(g)) != FOE_OK) return r;
    }
    for (size_t j = 1; j < g->members.size(); ++j)
        if (std::memcmp(&g->members[j]->hctl[0], &g->members[0]->hctl[0], sizeof(ImgCtl)) != 0)
            return fail(FOE_ERR_COMM, "slab %d diverged from slab 0 (control blocks differ)", (int)j);
    CK(cudaEventRecord(g->sync_ev, g->s));
    CK(cudaStreamWaitEvent(user, g->sync_ev, 0));
    return first_image_error(g->members[0]);
}

foe_status ipiano_slabs_get_iterate(const ipiano_slabs* g, double* w_out, float* u_out, void* stream) {
    if (!g) return fail(FOE_ERR_INVALID_ARGUMENT, "slabs is NULL");
    CK(cudaSetDevice(g->model->dev));
    ipiano_slabs* gg = const_cast<ipiano_slabs*>(g);
    cudaStream_t user = (cudaStream_t)stream;
    CK(cudaEventRecord(gg->sync_ev, user));
    CK(cudaStreamWaitEvent(gg->s, gg->sync_ev, 0));
    const size_t HWs = (size_t)g->Hs * g->W;
    for (size_t j = 0; j < g->members.size(); ++j) {
        const ipiano_state* st = g->members[j];
        const int gx = std::max(1, std::min(div_up((long long)HWs, 256), 4 * g->model->nsm));
        foe::k_iterate_out<<<dim3(gx, 1), 256, 0, gg->s>>>(st->ctl, st->w, HWs, w_out ? w_out + j * HWs : nullptr,
                                                            u_out ? u_out + j * HWs : nullptr, HWs,
                                                            st->model->term == FOE_DATA_IDIV);
        count_launch(1);
        CKL("k_iterate_out (slabs)");
    }
    CK(cudaEventRecord(gg->sync_ev, gg->s));
    CK(cudaStreamWaitEvent(user, gg->sync_ev, 0));
    return FOE_OK;
}

foe_status ipiano_slabs_halo_handle(const ipiano_slabs* g, void* handle_out) {
    if (!g || !handle_out) return fail(FOE_ERR_INVALID_ARGUMENT, "slabs or handle_out is NULL");
    if (!g->comm) return fail(FOE_ERR_INVALID_ARGUMENT, "in-process slabs exchange directly; no handle needed");
    CK(cudaSetDevice(g->model->dev));
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, g->halo));
    std::memcpy(handle_out, &h, sizeof(h));
    return FOE_OK;
}

foe_status ipiano_slabs_connect_peers(ipiano_slabs* g, const void* up_handle, const void* down_handle) {
    if (!g || !up_handle || !down_handle) return fail(FOE_ERR_INVALID_ARGUMENT, "slabs or a handle is NULL");
    if (!g->comm) return fail(FOE_ERR_INVALID_ARGUMENT, "in-process slabs exchange directly");
    if (g->p2p) return fail(FOE_ERR_INVALID_ARGUMENT, "peers already connected");
    CK(cudaSetDevice(g->model->dev));
    const int R = g->comm->nranks, r = g->comm->rank;
    const int up = (r + R - 1) % R, dn = (r + 1) % R;
    auto open = [&](const void* hb, int peer, double*& ptr, bool& opened) -> foe_status {
        if (peer == r) { ptr = g->halo; opened = false; return FOE_OK; }   // 1 rank: the ring is this slab
        cudaIpcMemHandle_t h;
        std::memcpy(&h, hb, sizeof(h));
        void* p = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(FOE_ERR_COMM, "cudaIpcOpenMemHandle of rank %d's ghost rows failed: %s", peer,
                        cudaGetErrorString(e));
        }
        ptr = (double*)p;
        opened = true;
        return FOE_OK;
    };
    foe_status rs = open(up_handle, up, g->peer_up, g->up_opened);
    if (rs != FOE_OK) return rs;
    if (dn == up) { g->peer_dn = g->peer_up; g->dn_opened = g->up_opened; }
    else if ((rs = open(down_handle, dn, g->peer_dn, g->dn_opened)) != FOE_OK) return rs;
    if (!g->barrier_buf) {
        CK(cudaMalloc((void**)&g->barrier_buf, sizeof(int)));
        CK(cudaMemset(g->barrier_buf, 0, sizeof(int)));
    }
    g->p2p = true;
    if (g->graph) { cudaGraphExecDestroy(g->graph); g->graph = nullptr; }   // recapture with the new path
    return FOE_OK;
}

foe_status ipiano_slabs_disconnect_peers(ipiano_slabs* g) {
    if (!g) return fail(FOE_ERR_INVALID_ARGUMENT, "slabs is NULL");
    CK(cudaSetDevice(g->model->dev));
    CK(cudaStreamSynchronize(g->s));
    if (g->up_opened) cudaIpcCloseMemHandle(g->peer_up);
    if (g->dn_opened && g->peer_dn != g->peer_up) cudaIpcCloseMemHandle(g->peer_dn);
    g->peer_up = g->peer_dn = nullptr;
    g->up_opened = g->dn_opened = false;
    g->p2p = false;
    if (g->graph) { cudaGraphExecDestroy(g->graph); g->graph = nullptr; }
    return FOE_OK;
}

foe_status ipiano_slabs_member(const ipiano_slabs* g, int j, ipiano_state** out) {
    if (!g || !out) return fail(FOE_ERR_INVALID_ARGUMENT, "slabs or out is NULL");
    if (j < 0 || j >= (int)g->members.size())
        return fail(FOE_ERR_INVALID_ARGUMENT, "member %d outside [0,%d)", j, (int)g->members.size());
    *out = g->members[j];
    return FOE_OK;
}

}  // extern "C"

// ========================================================= evaluation / synthesis

namespace {

foe_status check_eval(const void* a, const void* b, int B, int H, int W) {
    if (!a || !b) return fail(FOE_ERR_INVALID_ARGUMENT, "image pointers must be non-NULL");
    if (B < 1 || H < 1 || W < 1) return fail(FOE_ERR_INVALID_ARGUMENT, "B=%d H=%d W=%d must be >= 1", B, H, W);
    int dev = 0;
    CK(cudaGetDevice(&dev));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10 || prop.minor != 0)
        return fail(FOE_ERR_CUDA, "libfoe is built for sm_100a (B200); the current device is sm_%d%d", prop.major, prop.minor);
    return FOE_OK;
}

// per-image sums of per-block partials [B][nblk] -> host [B]
foe_status sum_parts(const double* part, int B, int nblk, double* host, cudaStream_t s) {
    double* dsum = nullptr;
    CK(cudaMallocAsync((void**)&dsum, sizeof(double) * B, s));
    foe::k_reduce_rows<<<B, kThreads, 0, s>>>(part, nblk, 1, 1, dsum);
    count_launch(1);
    CKL("k_reduce_rows");
    CK(cudaMemcpyAsync(host, dsum, sizeof(double) * B, cudaMemcpyDeviceToHost, s));
    CK(cudaFreeAsync(dsum, s));
    CK(cudaStreamSynchronize(s));
    return FOE_OK;
}

}  // namespace

extern "C" {

foe_status foe_psnr(const float* x, const float* ref, int B, int H, int W, double peak, double* psnr_out,
                    void* stream) {
    foe_status r = check_eval(x, ref, B, H, W);
    if (r != FOE_OK) return r;
    if (!psnr_out || !(peak > 0)) return fail(FOE_ERR_INVALID_ARGUMENT, "psnr_out must be non-NULL and peak > 0");
    cudaStream_t s = (cudaStream_t)stream;
    const size_t HW = (size_t)H * W;
    const int nblk = std::max(1, std::min(div_up((long long)HW, kThreads * 8), 256));
    double* part = nullptr;
    CK(cudaMallocAsync((void**)&part, sizeof(double) * B * nblk, s));
    foe::k_sq_err_part<<<dim3(nblk, B), kThreads, 0, s>>>(x, ref, HW, nblk, part);
    count_launch(1);
    CKL("k_sq_err_part");
    std::vector<double> sse(B);
    r = sum_parts(part, B, nblk, sse.data(), s);
    cudaFreeAsync(part, s);
    if (r != FOE_OK) return r;
    for (int b = 0; b < B; ++b) {
        const double mse = sse[b] / (double)HW;   // 10 log10(peak^2 / MSE), +inf at MSE = 0
        psnr_out[b] = mse == 0.0 ? INFINITY : 10.0 * std::log10(peak * peak / mse);
    }
    return FOE_OK;
}

foe_status foe_ssim(const float* x, const float* ref, int B, int H, int W, double peak, double* ssim_out,
                    void* stream) {
    foe_status r = check_eval(x, ref, B, H, W);
    if (r != FOE_OK) return r;
    if (!ssim_out || !(peak > 0)) return fail(FOE_ERR_INVALID_ARGUMENT, "ssim_out must be non-NULL and peak > 0");
    if (H < 11 || W < 11) return fail(FOE_ERR_INVALID_ARGUMENT, "image %dx%d smaller than the 11x11 SSIM window", H, W);
    cudaStream_t s = (cudaStream_t)stream;
    foe::SsimParams sp;
    double g[11], gs = 0.0;
    for (int i = 0; i < 11; ++i) { const double r_ = i - 5.0; g[i] = std::exp(-r_ * r_ / (2.0 * 1.5 * 1.5)); gs += g[i]; }
    for (int i = 0; i < 11; ++i) sp.w[i] = g[i] / gs;
    sp.c1 = (0.01 * peak) * (0.01 * peak);
    sp.c2 = (0.03 * peak) * (0.03 * peak);
    const size_t on = (size_t)(H - 10) * (W - 10);
    const int nblk = std::max(1, std::min(div_up((long long)on, kThreads), 512));
    double* part = nullptr;
    CK(cudaMallocAsync((void**)&part, sizeof(double) * B * nblk, s));
    foe::k_ssim_part<<<dim3(nblk, B), kThreads, 0, s>>>(x, ref, H, W, nblk, sp, part);
    count_launch(1);
    CKL("k_ssim_part");
    std::vector<double> sum(B);
    r = sum_parts(part, B, nblk, sum.data(), s);
    cudaFreeAsync(part, s);
    if (r != FOE_OK) return r;
    for (int b = 0; b < B; ++b) ssim_out[b] = sum[b] / (double)on;
    return FOE_OK;
}

foe_status foe_add_speckle(const float* u, int B, int H, int W, const double* looks, unsigned long long seed,
                           float* f_out, void* stream) {
    foe_status r = check_eval(u, f_out, B, H, W);
    if (r != FOE_OK) return r;
    if (!looks) return fail(FOE_ERR_INVALID_ARGUMENT, "looks is NULL");
    for (int b = 0; b < B; ++b)
        if (!(looks[b] >= 1.0) || !std::isfinite(looks[b]))
            return fail(FOE_ERR_INVALID_ARGUMENT, "looks[%d]=%g: this generator needs L >= 1", b, looks[b]);
    cudaStream_t s = (cudaStream_t)stream;
    double* dl = nullptr;
    unsigned int* capped = nullptr;
    CK(cudaMallocAsync((void**)&dl, sizeof(double) * B, s));
    CK(cudaMallocAsync((void**)&capped, sizeof(unsigned int), s));
    CK(cudaMemcpyAsync(dl, looks, sizeof(double) * B, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(capped, 0, sizeof(unsigned int), s));
    const size_t n = (size_t)B * H * W;
    int nsm = 148;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int grid = std::max(1, std::min(div_up((long long)n, 256), 8 * nsm));
    foe::k_add_speckle<<<grid, 256, 0, s>>>(u, dl, B, (size_t)H * W, seed, f_out, capped);
    count_launch(1);
    CKL("k_add_speckle");
    unsigned int hc = 0;
    CK(cudaMemcpyAsync(&hc, capped, sizeof(hc), cudaMemcpyDeviceToHost, s));
    CK(cudaFreeAsync(dl, s));
    CK(cudaFreeAsync(capped, s));
    CK(cudaStreamSynchronize(s));
    if (hc) return fail(FOE_ERR_NONFINITE, "%u pixels exceeded 64 Marsaglia-Tsang attempts", hc);
    return FOE_OK;
}

}  // extern "C"
