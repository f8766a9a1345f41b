/*
 * foe.h -- C ABI of libfoe, the B200 (sm_100a) hot path of FoE-prior despeckling
 * solved by iPiano (Chen, Pock et al., arXiv:1404.5344; PAPER.md = the paper text).
 *
 * The library solves the combined model, Eq.(10) ("From now on,
 * we will use the combined model (10)"):
 *
 *     min_w  F(w) + G(w),
 *     F(w) = E_FoE(e^w) = sum_i theta_i sum_p rho((k_i * e^w)_p),  rho(x) = log(1+x^2)
 *                                                       (Eq.(2))
 *     G(w) = sum_p (l1/2)(2 w_p + f_p^2 e^{-2 w_p}) + (l2/2)(e^{2 w_p} - 2 f_p^2 w_p)
 *
 * with u = e^w, by iPiano
 *
 *     w^{n+1} = (I + a dG)^{-1}( w^n - a grad F(w^n) + b (w^n - w^{n-1}) ),
 *     grad_w F = W sum_i theta_i K_i^T rho'(K_i e^w), W = diag(e^w)
 *
 * the prox of G by Newton's method, and the backtracking
 * Lipschitz test F(w+) <= F(w) + <grad F(w), w+ - w> + (L_n/2)||w+ - w||^2 with
 * a = safety * 2(1-b)/L_n.  l2 = 0 is model (8).
 * Readings where the paper is silent (periodic boundary, true convolution, f~ = max(f,1),
 * the step policy, ...) are listed in DESIGN.md as R-1 .. R-17.
 *
 * Conventions (all entry points):
 *  - Every call returns foe_status; no C++ exception crosses the ABI.  On error,
 *    foe_last_error() returns a thread-local message naming the offending argument.
 *  - Images are contiguous row-major [B][H][W] arrays (B images of H rows by W columns).
 *    "device" pointers are CUDA device memory on the model's device (e.g. a torch
 *    tensor's data_ptr()); "host" pointers are ordinary (pageable or pinned) host memory.
 *  - The caller owns every array it passes; the model and state own their internal
 *    device memory and free it in *_destroy.  Inputs are never modified.
 *  - `stream` is a cudaStream_t passed as void* (NULL = the legacy default stream).
 *    Calls are asynchronous on that stream unless they return host values, in which
 *    case they synchronise it before returning.
 *  - There is no CPU fallback: without a usable sm_100a device every call that needs
 *    one fails with FOE_ERR_CUDA.
 */
#ifndef FOE_H_
#define FOE_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    FOE_OK = 0,
    FOE_ERR_INVALID_ARGUMENT = 1,    /* bad size/pointer/parameter (message names it)          */
    FOE_ERR_CUDA = 2,                /* CUDA runtime error, or no sm_100 device                 */
    FOE_ERR_OUT_OF_MEMORY = 3,
    FOE_ERR_NONFINITE = 4,           /* accepted energy/iterate non-finite        */
    FOE_ERR_BACKTRACK_LIMIT = 5,     /* more than max_backtracks doublings        */
    FOE_ERR_PROX_NO_CONVERGENCE = 6, /* Newton cap exceeded in the prox           */
    FOE_ERR_DOMAIN = 7,              /* accepted |w| above the guard (R-11)           */
    FOE_ERR_COMM = 8,                /* multi-GPU communication error                           */
    FOE_ERR_UNSUPPORTED = 9          /* valid request this build does not implement             */
} foe_status;

typedef enum {
    FOE_DATA_COMBINED = 0, /* Eq.(10): l1, l2 as given                                         */
    FOE_DATA_NAKAGAMI = 1, /* Eq.(8): l2 forced to 0, l1 = lambda            */
    FOE_DATA_IDIV = 2      /* model (6): iterate u (not w = log u),
                              D(u,f) = (lambda/2)<u^2 - 2 f^2 log u, 1>, lambda = lambda[0]
                              (lambda[1] ignored; no preset: the paper prints none), grad_u F
                              without W, closed-form prox; u^0 = max(f,1)       */
} foe_data_term;

/* Kernel of the fused prior energy + gradient (rows a2-a7):
 *   FOE_STENCIL_FFMA    K1: paired fp32 FMA (FFMA2) correlations out of shared memory
 *   FOE_STENCIL_TENSOR  K8: tcgen05 tensor cores, TF32 with a 3-pass hi/lo split (fp32-level),
 *                       m = 7 with N_f <= 48 or m = 5 with N_f <= 32 (else FOE_ERR_UNSUPPORTED)
 *   FOE_STENCIL_AUTO    K8 where supported and the launch fills the GPU, else K1. */
#define FOE_STENCIL_AUTO 0
#define FOE_STENCIL_FFMA 1
#define FOE_STENCIL_TENSOR 2

/* Limits of this build (kernel-parameter-resident filter taps). */
#define FOE_MAX_FILTERS 64
#define FOE_MAX_TAPS 3136  /* n_filters * m * m */

const char* foe_last_error(void);
const char* foe_status_string(foe_status s);
/* Library version string, and the compiled target (e.g. "sm_100a"). */
const char* foe_version(void);
/* Number of CUDA kernels this library has launched in this process (graph replays count
 * each captured kernel); for launch accounting in benchmarks. */
long long foe_kernel_launches(void);

/* ------------------------------------------------------------------------------ model */

typedef struct foe_model foe_model;

/* Creates the FoE model {(k_i, theta_i)} of Eq.(2) plus the data-term weights of Eq.(10).
 *   filters  host fp32 [n_filters][m][m] row-major taps k_i
 *   m        odd filter side; this build has kernels for m in {3, 5, 7} (else FOE_ERR_UNSUPPORTED)
 *   alphas   host fp32 [n_filters], the weights theta_i > 0 ("alphas" in BASELINE.json)
 *   lambda   host fp64 [2] = {l1, l2} (Eq.(10)), both >= 0 and not both 0; NULL -> the
 *            paper's preset for looks_L (L=8 (550,0.02), L=3 (310,0.008),
 *            L=1 (160,0.004); L=5 (50,0.15))
 *   looks_L  number of looks L; required (1, 3, 5 or 8) iff lambda == NULL, else informational
 *            (L is folded into lambda, R-5)
 *   term     FOE_DATA_COMBINED, FOE_DATA_NAKAGAMI or FOE_DATA_IDIV.  For FOE_DATA_IDIV every
 *            "w" below is the iterate u itself (device fp64), and lambda must be given
 *   cuda_device  CUDA ordinal the model's kernels run on
 * Errors: FOE_ERR_INVALID_ARGUMENT (m even/< 3, n_filters < 1 or > FOE_MAX_FILTERS,
 * n_filters*m*m > FOE_MAX_TAPS, theta_i <= 0 or non-finite (message names filter i),
 * non-finite taps, bad lambda/looks), FOE_ERR_CUDA (device unusable or not sm_100).
 * The model is immutable after creation and may be shared read-only between threads. */
foe_status foe_model_create(const float* filters, int n_filters, int m, const float* alphas,
                            const double* lambda, double looks_L, foe_data_term term,
                            int cuda_device, foe_model** out);
void foe_model_destroy(foe_model* model);
/* Stencil used by foe_energy_grad with this model (default FOE_STENCIL_AUTO; a tuning and
 * testing knob: do not change it while another thread uses the model).
 * FOE_ERR_UNSUPPORTED if the bank has no tensor-core kernel and FOE_STENCIL_TENSOR is asked. */
foe_status foe_model_set_stencil(foe_model* model, int stencil);

/* ------------------------------------------------------------------ energy / gradient */

/* Energy and prior gradient at the log-amplitude w:
 *   w                device fp64 [B][H][W]
 *   f                device fp32 [B][H][W] observation; used only for data_energy (may be NULL
 *                    if data_energy is NULL); f~ = max(f,1) is applied internally (R-4)
 *   lambda_per_image host fp64 [B][2] or NULL (-> the model's {l1,l2})
 *   prior_energy     host fp64 [B] or NULL: F(w) = E_FoE(e^w)
 *   data_energy      host fp64 [B] or NULL: G(w) of Eq.(10)
 *   grad             device fp32 [B][H][W] or NULL: grad_w F
 * Requires m <= min(H, W).  Periodic boundary (R-3).  Synchronises `stream`
 * when a host output is requested. */
foe_status foe_energy_grad(const foe_model* model, const double* w, const float* f, int B, int H,
                           int W, const double* lambda_per_image, double* prior_energy,
                           double* data_energy, float* grad, void* stream);

/* Hessian-vector product of F at w (R-10), device fp64 w, v -> device fp32 hv. */
foe_status foe_hvp(const foe_model* model, const double* w, const double* v, int B, int H, int W,
                   float* hv, void* stream);

/* Lipschitz initialisation (R-10): rho_hat = |Rayleigh quotient| after
 * `power_iters` power-iteration steps on the prior Hessian at w^0 = log max(f,1), from
 * the caller's start vectors v0 (device fp64 [B][H][W], any scale; the method's random
 * draw is an input).  rho_out (host [B], may be NULL) and L_out (host [B]) =
 * 2^ceil(log2 rho_hat).  Synchronises `stream`. */
foe_status foe_estimate_lipschitz(const foe_model* model, const float* f, int B, int H, int W,
                                  const double* v0, int power_iters, double* rho_out,
                                  double* L_out, void* stream);

/* ---------------------------------------------------------------------------- iPiano */

typedef struct {
    double beta;             /* inertia b in [0,1); graded policy 0.4 (R-9); SPEC default 0.8      */
    double step_safety;      /* a = step_safety * 2(1-b)/L_n, in (0,1]; 0.95          */
    double backtrack_factor; /* eta > 1: L_n <- eta L_n on a failed test; 2           */
    double shrink;           /* L_{n+1} = shrink * L_n after an accept, in (0,1]; 1 (R-9), SPEC 0.5  */
    int max_iters;           /* accepted iterations, >= 1                                            */
    int max_backtracks;      /* failed tests per iteration before FOE_ERR_BACKTRACK_LIMIT; 60       */
    int newton_max_iters;    /* Newton cap of the prox before FOE_ERR_PROX_NO_CONVERGENCE; 30       */
    double newton_tol;       /* |phi| tolerance of the prox root (fp64); 1e-12        */
    double rel_change_tol;   /* stop when ||w+ - w|| / max(||w||,1) < tol; 0 = never (benchmarks)    */
    double w_guard;          /* accepted |w| must stay <= w_guard; 40 (R-11)                          */
    int record_trace;        /* 1: keep the per-iteration trace on device                             */
    int filter_groups;       /* 0 = automatic; else split the N_f filters over this many CTAs
                                per tile (partial gradients summed in fixed order)                    */
    int stencil;             /* prior energy+gradient kernel: FOE_STENCIL_AUTO / _FFMA / _TENSOR     */
    int solver;              /* trial-loop driver: FOE_SOLVER_AUTO / _GRAPH / _PERSISTENT (below)    */
    int tile_rows;           /* tensor-core stencil output rows per tile: 0 = automatic (fewest waves
                                x rows), else one of 4, 8, 16, 32, 64; batch path only (slabs: 64) */
} ipiano_config;

/* Trial-loop drivers.  Both run the same K2 -> K1 -> K3 round per trial
 * (inertial point + prox, prior energy+gradient at the candidate, backtracking decision):
 *   FOE_SOLVER_GRAPH       three dependent launches per round, captured as a CUDA graph of 10
 *                          rounds; any size, either stencil.
 *   FOE_SOLVER_PERSISTENT  ONE cooperative launch runs all rounds: a co-resident grid does K2
 *                          and K1 as grid-strided phases separated by grid barriers, and every
 *                          CTA takes the (identical, fixed-order) decision itself.  FFMA stencil
 *                          only (FOE_ERR_UNSUPPORTED with FOE_STENCIL_TENSOR); for images that
 *                          cannot fill the GPU, where launches and their gaps dominate a round.
 *   FOE_SOLVER_AUTO        persistent when the state resolves to the FFMA stencil and
 *                          B*H*W < 2^16 (config c1; < 2^18 for banks without a tensor-core
 *                          stencil), else the graph (c2, c3: the tensor-core stencil in 4- and
 *                          8-row tiles).
 * ipiano_profile(st, 1) (per-launch K1 timing) always uses the graph driver. */
#define FOE_SOLVER_AUTO 0
#define FOE_SOLVER_GRAPH 1
#define FOE_SOLVER_PERSISTENT 2

/* Fills the defaults above (graded policy). */
void ipiano_config_default(ipiano_config* cfg);

/* Trace record per accepted iteration n (row 0 = the initial point w^0), fp64. */
typedef struct {
    double F;       /* F(w^n)                                             */
    double G;       /* G(w^n)                                             */
    double H;       /* F + G                                              */
    double L;       /* L_n used by the accepted trial                     */
    double trials;  /* trials of iteration n (1 = accepted at once)       */
    double margin;  /* F(w) + <g,D> + L/2 ||D||^2 - F(w+) >= 0             */
    double newton;  /* max Newton iterations of the accepted prox         */
    double relchg;  /* ||w^n - w^{n-1}|| / max(||w^{n-1}||, 1)           */
} ipiano_trace_rec;

typedef struct ipiano_state ipiano_state;

/* Allocates and initialises a batch of B independent problems (one per image):
 *   f                 device fp32 [B][H][W] observations (copied into the state; f~ = max(f,1))
 *   lambda_per_image  host fp64 [B][2] or NULL (-> model's)
 *   lipschitz_init    host fp64 [B], each > 0 (from foe_estimate_lipschitz, or the caller's)
 *   cfg               NULL -> defaults
 * Sets w^0 = log f~, w^{-1} = w^0 (R-8), evaluates F(w^0) and grad F(w^0) on `stream`.
 * Errors: FOE_ERR_INVALID_ARGUMENT (B < 1, H or W < m, bad cfg: beta outside [0,1),
 * max_iters < 1, step_safety outside (0,1], backtrack_factor <= 1, shrink outside (0,1]). */
foe_status ipiano_state_create(const foe_model* model, const float* f, int B, int H, int W,
                               const double* lambda_per_image, const double* lipschitz_init,
                               const ipiano_config* cfg, void* stream, ipiano_state** out);

/* Re-initialises an existing state from new observations f (same B, H, W; device fp32) and
 * Lipschitz initialisations, without reallocating: w^0 = log f~, w^{-1} = w^0, F(w^0),
 * grad F(w^0) (the same a1 step as ipiano_state_create).  Asynchronous on `stream`. */
foe_status ipiano_state_reset(ipiano_state* st, const float* f, const double* lipschitz_init, void* stream);

/* Advances every unfinished image by exactly one accepted iPiano iteration (as many
 * backtracking trials as it needs), then synchronises.  accepted_iters_out (host [B] or
 * NULL) receives each image's accepted-iteration count.  Returns the first per-image
 * error status if any image failed. */
foe_status ipiano_step(ipiano_state* st, void* stream, int* accepted_iters_out);

/* Runs until every image has max_iters accepted iterations (or stopped on
 * rel_change_tol, or failed).  Trial rounds are launched asynchronously in chunks (as a
 * CUDA graph) with one synchronisation per chunk. */
foe_status ipiano_solve(ipiano_state* st, void* stream);

/* Copies the current iterate out: w_out device fp64 [B][H][W] and/or u_out device fp32
 * [B][H][W] = e^w ("with u = e^w"); either may be NULL. */
foe_status ipiano_get_iterate(const ipiano_state* st, double* w_out, float* u_out, void* stream);

/* Per-image counters (host arrays [B], each may be NULL): accepted iterations, total
 * trials, status (foe_status per image), current L_n.  Synchronises the state's stream. */
foe_status ipiano_get_counters(const ipiano_state* st, int* iters, int* trials, int* status,
                               double* lipschitz);

/* Copies the trace to host: [B][max_iters+1] ipiano_trace_rec (bytes must be at least
 * B*(max_iters+1)*sizeof(ipiano_trace_rec)); rows past an image's iteration count are 0. */
foe_status ipiano_get_trace(const ipiano_state* st, void* host_trace, size_t bytes);

/* Device time (ms) spent in the fused prior-gradient kernel since the last call, and the
 * number of its launches; enabled by ipiano_profile(st, 1) (CUDA events around each launch). */
foe_status ipiano_profile(ipiano_state* st, int enable);
foe_status ipiano_profile_read(ipiano_state* st, double* k1_ms, long long* k1_launches,
                               long long* total_launches);
/* The same for K2 (k_inertial_prox: inertial step + prox + test partials) of the graph driver
 * (events before K2 and before the prior kernel of each profiled round); resets its counters. */
foe_status ipiano_profile_read_k2(ipiano_state* st, double* k2_ms, long long* k2_launches);

/* The stencil this state resolved to (FOE_STENCIL_FFMA or FOE_STENCIL_TENSOR). */
int ipiano_state_stencil(const ipiano_state* st);
/* The tensor-core stencil's tiling of a state (diagnostics, bench.py's executed-flops count):
 * output rows and columns per tile (64 x 122 with halos; x 128 without column halos) and the halo
 * mode -- 0 row and column halos, 1 no row halos, 2 neither (K8).  Zeros for
 * an FFMA-stencil state.  FOE_ERR_INVALID_ARGUMENT for a NULL state or output. */
foe_status ipiano_state_tiling(const ipiano_state* st, int* tile_rows, int* tile_cols, int* halo_mode);

/* The trial-loop driver this state resolved to (FOE_SOLVER_GRAPH or FOE_SOLVER_PERSISTENT). */
int ipiano_state_solver(const ipiano_state* st);

void ipiano_state_destroy(ipiano_state* st);

/* One-shot convenience: state_create + solve + get_iterate + get_trace + destroy.  The model
 * keeps one solver workspace (state + host-I/O staging buffers) for repeated calls of the same
 * B, H, W and configuration, so that a call after the first does no device allocation (a call
 * concurrent with another on the same model uses a private workspace); foe_model_destroy
 * frees it.
 *   f      fp32 [B][H][W], host OR device (detected); host buffers are copied in/out on
 *          `stream` inside the call
 *   u_out  fp32 [B][H][W] = e^w, host or device
 *   trace  host, may be NULL (then trace_bytes is ignored)
 * Synchronises `stream`. */
foe_status ipiano_run(const foe_model* model, const float* f, int B, int H, int W,
                      const double* lambda_per_image, const double* lipschitz_init,
                      const ipiano_config* cfg, float* u_out, void* trace, size_t trace_bytes,
                      void* stream);

/* ------------------------------------------------------------------ row slabs (multi-GPU) */

/* One periodic scene split into equal row slabs (BASELINE.json configs[4]):
 * per backtracking trial every slab computes w+ on its rows (K2), exchanges kHalo = 6 ghost
 * rows (= m-1 for m <= 7: the energy needs +-3 rows, the gradient +-6) with its two ring
 * neighbours, evaluates F and grad F on its rows (K1), and all slabs combine per-64-row-band
 * partials of the test into one global array in a fixed order, so every slab takes the same
 * decision and the result is bitwise independent of the number of slabs. */
typedef struct foe_comm foe_comm;

/* NCCL unique id (128 bytes) for foe_comm_create; call on one rank and broadcast the bytes
 * (e.g. with torch.distributed).  libnccl.so.2 is resolved at run time (the copy already
 * loaded by the process, else the system one); FOE_ERR_COMM if it cannot be loaded. */
foe_status foe_comm_unique_id(void* id_out);
/* Creates this rank's NCCL communicator (one process per GPU; collective over the nranks
 * processes).  cuda_device must be the device of the models used with it. */
foe_status foe_comm_create(const void* id, int nranks, int rank, int cuda_device, foe_comm** out);
/* SURVEY.md 8(b)'s name of the same call: foe_comm_create on the calling thread's current CUDA
 * device (cudaGetDevice); FOE_ERR_CUDA if that query fails. */
foe_status foe_comm_init(const void* nccl_unique_id, int nranks, int rank, foe_comm** out);
void foe_comm_destroy(foe_comm* comm);

/* The ghost-row exchange of one trial as the NCCL point-to-point calls
 * rank `rank` of `nranks` posts, in this order, on every rank (so that two messages between the
 * same pair of ranks -- 2 ranks, or 1 rank with itself -- match): plan_out[4][3] = {op, peer
 * rank, buffer}, op FOE_HALO_SEND / _RECV, buffer FOE_HALO_TOP_ROWS (this slab's first kHalo = 6
 * rows), _BOTTOM_GHOST (the ghost rows below the slab), _BOTTOM_ROWS (its last 6 rows),
 * _TOP_GHOST.  Host only (no CUDA call); the library's exchange follows it, and
 * tests/test_dist.py replays it with gloo.  FOE_ERR_INVALID_ARGUMENT unless 0 <= rank < nranks. */
#define FOE_HALO_SEND 0
#define FOE_HALO_RECV 1
#define FOE_HALO_TOP_ROWS 0
#define FOE_HALO_BOTTOM_GHOST 1
#define FOE_HALO_BOTTOM_ROWS 2
#define FOE_HALO_TOP_GHOST 3
foe_status foe_slab_exchange_plan(int nranks, int rank, int* plan_out);

typedef struct ipiano_slabs ipiano_slabs;

/* Creates the slab decomposition of ONE scene of H_global x W pixels and initialises it
 * (a1 on every slab, ghost rows exchanged, F(w^0), grad F(w^0)).
 *   comm == NULL: all `nslabs` slabs live in this process on the model's device (ghost rows
 *       and band partials move by device copies); f = the whole scene, device fp32
 *       [H_global][W].
 *   comm != NULL: this process owns slab comm->rank only (nslabs is taken from comm);
 *       f = that slab, device fp32 [H_global/nranks][W] = scene rows
 *       [rank H_global/nranks, (rank+1) H_global/nranks).
 *   lambda        host fp64 [2] or NULL (-> the model's)
 *   lipschitz_init  L_0 > 0, identical on every rank
 * Requires H_global a multiple of 64 * nslabs (whole 64-row bands per slab), W a multiple
 * of 32.  Errors: FOE_ERR_INVALID_ARGUMENT, FOE_ERR_CUDA, FOE_ERR_OUT_OF_MEMORY,
 * FOE_ERR_COMM (NCCL failure). */
foe_status ipiano_slabs_create(const foe_model* model, const float* f, int H_global, int W, int nslabs,
                               const double* lambda, double lipschitz_init, const ipiano_config* cfg,
                               const foe_comm* comm, void* stream, ipiano_slabs** out);
/* Re-initialises from new observations f (same layout as in create). */
foe_status ipiano_slabs_reset(ipiano_slabs* slabs, const float* f, double lipschitz_init, void* stream);
/* Runs max_iters accepted iterations (all ranks must call it; trial rounds in CUDA-graph
 * chunks, one host synchronisation per chunk).  FOE_ERR_COMM if slabs disagree. */
foe_status ipiano_slabs_solve(ipiano_slabs* slabs, void* stream);
/* Runs accepted iterations until min(target_iters, max_iters) are done (SURVEY.md 8(c) P2
 * teacher forcing steps a scene this way); ipiano_slabs_solve = advance to max_iters.  All
 * ranks must call it with the same target.  FOE_ERR_INVALID_ARGUMENT if target_iters < 0. */
foe_status ipiano_slabs_advance(ipiano_slabs* slabs, int target_iters, void* stream);
/* u = e^w (and/or w) of the slabs owned by this process: the whole scene when comm == NULL,
 * this rank's slab otherwise (device, [rows][W]). */
foe_status ipiano_slabs_get_iterate(const ipiano_slabs* slabs, double* w_out, float* u_out, void* stream);
/* Fused ghost-row exchange across processes (one GPU each, peer access over NVLink): K2 stores
 * its boundary rows straight into the neighbours' ghost buffers through CUDA IPC mappings,
 * replacing the ncclSend/ncclRecv step by a 1-element NCCL all-reduce that orders every rank's
 * K2 before any rank's K1.  Each rank exports its handle (64 bytes), the ranks exchange them
 * (e.g. torch.distributed.all_gather_object), and every rank connects its ring neighbours
 * (up = rank-1, down = rank+1 mod nranks; its own handle where a neighbour is itself).
 * In-process slabs (comm == NULL) always exchange this way (device pointers, no handles).
 * FOE_ERR_COMM if a mapping cannot be opened (no peer access): keep the NCCL path then. */
foe_status ipiano_slabs_halo_handle(const ipiano_slabs* slabs, void* handle_out);
foe_status ipiano_slabs_connect_peers(ipiano_slabs* slabs, const void* up_handle, const void* down_handle);
/* Back to the ncclSend/ncclRecv exchange (every rank must use the same path: when any rank
 * fails to connect, all disconnect).  Re-initialise (ipiano_slabs_reset) after either call. */
foe_status ipiano_slabs_disconnect_peers(ipiano_slabs* slabs);

/* The per-slab iPiano state j of this process (for ipiano_get_counters / ipiano_get_trace /
 * ipiano_profile / ipiano_profile_read; every slab holds the same control block and trace).
 * The returned state is owned by `slabs`: do not destroy it. */
foe_status ipiano_slabs_member(const ipiano_slabs* slabs, int j, ipiano_state** out);
void ipiano_slabs_destroy(ipiano_slabs* slabs);

/* ------------------------------------------------- evaluation and synthesis */

/* Pointers are device fp32 [B][H][W] arrays on the CURRENT CUDA device; results are host [B].
 * All three synchronise `stream`.
 *   foe_psnr: 10 log10(peak^2 / MSE) per image, +inf when x == ref.
 *   foe_ssim: mean local SSIM over the valid region with an 11x11 Gaussian window (sigma 1.5),
 *             K1 = 0.01, K2 = 0.03, C = (K peak)^2 (Wang et al., cited by the
 *             paper's Sec. III); H, W >= 11.
 *   foe_add_speckle: f = u sqrt(s), s ~ Gamma(looks[b], scale 1/looks[b]) (the amplitude model,
 *             DESIGN.md R-14), looks[b] >= 1; Marsaglia-Tsang driven by Philox4x32-10 with
 *             counter (p lo, p hi, attempt, 0) for the global pixel index p = b H W + y W + x
 *             and key (seed lo, seed hi): the result depends only on (u, looks, seed). */
foe_status foe_psnr(const float* x, const float* ref, int B, int H, int W, double peak, double* psnr_out,
                    void* stream);
foe_status foe_ssim(const float* x, const float* ref, int B, int H, int W, double peak, double* ssim_out,
                    void* stream);
foe_status foe_add_speckle(const float* u, int B, int H, int W, const double* looks, unsigned long long seed,
                           float* f_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FOE_H_ */
