/*
 * foe_oracle.c -- fp64 CPU oracle for the FoE/iPiano despeckling hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  The
 * product path (paper_1404_5344_b200/) never imports, links or executes it, and
 * this file shares no code, header, table or constant generator with the CUDA
 * path.
 *
 * It is a plain, slow, obviously-correct transcription of the paper, in the
 * paper's order and notation, in double precision:
 *
 *   PAPER.md:86-98  Eq.(2)  E_FoE(u) = sum_i theta_i sum_p rho((k_i * u)_p),
 *                           rho(x) = log(1 + x^2)
 *   PAPER.md:176-183        grad_w F = sum_i theta_i W K_i^T rho'(K_i e^w),
 *                           rho'(x) = 2x/(1+x^2), W = diag(e^w)
 *   PAPER.md:243-249 Eq.(10) combined data term
 *                           G(w) = (l1/2)<2w + f^2 e^{-2w},1> + (l2/2)<e^{2w} - 2 f^2 w,1>
 *   PAPER.md:185-192 Eq.(9)  prox of G solved by Newton's method
 *   PAPER.md:162-166        iPiano: w+ = (I + a dG)^{-1}(w - a grad F(w) + b (w - w-))
 *   PAPER.md:143-150, :194-204  variant model (6) in u: D = (lambda/2)<u^2 - 2f^2 log u,1>,
 *                           closed-form prox (FOE_DATA_IDIV on the GPU side)
 *   SPEC.md:287              backtracking on the descent-lemma inequality
 *
 * Readings where the paper is silent are listed in DESIGN.md (R-1 .. R-17) and
 * cited inline as [R-n].
 *
 * Numerics: every reduction is a fixed-order fp64 sum -- per-row partials (each
 * row summed left to right by one thread) then the rows summed in row order --
 * so results do not depend on the OpenMP thread count.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_ERR_ARG 1
#define ORC_ERR_NONFINITE 4
#define ORC_ERR_BACKTRACK 5
#define ORC_ERR_PROX 6
#define ORC_ERR_DOMAIN 7

/* -------------------------------------------------------------------------------- */
/* Periodic convolution and its adjoint (Eq.(2) "k_i * u"; reading R-2, R-3)          */
/* -------------------------------------------------------------------------------- */

static int wrapi(int i, int n) { i %= n; return i < 0 ? i + n : i; }

/* (k * u)[y,x] = sum_{a,b} k[a][b] u[(y - a + c) mod H][(x - b + c) mod W], c=(m-1)/2.
 * True convolution (kernel flipped), centred, periodic boundary [R-2, R-3]. */
void orc_conv(const double* u, int H, int W, const double* k, int m, double* out)
{
    const int c = (m - 1) / 2;
    int* ry = (int*)malloc(sizeof(int) * (size_t)m * H);
    int* cx = (int*)malloc(sizeof(int) * (size_t)m * W);
    for (int a = 0; a < m; ++a)
        for (int y = 0; y < H; ++y) ry[a * H + y] = wrapi(y - a + c, H);
    for (int b = 0; b < m; ++b)
        for (int x = 0; x < W; ++x) cx[b * W + x] = wrapi(x - b + c, W);
#pragma omp parallel for schedule(static)
    for (int y = 0; y < H; ++y) {
        for (int x = 0; x < W; ++x) {
            double s = 0.0;
            for (int a = 0; a < m; ++a) {
                const double* urow = u + (size_t)ry[a * H + y] * W;
                for (int b = 0; b < m; ++b) s += k[a * m + b] * urow[cx[b * W + x]];
            }
            out[(size_t)y * W + x] = s;
        }
    }
    free(ry);
    free(cx);
}

/* K^T v: the exact adjoint of orc_conv under <.,.>:
 * (K^T v)[y,x] = sum_{a,b} k[a][b] v[(y + a - c) mod H][(x + b - c) mod W]
 * (correlation with the same kernel). */
void orc_conv_adj(const double* v, int H, int W, const double* k, int m, double* out)
{
    const int c = (m - 1) / 2;
    int* ry = (int*)malloc(sizeof(int) * (size_t)m * H);
    int* cx = (int*)malloc(sizeof(int) * (size_t)m * W);
    for (int a = 0; a < m; ++a)
        for (int y = 0; y < H; ++y) ry[a * H + y] = wrapi(y + a - c, H);
    for (int b = 0; b < m; ++b)
        for (int x = 0; x < W; ++x) cx[b * W + x] = wrapi(x + b - c, W);
#pragma omp parallel for schedule(static)
    for (int y = 0; y < H; ++y) {
        for (int x = 0; x < W; ++x) {
            double s = 0.0;
            for (int a = 0; a < m; ++a) {
                const double* vrow = v + (size_t)ry[a * H + y] * W;
                for (int b = 0; b < m; ++b) s += k[a * m + b] * vrow[cx[b * W + x]];
            }
            out[(size_t)y * W + x] = s;
        }
    }
    free(ry);
    free(cx);
}

/* -------------------------------------------------------------------------------- */
/* Lorentzian potential                                            */
/* -------------------------------------------------------------------------------- */

double orc_rho(double x) { return log(1.0 + x * x); }          /* rho(x) = log(1+x^2)   */
double orc_rho_prime(double x) { return 2.0 * x / (1.0 + x * x); } /* rho'(x)=2x/(1+x^2) */
/* rho''(x) = 2(1 - x^2)/(1 + x^2)^2 (derivative of rho'; used by the Hessian-vector
 * product of the Lipschitz estimate [R-10]). */
double orc_rho_second(double x) { double d = 1.0 + x * x; return 2.0 * (1.0 - x * x) / (d * d); }

/* fixed-order sum of an [H][W] array: rows left-to-right, then rows top-to-bottom */
static double sum_rows(const double* a, int H, int W, double* rowbuf)
{
#pragma omp parallel for schedule(static)
    for (int y = 0; y < H; ++y) {
        double s = 0.0;
        for (int x = 0; x < W; ++x) s += a[(size_t)y * W + x];
        rowbuf[y] = s;
    }
    double t = 0.0;
    for (int y = 0; y < H; ++y) t += rowbuf[y];
    return t;
}

/* -------------------------------------------------------------------------------- */
/* FoE prior energy and gradient                                                       */
/* -------------------------------------------------------------------------------- */

/* u-domain: F = sum_i theta_i sum_p rho((k_i*u)_p);
 * grad_u F = sum_i theta_i K_i^T rho'(K_i u).  grad may be NULL. */
int orc_energy_grad_u(const double* u, int H, int W, const double* k, const double* theta,
                      int nf, int m, double* F_out, double* grad)
{
    const size_t N = (size_t)H * W;
    double* r = (double*)malloc(sizeof(double) * N);
    double* t = (double*)malloc(sizeof(double) * N);
    double* q = (double*)malloc(sizeof(double) * N);
    double* rowbuf = (double*)malloc(sizeof(double) * (size_t)H);
    if (grad) memset(grad, 0, sizeof(double) * N);
    double F = 0.0;
    for (int i = 0; i < nf; ++i) {
        const double* ki = k + (size_t)i * m * m;
        orc_conv(u, H, W, ki, m, r);                           /* r_i = k_i * u        */
        for (size_t p = 0; p < N; ++p) t[p] = orc_rho(r[p]);   /* rho(r_i)             */
        F += theta[i] * sum_rows(t, H, W, rowbuf);             /* theta_i sum_p rho    */
        if (grad) {
            for (size_t p = 0; p < N; ++p) t[p] = orc_rho_prime(r[p]);  /* rho'(K_i u) */
            orc_conv_adj(t, H, W, ki, m, q);                   /* K_i^T rho'(K_i u)    */
            for (size_t p = 0; p < N; ++p) grad[p] += theta[i] * q[p];
        }
    }
    *F_out = F;
    free(r); free(t); free(q); free(rowbuf);
    return ORC_OK;
}

/* w-domain: F(w) = E_FoE(e^w);
 * grad_w F = W * sum_i theta_i K_i^T rho'(K_i e^w), W = diag(e^w) applied after the
 * sum (chain rule, reading R-7).  grad may be NULL. */
int orc_energy_grad_w(const double* w, int H, int W, const double* k, const double* theta,
                      int nf, int m, double* F_out, double* grad)
{
    const size_t N = (size_t)H * W;
    double* u = (double*)malloc(sizeof(double) * N);
    for (size_t p = 0; p < N; ++p) u[p] = exp(w[p]);          /* u = e^w */
    int st = orc_energy_grad_u(u, H, W, k, theta, nf, m, F_out, grad);
    if (grad)
        for (size_t p = 0; p < N; ++p) grad[p] *= u[p];       /* W = diag(e^w) */
    free(u);
    return st;
}

/* Hessian-vector product of F(w) = E_FoE(e^w) [R-10]:
 *   d/de grad_w F(w + e v) |_{e=0}
 *     = v (.) grad_w F(w) + u (.) sum_i theta_i K_i^T [ rho''(K_i u) (.) K_i (u (.) v) ],  u = e^w.
 * (product rule on u (.) s(u) with du = u (.) v). */
int orc_hvp_w(const double* w, const double* v, int H, int W, const double* k,
              const double* theta, int nf, int m, double* hv)
{
    const size_t N = (size_t)H * W;
    double* u = (double*)malloc(sizeof(double) * N);
    double* uv = (double*)malloc(sizeof(double) * N);
    double* g = (double*)malloc(sizeof(double) * N);
    double* r = (double*)malloc(sizeof(double) * N);
    double* t = (double*)malloc(sizeof(double) * N);
    double* q = (double*)malloc(sizeof(double) * N);
    double F;
    for (size_t p = 0; p < N; ++p) { u[p] = exp(w[p]); uv[p] = u[p] * v[p]; }
    orc_energy_grad_w(w, H, W, k, theta, nf, m, &F, g);
    memset(hv, 0, sizeof(double) * N);
    for (int i = 0; i < nf; ++i) {
        const double* ki = k + (size_t)i * m * m;
        orc_conv(u, H, W, ki, m, r);                          /* K_i u          */
        orc_conv(uv, H, W, ki, m, t);                         /* K_i (u v)      */
        for (size_t p = 0; p < N; ++p) t[p] *= orc_rho_second(r[p]);
        orc_conv_adj(t, H, W, ki, m, q);
        for (size_t p = 0; p < N; ++p) hv[p] += theta[i] * q[p];
    }
    for (size_t p = 0; p < N; ++p) hv[p] = v[p] * g[p] + u[p] * hv[p];
    free(u); free(uv); free(g); free(r); free(t); free(q);
    return ORC_OK;
}

/* -------------------------------------------------------------------------------- */
/* Combined data term, Eq.(10)                                      */
/* -------------------------------------------------------------------------------- */

/* G(w) = sum_p (l1/2)(2 w_p + f_p^2 e^{-2w_p}) + (l2/2)(e^{2w_p} - 2 f_p^2 w_p)
 * (summed over pixels like (4) and (6), reading R-6); ft = max(f,1) [R-4]. */
double orc_data_energy(const double* w, const double* ft, int H, int W, double l1, double l2)
{
    const size_t N = (size_t)H * W;
    double* t = (double*)malloc(sizeof(double) * N);
    double* rowbuf = (double*)malloc(sizeof(double) * (size_t)H);
    for (size_t p = 0; p < N; ++p) {
        const double f2 = ft[p] * ft[p];
        t[p] = 0.5 * l1 * (2.0 * w[p] + f2 * exp(-2.0 * w[p]))
             + 0.5 * l2 * (exp(2.0 * w[p]) - 2.0 * f2 * w[p]);
    }
    double G = sum_rows(t, H, W, rowbuf);
    free(t); free(rowbuf);
    return G;
}

/* Prox of tau*G at what, one pixel (Eq.(9) generalised to Eq.(10), PAPER.md:185-192,
 * :248-249): the unique root z of
 *     phi(z) = z - what + tau [ l1 (1 - f^2 e^{-2z}) + l2 (e^{2z} - f^2) ],
 * phi'(z) = 1 + tau [ 2 l1 f^2 e^{-2z} + 2 l2 e^{2z} ] > 0.
 * Newton from z = what, safeguarded by bisection on the bracket
 * [min(what, log f) - 1, max(what, log f) + 1], stopping at |phi| <= tol
 * or when a further step cannot change z in fp64.  Returns the number
 * of Newton updates, or -1 if the cap is exceeded. */
int orc_prox_pixel(double what, double ft, double tau, double l1, double l2, double tol,
                   int cap, double* z_out, double* resid_out)
{
    const double lf = log(ft), f2 = ft * ft;
    double lo = fmin(what, lf) - 1.0, hi = fmax(what, lf) + 1.0;
    double z = what;
    for (int it = 0; it <= cap; ++it) {
        const double em = exp(-2.0 * z), ep = exp(2.0 * z);
        const double phi = z - what + tau * (l1 * (1.0 - f2 * em) + l2 * (ep - f2));
        if (fabs(phi) <= tol) { *z_out = z; *resid_out = fabs(phi); return it; }
        if (phi > 0.0) hi = z; else lo = z;
        const double dphi = 1.0 + tau * (2.0 * l1 * f2 * em + 2.0 * l2 * ep);
        double zn = z - phi / dphi;
        if (!(zn > lo && zn < hi)) zn = 0.5 * (lo + hi);      /* bisection safeguard */
        if (zn == z) { *z_out = z; *resid_out = fabs(phi); return it; }
        z = zn;
    }
    *z_out = z;
    *resid_out = INFINITY;
    return -1;
}

/* Prox over an image; returns max Newton iterations, or -1 (first failing pixel in
 * *bad_pixel). */
int orc_prox(const double* what, const double* ft, size_t N, double tau, double l1, double l2,
             double tol, int cap, double* out, double* max_resid, long long* bad_pixel)
{
    int maxit = 0;
    double mres = 0.0;
    long long bad = -1;
    for (size_t p = 0; p < N; ++p) {
        double res;
        int it = orc_prox_pixel(what[p], ft[p], tau, l1, l2, tol, cap, &out[p], &res);
        if (it < 0) { if (bad < 0) bad = (long long)p; continue; }
        if (it > maxit) maxit = it;
        if (res > mres) mres = res;
    }
    if (max_resid) *max_resid = mres;
    if (bad_pixel) *bad_pixel = bad;
    return bad >= 0 ? -1 : maxit;
}

/* -------------------------------------------------------------------------------- */
/* iPiano with backtracking -- algorithm C-0         */
/* -------------------------------------------------------------------------------- */

typedef struct {
    double beta;             /* inertia b, 0 <= b < 1                                 */
    double step_safety;      /* a = safety * 2(1-b)/L_n                 */
    double lipschitz_init;   /* L_0 > 0 [R-10]                                        */
    double backtrack_factor; /* eta > 1: L <- eta L on a failed test    */
    double shrink;           /* L <- shrink L after an accepted step [R-9]            */
    int max_iters;           /* accepted iterations [R-12]                            */
    int max_backtracks;      /* 60                                      */
    int newton_max_iters;    /* 30                                      */
    double newton_tol;       /* 1e-12                                   */
    double rel_change_tol;   /* 0 = run exactly max_iters (R-12)         */
    double w_guard;          /* |w| bound on accepted iterates, 40 [R-11]             */
} orc_cfg;

/* trace record per accepted iteration (row 0 = the initial point) */
enum { TR_F = 0, TR_G, TR_H, TR_L, TR_TRIALS, TR_MARGIN, TR_NEWTON, TR_RELCHG, TR_FIELDS };

/* One iPiano trial from (w, w_prev, g = grad F(w), F = F(w)) at Lipschitz estimate L:
 *   a = safety 2(1-b)/L;  what = w - a g + b (w - w_prev);  w+ = prox_{aG}(what);
 *   test F(w+) <= F(w) + <g, w+ - w> + (L/2)||w+ - w||^2.
 * Outputs (any may be NULL except wplus): what, wplus, gplus = grad F(w+), and
 * out[8] = {F+, <g,D>, ||D||^2, G(w+), margin, accepted, newton_max, ||w||^2}.
 * Returns ORC_OK, or ORC_ERR_PROX if the Newton cap was exceeded. */
int orc_ipiano_trial(const double* w, const double* wprev, const double* g, double F, double L,
                     const double* ft, int H, int W, const double* k, const double* theta,
                     int nf, int m, double l1, double l2, const orc_cfg* cfg,
                     double* what_out, double* wplus, double* gplus, double* out)
{
    const size_t N = (size_t)H * W;
    const double alpha = cfg->step_safety * 2.0 * (1.0 - cfg->beta) / L;
    double* what = what_out ? what_out : (double*)malloc(sizeof(double) * N);
    double* t = (double*)malloc(sizeof(double) * N);
    double* rowbuf = (double*)malloc(sizeof(double) * (size_t)H);
    for (size_t p = 0; p < N; ++p)
        what[p] = w[p] - alpha * g[p] + cfg->beta * (w[p] - wprev[p]);
    long long bad;
    int nit = orc_prox(what, ft, N, alpha, l1, l2, cfg->newton_tol, cfg->newton_max_iters,
                       wplus, NULL, &bad);
    int st = nit < 0 ? ORC_ERR_PROX : ORC_OK;
    double Fp = NAN;
    orc_energy_grad_w(wplus, H, W, k, theta, nf, m, &Fp, gplus);
    for (size_t p = 0; p < N; ++p) t[p] = g[p] * (wplus[p] - w[p]);
    const double gd = sum_rows(t, H, W, rowbuf);
    for (size_t p = 0; p < N; ++p) t[p] = (wplus[p] - w[p]) * (wplus[p] - w[p]);
    const double dd = sum_rows(t, H, W, rowbuf);
    for (size_t p = 0; p < N; ++p) t[p] = w[p] * w[p];
    const double ww = sum_rows(t, H, W, rowbuf);
    const double Gp = orc_data_energy(wplus, ft, H, W, l1, l2);
    const double margin = F + gd + 0.5 * L * dd - Fp;
    /* a non-finite trial counts as a failed test [R-11] */
    const int ok = isfinite(Fp) && isfinite(gd) && isfinite(dd) && isfinite(Gp) && margin >= 0.0;
    if (out) {
        out[0] = Fp; out[1] = gd; out[2] = dd; out[3] = Gp; out[4] = margin;
        out[5] = ok ? 1.0 : 0.0; out[6] = (double)nit; out[7] = ww;
    }
    if (!what_out) free(what);
    free(t); free(rowbuf);
    return st;
}

/* Full run of algorithm C-0 on one image.  f is the fp32 observation; ft = max(f,1)
 * [R-4]; w^0 = log ft; w^{-1} = w^0 [R-8]; L = L_init.  Writes the final w and the
 * trace [(max_iters+1)][TR_FIELDS].  Returns ORC_OK or an error code; *iters_run /
 * *total_trials report progress either way. */
int orc_ipiano_run(const float* f, int H, int W, const double* k, const double* theta,
                   int nf, int m, double l1, double l2, const orc_cfg* cfg,
                   double* w_out, double* trace, int* iters_run, int* total_trials)
{
    const size_t N = (size_t)H * W;
    double* ft = (double*)malloc(sizeof(double) * N);
    double* w = (double*)malloc(sizeof(double) * N);
    double* wp = (double*)malloc(sizeof(double) * N);
    double* wn = (double*)malloc(sizeof(double) * N);
    double* g = (double*)malloc(sizeof(double) * N);
    double* gn = (double*)malloc(sizeof(double) * N);
    int st = ORC_OK, n = 0, trials_total = 0;
    for (size_t p = 0; p < N; ++p) {
        ft[p] = fmax((double)f[p], 1.0);                  /* f~ = max(f,1)   [R-4] */
        w[p] = log(ft[p]);                                /* w^0 = log f~          */
        wp[p] = w[p];                                     /* w^{-1} = w^0    [R-8] */
    }
    double F;
    orc_energy_grad_w(w, H, W, k, theta, nf, m, &F, g);
    double L = cfg->lipschitz_init;
    if (trace) {
        double* r0 = trace;
        r0[TR_F] = F; r0[TR_G] = orc_data_energy(w, ft, H, W, l1, l2); r0[TR_H] = F + r0[TR_G];
        r0[TR_L] = L; r0[TR_TRIALS] = 0; r0[TR_MARGIN] = 0; r0[TR_NEWTON] = 0; r0[TR_RELCHG] = 0;
    }
    if (!isfinite(F)) st = ORC_ERR_NONFINITE;
    while (st == ORC_OK && n < cfg->max_iters) {
        int trials = 0;
        double out[8];
        for (;;) {
            ++trials; ++trials_total;
            int ts = orc_ipiano_trial(w, wp, g, F, L, ft, H, W, k, theta, nf, m, l1, l2, cfg,
                                      NULL, wn, gn, out);
            if (ts != ORC_OK) { st = ts; break; }
            if (out[5] != 0.0) break;
            if (trials > cfg->max_backtracks) { st = ORC_ERR_BACKTRACK; break; }
            L *= cfg->backtrack_factor;                   /* double L_n */
        }
        if (st != ORC_OK) break;
        double wmax = 0.0;
        for (size_t p = 0; p < N; ++p) wmax = fmax(wmax, fabs(wn[p]));
        if (!(wmax <= cfg->w_guard)) { st = isfinite(wmax) ? ORC_ERR_DOMAIN : ORC_ERR_NONFINITE; }
        /* accept: w- <- w, w <- w+, g <- grad F(w+), F <- F+ */
        double* tmp = wp; wp = w; w = wn; wn = tmp;
        tmp = g; g = gn; gn = tmp;
        F = out[0];
        ++n;
        const double relchg = sqrt(out[2]) / fmax(sqrt(out[7]), 1.0);
        if (trace) {
            double* r = trace + (size_t)n * TR_FIELDS;
            r[TR_F] = F; r[TR_G] = out[3]; r[TR_H] = F + out[3]; r[TR_L] = L;
            r[TR_TRIALS] = trials; r[TR_MARGIN] = out[4]; r[TR_NEWTON] = out[6];
            r[TR_RELCHG] = relchg;
        }
        L *= cfg->shrink;                                 /* [R-9] */
        if (cfg->rel_change_tol > 0.0 && relchg < cfg->rel_change_tol) break;
    }
    memcpy(w_out, w, sizeof(double) * N);
    if (iters_run) *iters_run = n;
    if (total_trials) *total_trials = trials_total;
    free(ft); free(w); free(wp); free(wn); free(g); free(gn);
    return st;
}


/* Lipschitz estimate [R-10]: |Rayleigh quotient| after `iters` power-iteration steps
 * on the prior Hessian at w^0 = log max(f,1), from the start vector v0 (an input):
 *   v <- v0/||v0||;  repeat: h = Hess v; rq = <v,h>; v <- h/||h||.
 * Returns rho_hat; *L_pow2 = 2^ceil(log2 rho_hat). */
double orc_estimate_lipschitz(const float* f, int H, int W, const double* k, const double* theta,
                              int nf, int m, const double* v0, int iters, double* L_pow2)
{
    const size_t N = (size_t)H * W;
    double* w = (double*)malloc(sizeof(double) * N);
    double* v = (double*)malloc(sizeof(double) * N);
    double* h = (double*)malloc(sizeof(double) * N);
    double* t = (double*)malloc(sizeof(double) * N);
    double* rowbuf = (double*)malloc(sizeof(double) * (size_t)H);
    for (size_t p = 0; p < N; ++p) w[p] = log(fmax((double)f[p], 1.0));
    for (size_t p = 0; p < N; ++p) t[p] = v0[p] * v0[p];
    double nv = sqrt(sum_rows(t, H, W, rowbuf));
    for (size_t p = 0; p < N; ++p) v[p] = v0[p] / nv;
    double rq = 0.0;
    for (int it = 0; it < iters; ++it) {
        orc_hvp_w(w, v, H, W, k, theta, nf, m, h);
        for (size_t p = 0; p < N; ++p) t[p] = v[p] * h[p];
        rq = sum_rows(t, H, W, rowbuf);
        for (size_t p = 0; p < N; ++p) t[p] = h[p] * h[p];
        const double nh = sqrt(sum_rows(t, H, W, rowbuf));
        for (size_t p = 0; p < N; ++p) v[p] = h[p] / nh;
    }
    const double rho = fabs(rq);
    if (L_pow2) *L_pow2 = ldexp(1.0, (int)ceil(log2(rho)));
    free(w); free(v); free(h); free(t); free(rowbuf);
    return rho;
}

/* -------------------------------------------------------------------------------- */
/* Variant model (6) in u: I-divergence data term         */
/* -------------------------------------------------------------------------------- */

/* D(u,f) = (lambda/2) <u^2 - 2 f^2 log u, 1> (Eq.(5)); u > 0 (else NaN). */
double orc_idiv_energy(const double* u, const double* ft, int H, int W, double lam)
{
    const size_t N = (size_t)H * W;
    double* t = (double*)malloc(sizeof(double) * N);
    double* rowbuf = (double*)malloc(sizeof(double) * (size_t)H);
    for (size_t p = 0; p < N; ++p)
        t[p] = u[p] > 0.0 ? 0.5 * lam * (u[p] * u[p] - 2.0 * ft[p] * ft[p] * log(u[p])) : NAN;
    const double e = sum_rows(t, H, W, rowbuf);
    free(t); free(rowbuf);
    return e;
}

/* (I + tau dG)^{-1}(uhat), pointwise closed form:
 *   u_p = (uhat_p + sqrt(uhat_p^2 + 4 (1 + tau lam) tau lam f_p^2)) / (2 (1 + tau lam)). */
double orc_idiv_prox_pixel(double uhat, double ft, double tau, double lam)
{
    const double tl = tau * lam;
    return (uhat + sqrt(uhat * uhat + 4.0 * (1.0 + tl) * tl * ft * ft)) / (2.0 * (1.0 + tl));
}

/* Hessian-vector product of F(u) = E_FoE(u): sum_i theta_i K_i^T [rho''(K_i u) (.) K_i v] */
int orc_hvp_u(const double* u, const double* v, int H, int W, const double* k,
              const double* theta, int nf, int m, double* hv)
{
    const size_t N = (size_t)H * W;
    double* r = (double*)malloc(sizeof(double) * N);
    double* t = (double*)malloc(sizeof(double) * N);
    double* q = (double*)malloc(sizeof(double) * N);
    memset(hv, 0, sizeof(double) * N);
    for (int i = 0; i < nf; ++i) {
        const double* ki = k + (size_t)i * m * m;
        orc_conv(u, H, W, ki, m, r);                          /* K_i u  */
        orc_conv(v, H, W, ki, m, t);                          /* K_i v  */
        for (size_t p = 0; p < N; ++p) t[p] *= orc_rho_second(r[p]);
        orc_conv_adj(t, H, W, ki, m, q);
        for (size_t p = 0; p < N; ++p) hv[p] += theta[i] * q[p];
    }
    free(r); free(t); free(q);
    return ORC_OK;
}

/* One iPiano trial of model (6) in u, as orc_ipiano_trial
 * with grad_u F, the closed-form prox and D of Eq.(5).  out[8] as orc_ipiano_trial
 * (out[6] = 0: no Newton). */
int orc_ipiano_trial_u(const double* u, const double* uprev, const double* g, double F, double L,
                       const double* ft, int H, int W, const double* k, const double* theta,
                       int nf, int m, double lam, const orc_cfg* cfg,
                       double* uhat_out, double* uplus, double* gplus, double* out)
{
    const size_t N = (size_t)H * W;
    const double alpha = cfg->step_safety * 2.0 * (1.0 - cfg->beta) / L;
    double* uhat = uhat_out ? uhat_out : (double*)malloc(sizeof(double) * N);
    double* t = (double*)malloc(sizeof(double) * N);
    double* rowbuf = (double*)malloc(sizeof(double) * (size_t)H);
    for (size_t p = 0; p < N; ++p) {
        uhat[p] = u[p] - alpha * g[p] + cfg->beta * (u[p] - uprev[p]);
        uplus[p] = orc_idiv_prox_pixel(uhat[p], ft[p], alpha, lam);
    }
    double Fp = NAN;
    orc_energy_grad_u(uplus, H, W, k, theta, nf, m, &Fp, gplus);
    for (size_t p = 0; p < N; ++p) t[p] = g[p] * (uplus[p] - u[p]);
    const double gd = sum_rows(t, H, W, rowbuf);
    for (size_t p = 0; p < N; ++p) t[p] = (uplus[p] - u[p]) * (uplus[p] - u[p]);
    const double dd = sum_rows(t, H, W, rowbuf);
    for (size_t p = 0; p < N; ++p) t[p] = u[p] * u[p];
    const double uu = sum_rows(t, H, W, rowbuf);
    const double Gp = orc_idiv_energy(uplus, ft, H, W, lam);
    const double margin = F + gd + 0.5 * L * dd - Fp;
    const int ok = isfinite(Fp) && isfinite(gd) && isfinite(dd) && isfinite(Gp) && margin >= 0.0;
    if (out) {
        out[0] = Fp; out[1] = gd; out[2] = dd; out[3] = Gp; out[4] = margin;
        out[5] = ok ? 1.0 : 0.0; out[6] = 0.0; out[7] = uu;
    }
    if (!uhat_out) free(uhat);
    free(t); free(rowbuf);
    return ORC_OK;
}

/* Full run of model (6): u^0 = f~, u^{-1} = u^0 [R-8], L = L_init; the
 * same backtracking, acceptance, trace and stopping rules as orc_ipiano_run.  The
 * guard [R-11] becomes: an accepted iterate must be finite and positive. */
int orc_ipiano_run_u(const float* f, int H, int W, const double* k, const double* theta,
                     int nf, int m, double lam, const orc_cfg* cfg,
                     double* u_out, double* trace, int* iters_run, int* total_trials)
{
    const size_t N = (size_t)H * W;
    double* ft = (double*)malloc(sizeof(double) * N);
    double* u = (double*)malloc(sizeof(double) * N);
    double* up = (double*)malloc(sizeof(double) * N);
    double* un = (double*)malloc(sizeof(double) * N);
    double* g = (double*)malloc(sizeof(double) * N);
    double* gn = (double*)malloc(sizeof(double) * N);
    int st = ORC_OK, n = 0, trials_total = 0;
    for (size_t p = 0; p < N; ++p) {
        ft[p] = fmax((double)f[p], 1.0);                  /* f~ = max(f,1)   [R-4] */
        u[p] = ft[p];                                     /* u^0 = f~ */
        up[p] = u[p];                                     /* u^{-1} = u^0    [R-8] */
    }
    double F;
    orc_energy_grad_u(u, H, W, k, theta, nf, m, &F, g);
    double L = cfg->lipschitz_init;
    if (trace) {
        double* r0 = trace;
        r0[TR_F] = F; r0[TR_G] = orc_idiv_energy(u, ft, H, W, lam); r0[TR_H] = F + r0[TR_G];
        r0[TR_L] = L; r0[TR_TRIALS] = 0; r0[TR_MARGIN] = 0; r0[TR_NEWTON] = 0; r0[TR_RELCHG] = 0;
    }
    if (!isfinite(F)) st = ORC_ERR_NONFINITE;
    while (st == ORC_OK && n < cfg->max_iters) {
        int trials = 0;
        double out[8];
        for (;;) {
            ++trials; ++trials_total;
            orc_ipiano_trial_u(u, up, g, F, L, ft, H, W, k, theta, nf, m, lam, cfg, NULL, un, gn, out);
            if (out[5] != 0.0) break;
            if (trials > cfg->max_backtracks) { st = ORC_ERR_BACKTRACK; break; }
            L *= cfg->backtrack_factor;                   /* double L_n */
        }
        if (st != ORC_OK) break;
        for (size_t p = 0; p < N; ++p)
            if (!(un[p] > 0.0) || !isfinite(un[p])) { st = isfinite(un[p]) ? ORC_ERR_DOMAIN : ORC_ERR_NONFINITE; break; }
        double* tmp = up; up = u; u = un; un = tmp;
        tmp = g; g = gn; gn = tmp;
        F = out[0];
        ++n;
        const double relchg = sqrt(out[2]) / fmax(sqrt(out[7]), 1.0);
        if (trace) {
            double* r = trace + (size_t)n * TR_FIELDS;
            r[TR_F] = F; r[TR_G] = out[3]; r[TR_H] = F + out[3]; r[TR_L] = L;
            r[TR_TRIALS] = trials; r[TR_MARGIN] = out[4]; r[TR_NEWTON] = 0;
            r[TR_RELCHG] = relchg;
        }
        L *= cfg->shrink;                                 /* [R-9] */
        if (cfg->rel_change_tol > 0.0 && relchg < cfg->rel_change_tol) break;
    }
    memcpy(u_out, u, sizeof(double) * N);
    if (iters_run) *iters_run = n;
    if (total_trials) *total_trials = trials_total;
    free(ft); free(u); free(up); free(un); free(g); free(gn);
    return st;
}

/* Lipschitz estimate of model (6) [R-10 applied in u]: power iteration on the Hessian of
 * F(u) at u^0 = f~. */
double orc_estimate_lipschitz_u(const float* f, int H, int W, const double* k, const double* theta,
                                int nf, int m, const double* v0, int iters, double* L_pow2)
{
    const size_t N = (size_t)H * W;
    double* u = (double*)malloc(sizeof(double) * N);
    double* v = (double*)malloc(sizeof(double) * N);
    double* h = (double*)malloc(sizeof(double) * N);
    double* t = (double*)malloc(sizeof(double) * N);
    double* rowbuf = (double*)malloc(sizeof(double) * (size_t)H);
    for (size_t p = 0; p < N; ++p) u[p] = fmax((double)f[p], 1.0);
    for (size_t p = 0; p < N; ++p) t[p] = v0[p] * v0[p];
    double nv = sqrt(sum_rows(t, H, W, rowbuf));
    for (size_t p = 0; p < N; ++p) v[p] = v0[p] / nv;
    double rq = 0.0;
    for (int it = 0; it < iters; ++it) {
        orc_hvp_u(u, v, H, W, k, theta, nf, m, h);
        for (size_t p = 0; p < N; ++p) t[p] = v[p] * h[p];
        rq = sum_rows(t, H, W, rowbuf);
        for (size_t p = 0; p < N; ++p) t[p] = h[p] * h[p];
        const double nh = sqrt(sum_rows(t, H, W, rowbuf));
        for (size_t p = 0; p < N; ++p) v[p] = h[p] / nh;
    }
    const double rho = fabs(rq);
    if (L_pow2) *L_pow2 = ldexp(1.0, (int)ceil(log2(rho)));
    free(u); free(v); free(h); free(t); free(rowbuf);
    return rho;
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
