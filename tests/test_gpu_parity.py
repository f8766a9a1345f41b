"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Tolerances (BASELINE.json north_star): single-step gradient and update relative L2
<= 1e-5; final image after the full iteration count relative L2 <= 1e-4 and PSNR
against the clean image within 0.01 dB.  Energies are compared at 1e-6 relative
(fp32 stencil, fp64 accumulation -- DESIGN.md "Precision").
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import foe_synth as S  # noqa: E402
import oracle  # noqa: E402
import paper_1404_5344_b200 as P  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _require_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    P.lib()  # loud failure if libfoe.so cannot be loaded


def rel_l2(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _model(filters, theta, lam=(310.0, 0.008)):
    return P.foe_model_create(filters, theta, lam=lam)


def _cuda(a, dtype):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


# ------------------------------------------------------------------ energy + gradient

@pytest.mark.parametrize("m,nf,B,H,W", [
    (7, 48, 1, 64, 64),     # exactly one tile
    (7, 48, 2, 100, 77),    # ragged tails in both axes, 2 images
    (7, 12, 1, 12, 12),     # image smaller than a tile (multiple wraps), partial filter chunk
    (5, 24, 1, 130, 129),   # c1 filter size, 3x3 tiles with 2/1-pixel tails
    (3, 8, 3, 70, 65),      # m = 3
    (7, 48, 1, 256, 256),   # c2 geometry (split-N_f filter groups)
])
def test_energy_grad_parity(m, nf, B, H, W):
    k, th = S.random_filter_bank(nf, m, 1000 + m + nf)
    rng = np.random.default_rng(H * W + B)
    f = np.stack([S.add_speckle(S.piecewise_smooth_scene(H, W, 10 + b), 3, 20 + b) for b in range(B)])
    w = np.log(np.maximum(f.astype(np.float64), 1.0)) + 0.01 * rng.standard_normal(f.shape)
    md = _model(k, th)
    Fg, Gg, g = P.foe_energy_grad(md, _cuda(w, torch.float64), f=_cuda(f, torch.float32), data=True,
                                  lam_per_image=np.tile([310.0, 0.008], B))
    g = g.cpu().numpy()
    ft = oracle.ftilde(f)
    for b in range(B):
        Fo, go = oracle.energy_grad_w(w[b], k, th)
        assert rel_l2(g[b], go) <= 1e-5, (b, rel_l2(g[b], go))
        assert Fg[b] == pytest.approx(Fo, rel=1e-6)
        assert Gg[b] == pytest.approx(oracle.data_energy(w[b], ft[b], 310.0, 0.008), rel=1e-12)


def test_energy_grad_constant_image_and_zero_mean():
    # zero prior gradient on a constant image for zero-mean filters (BASELINE north_star pin,
    # here through the CUDA path): |g| at fp32 rounding level of c * sum(k)
    k, th = S.random_filter_bank(48, 7, 5)
    w = np.full((1, 96, 80), math.log(120.0))
    md = _model(k, th)
    F, _, g = P.foe_energy_grad(md, _cuda(w, torch.float64))
    assert np.abs(g.cpu().numpy()).max() < 1e-4
    assert F[0] < 1e-6


def test_hvp_parity():
    k, th = S.random_filter_bank(24, 7, 6)
    f = S.add_speckle(S.piecewise_smooth_scene(70, 90, 3), 1, 4)[None]
    w = np.log(np.maximum(f.astype(np.float64), 1.0))
    v = np.random.default_rng(0).standard_normal(w.shape)
    md = _model(k, th)
    hv = P.foe_hvp(md, _cuda(w, torch.float64), _cuda(v, torch.float64)).cpu().numpy()
    ho = oracle.hvp_w(w[0], v[0], k, th)
    # setup-only quantity (Lipschitz initialisation, R-10): only the power of two of the
    # Rayleigh quotient is used, so 1e-4 suffices; rho''(r) = 2(1-r^2)/(1+r^2)^2 cancels
    # near |r| = 1 in fp32, which is why it is looser than the gradient's 1e-5
    assert rel_l2(hv[0], ho) <= 1e-4


def test_lipschitz_estimate_same_power_of_two():
    cfg = S.config("c1")
    d = S.make_inputs(cfg)
    v0 = S.lipschitz_start_vector(1, cfg.H, cfg.W)
    md = _model(d["filters"], d["theta"])
    rho, L = P.foe_estimate_lipschitz(md, _cuda(d["f"], torch.float32), _cuda(v0, torch.float64), 25)
    rho_o, L_o = oracle.estimate_lipschitz(d["f"][0], d["filters"], d["theta"], v0[0], 25)
    assert rho[0] == pytest.approx(rho_o, rel=1e-4)
    assert L[0] == L_o


def test_lipschitz_estimate_stored_S_batch_ragged():
    """The 48 x 7x7 bank on two ragged images (150 x 260: halo responses read across the wrap from
    the neighbour tiles' stored S_i = rho''(K_i u)/2, k_hvp_s): rho to 1e-4 and the same power of two
    as the oracle for each image (R-10)."""
    cfg = S.config("c4", B=2, H=150, W=260)
    d = S.make_inputs(cfg)
    v0 = S.lipschitz_start_vector(2, cfg.H, cfg.W)
    md = _model(d["filters"], d["theta"])
    rho, L = P.foe_estimate_lipschitz(md, _cuda(d["f"], torch.float32), _cuda(v0, torch.float64), 25)
    for b in range(2):
        rho_o, L_o = oracle.estimate_lipschitz(d["f"][b], d["filters"], d["theta"], v0[b], 25)
        assert rho[b] == pytest.approx(rho_o, rel=1e-4), (b, rho[b], rho_o)
        assert L[b] == L_o


# ---------------------------------------------------------------------- iPiano steps

def _setup(name, **over):
    cfg = S.config(name, **over)
    d = S.make_inputs(cfg)
    v0 = S.lipschitz_start_vector(cfg.B, cfg.H, cfg.W)
    L0 = np.array([oracle.estimate_lipschitz(d["f"][b], d["filters"], d["theta"], v0[b])[1]
                   for b in range(cfg.B)])
    return cfg, d, L0


def test_single_step_parity_P1():
    # P1: from identical (w, w_prev = w, L) the first iPiano trial (gradient, w+, test) agrees
    cfg, d, L0 = _setup("c2", H=96, W=80, iters=3)
    md = _model(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]))
    st = P.ipiano_state_create(md, _cuda(d["f"], torch.float32), d["lambdas"], L0,
                               P.ipiano_config_default(max_iters=3))
    it = P.ipiano_step(st)
    assert it[0] == 1
    w_gpu, _ = P.ipiano_get_iterate(st, want_u=False)
    tr = P.ipiano_get_trace(st)[0]
    f = d["f"][0]
    w0 = np.log(oracle.ftilde(f))
    F0, g0 = oracle.energy_grad_w(w0, d["filters"], d["theta"])
    l1, l2 = d["lambdas"][0]
    r = oracle.ipiano_trial(w0, w0, g0, F0, L0[0], f, d["filters"], d["theta"], l1, l2,
                            oracle.make_cfg(L0[0], 3))
    assert r["accepted"] and tr[1, 4] == 1
    wg = w_gpu.cpu().numpy()[0]
    assert rel_l2(wg - w0, r["wplus"] - w0) <= 1e-5          # the update w+ - w
    assert tr[0, 0] == pytest.approx(F0, rel=1e-6)
    assert tr[1, 0] == pytest.approx(r["Fplus"], rel=1e-6)
    assert tr[1, 1] == pytest.approx(r["Gplus"], rel=1e-9)
    assert tr[1, 5] == pytest.approx(r["margin"], rel=1e-2, abs=1e-6 * abs(F0))
    # gradient at the candidate, through foe_energy_grad on the GPU iterate
    _, _, g1 = P.foe_energy_grad(md, w_gpu)
    _, go1 = oracle.energy_grad_w(wg, d["filters"], d["theta"])
    assert rel_l2(g1.cpu().numpy()[0], go1) <= 1e-5


@pytest.mark.parametrize("policy", ["recommended", "spec"])
@pytest.mark.parametrize("stencil", [P.FOE_STENCIL_FFMA, P.FOE_STENCIL_TENSOR])
def test_teacher_forced_trajectory_P2(policy, stencil):
    # P2: every GPU step is re-done by the oracle from the GPU's own state (w, w_prev, L):
    # per-step update parity <= 1e-5 and identical decisions unless |margin| is a near-tie.
    # Under the SPEC policy (beta = 0.8, L halves after each accept; SURVEY
    # 8(f) f3) this is the certificate: the long run is chaotic under rounding (R-9).
    cfg, d, L0 = _setup("c2", H=128, W=96, iters=12)
    md = _model(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]))
    pol = dict(beta=0.8, shrink=0.5) if policy == "spec" else {}
    st = P.ipiano_state_create(md, _cuda(d["f"], torch.float32), d["lambdas"], L0,
                               P.ipiano_config_default(max_iters=12, stencil=stencil, **pol))
    f = d["f"][0]
    l1, l2 = d["lambdas"][0]
    w_prev = np.log(oracle.ftilde(f))
    w_cur = w_prev.copy()
    for n in range(12):
        Lg = P.ipiano_get_counters(st)["L"][0]
        P.ipiano_step(st)
        wg, _ = P.ipiano_get_iterate(st, want_u=False)
        wg = wg.cpu().numpy()[0]
        tr = P.ipiano_get_trace(st)[0]
        F, g = oracle.energy_grad_w(w_cur, d["filters"], d["theta"])
        L = Lg
        trials = 0
        while True:
            trials += 1
            r = oracle.ipiano_trial(w_cur, w_prev, g, F, L, f, d["filters"], d["theta"], l1, l2,
                                    oracle.make_cfg(L, 1, **pol))
            if r["accepted"]:
                break
            L *= 2
        assert trials == tr[n + 1, 4] or abs(r["margin"]) < 1e-6 * abs(F)
        assert rel_l2(wg - w_cur, r["wplus"] - w_cur) <= 1e-5, n
        w_prev, w_cur = w_cur, wg


def _free_run(cfg, d, L0, groups=0):
    md = _model(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]))
    c = P.ipiano_config_default(max_iters=cfg.iters, filter_groups=groups)
    st = P.ipiano_state_create(md, _cuda(d["f"], torch.float32), d["lambdas"], L0, c)
    P.ipiano_solve(st)
    w, u = P.ipiano_get_iterate(st)
    return w.cpu().numpy(), u.cpu().numpy(), P.ipiano_get_trace(st), P.ipiano_get_counters(st)


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_free_running_full_config_P3(name):
    # P3 on the full BASELINE configs 1 and 2 (128^2 x 100 it; 256^2 x 200 it)
    cfg, d, L0 = _setup(name)
    w, u, tr, cnt = _free_run(cfg, d, L0)
    assert cnt["status"][0] == 0 and cnt["iters"][0] == cfg.iters
    l1, l2 = d["lambdas"][0]
    ref = oracle.ipiano_run(d["f"][0], d["filters"], d["theta"], l1, l2, oracle.make_cfg(L0[0], cfg.iters))
    assert ref["status"] == 0
    assert rel_l2(u[0], ref["u"]) <= 1e-4
    clean = d["clean"][0]
    assert abs(oracle.psnr(u[0], clean) - oracle.psnr(ref["u"], clean)) <= 0.01
    np.testing.assert_array_equal(tr[0, 1:, 3], ref["trace"][1:, 3])   # same L_n decisions
    np.testing.assert_array_equal(tr[0, 1:, 4], ref["trace"][1:, 4])   # same trial counts
    np.testing.assert_allclose(tr[0, :, 2], ref["trace"][:, 2], rtol=1e-6)  # H trace


def test_batch_invariance_and_determinism():
    cfg, d, L0 = _setup("c4", B=3, H=128, W=128, iters=6)
    md = _model(d["filters"], d["theta"])
    c = P.ipiano_config_default(max_iters=6, filter_groups=2)
    runs = []
    for _ in range(2):
        st = P.ipiano_state_create(md, _cuda(d["f"], torch.float32), d["lambdas"], L0, c)
        P.ipiano_solve(st)
        runs.append((P.ipiano_get_iterate(st)[0].cpu().numpy(), P.ipiano_get_trace(st)))
    np.testing.assert_array_equal(runs[0][0], runs[1][0])
    np.testing.assert_array_equal(runs[0][1], runs[1][1])
    st = P.ipiano_state_create(md, _cuda(d["f"][1:2], torch.float32), d["lambdas"][1:2], L0[1:2], c)
    P.ipiano_solve(st)
    np.testing.assert_array_equal(P.ipiano_get_iterate(st)[0].cpu().numpy()[0], runs[0][0][1])


def test_ipiano_run_host_and_device_agree():
    cfg, d, L0 = _setup("c1", H=64, W=64, iters=5)
    md = _model(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]))
    c = P.ipiano_config_default(max_iters=5)
    u_h, tr_h = P.ipiano_run(md, d["f"], d["lambdas"], L0, c)
    u_d, tr_d = P.ipiano_run(md, _cuda(d["f"], torch.float32), d["lambdas"], L0, c)
    np.testing.assert_array_equal(u_h, u_d.cpu().numpy())
    np.testing.assert_array_equal(tr_h, tr_d)


def test_spec_policy_runs_and_descends():
    # SPEC.md:310-311 policy (beta = 0.8, L halves after each accept): decisions follow
    # the same test; H decreases overall and trials average ~2 per iteration
    cfg, d, L0 = _setup("c1", H=64, W=64, iters=30)
    md = _model(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]))
    c = P.ipiano_config_default(max_iters=30, beta=0.8, shrink=0.5)
    st = P.ipiano_state_create(md, _cuda(d["f"], torch.float32), d["lambdas"], L0, c)
    P.ipiano_solve(st)
    tr = P.ipiano_get_trace(st)[0]
    assert tr[-1, 2] < tr[0, 2]
    assert np.all(tr[1:, 5] >= 0)


def test_error_contracts():
    k, th = S.random_filter_bank(4, 7, 1)
    with pytest.raises(P.FoeError) as e:
        P.foe_model_create(k, -th)
    assert e.value.status == 1 and "filter 0" in e.value.message
    with pytest.raises(P.FoeError) as e:
        P.foe_model_create(np.zeros((2, 4, 4), np.float32), [1, 1])
    assert e.value.status == 1
    with pytest.raises(P.FoeError) as e:
        P.foe_model_create(k, th, lam=(0.0, 0.0))
    assert e.value.status == 1
    md = P.foe_model_create(k, th, looks=8)
    with pytest.raises(P.FoeError) as e:   # image smaller than the filter
        P.foe_energy_grad(md, torch.zeros((1, 5, 5), dtype=torch.float64, device="cuda"))
    assert e.value.status == 1
    f = torch.full((1, 32, 32), 50.0, device="cuda")
    with pytest.raises(P.FoeError) as e:
        P.ipiano_state_create(md, f, None, [1e5], P.ipiano_config_default(beta=1.0))
    assert e.value.status == 1


# ------------------------------------------------- full BASELINE sizes, sampled outputs

def _crop_periodic(img, y, x, r):
    ys = np.arange(y - r, y + r + 1) % img.shape[0]
    xs = np.arange(x - r, x + r + 1) % img.shape[1]
    return img[np.ix_(ys, xs)]


def _sampled_grad_check(w, g, filters, theta, n, seed):
    # grad at p depends on w within p +- (m-1): a periodic crop of side 2(m-1)+1 around p
    # gives the exact full-image value at the crop centre (no wrap inside the support)
    m = filters.shape[1]
    r = m - 1
    rng = np.random.default_rng(seed)
    H, W = w.shape
    ys = np.concatenate([rng.integers(0, H, n - 4), [0, H - 1, 0, H - 1]])
    xs = np.concatenate([rng.integers(0, W, n - 4), [0, W - 1, W - 1, 0]])
    ref = np.empty(n)
    for i, (y, x) in enumerate(zip(ys, xs)):
        _, gc = oracle.energy_grad_w(_crop_periodic(w, y, x, r), filters, theta)
        ref[i] = gc[r, r]
    got = g[ys, xs]
    return rel_l2(got, ref)


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_full_size_sampled_gradient(name):
    cfg = S.config(name)
    imgs = [0, 37, 63] if name == "c4" else None
    d = S.make_inputs(cfg, images=imgs)
    md = _model(d["filters"], d["theta"])
    w = np.log(np.maximum(d["f"].astype(np.float64), 1.0))
    F, _, g = P.foe_energy_grad(md, _cuda(w, torch.float64))
    g = g.cpu().numpy()
    for b in range(w.shape[0]):
        assert _sampled_grad_check(w[b], g[b], d["filters"], d["theta"], 200, b) <= 1e-5
    if name == "c3":
        assert F[0] == pytest.approx(oracle.energy_grad_w(w[0], d["filters"], d["theta"], False), rel=1e-6)


def test_c4_bench_launch_configuration_two_iterations():
    # the bench's launch configuration (all 64 images, automatic filter groups) for two
    # iterations; two sampled images are re-run by the oracle
    cfg = S.config("c4", iters=2)
    d = S.make_inputs(cfg)
    md = _model(d["filters"], d["theta"])
    v0 = S.lipschitz_start_vector(cfg.B, cfg.H, cfg.W)
    rho, L0 = P.foe_estimate_lipschitz(md, _cuda(d["f"], torch.float32), _cuda(v0, torch.float64))
    c = P.ipiano_config_default(max_iters=2)
    st = P.ipiano_state_create(md, _cuda(d["f"], torch.float32), d["lambdas"], L0, c)
    P.ipiano_solve(st)
    w, u = P.ipiano_get_iterate(st)
    u = u.cpu().numpy()
    for b in (5, 50):
        l1, l2 = d["lambdas"][b]
        ref = oracle.ipiano_run(d["f"][b], d["filters"], d["theta"], l1, l2, oracle.make_cfg(L0[b], 2))
        assert rel_l2(u[b], ref["u"]) <= 1e-5


def test_ipiano_run_workspace_reuse_is_exact():
    """ipiano_run keeps one workspace per model: a repeated call with new inputs and lambdas
    (host buffers, then device buffers) gives bit-identical results to a fresh state."""
    cfg = S.config("c2", H=96, W=80, iters=8, B=2)
    d = S.make_inputs(cfg, images=[0, 1])
    md = _model(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]))
    L0 = np.array([2.0 ** 18, 2.0 ** 17])
    c = P.ipiano_config_default(max_iters=cfg.iters)
    outs = []
    for scale, lam in ((1.0, d["lambdas"]), (1.3, d["lambdas"][::-1].copy())):
        f = (d["f"] * scale).astype(np.float32)
        u_h, tr_h = P.ipiano_run(md, f, lam, L0, c)                       # host in/out (cached)
        u_d, tr_d = P.ipiano_run(md, _cuda(f, torch.float32), lam, L0, c)  # device in/out (cached)
        st = P.ipiano_state_create(md, _cuda(f, torch.float32), lam, L0, c)   # fresh state
        P.ipiano_solve(st)
        _, u_f = P.ipiano_get_iterate(st, want_w=False)
        tr_f = P.ipiano_get_trace(st)
        np.testing.assert_array_equal(u_h, u_f.cpu().numpy())
        np.testing.assert_array_equal(u_d.cpu().numpy(), u_f.cpu().numpy())
        np.testing.assert_array_equal(tr_h, tr_f)
        outs.append(u_h)
    assert not np.array_equal(outs[0], outs[1])


@pytest.fixture(scope="module")
def c3_oracle_run():
    """The fp64 oracle's full c3 trajectory (512^2, L=8, 48 x 7x7, 300 iterations; ~1 min on
    16 host cores), shared by the P3 tests of both stencils."""
    cfg, d, L0 = _setup("c3")
    l1, l2 = d["lambdas"][0]
    ref = oracle.ipiano_run(d["f"][0], d["filters"], d["theta"], l1, l2, oracle.make_cfg(L0[0], cfg.iters))
    assert ref["status"] == 0
    return cfg, d, L0, ref


@pytest.mark.parametrize("stencil", [P.FOE_STENCIL_FFMA, P.FOE_STENCIL_TENSOR])
def test_free_running_c3_P3(c3_oracle_run, stencil):
    """P3 on the full BASELINE config 3 (512^2 x 300 iterations) on both prior stencils."""
    cfg, d, L0, ref = c3_oracle_run
    md = _model(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]))
    c = P.ipiano_config_default(max_iters=cfg.iters, stencil=stencil)
    st = P.ipiano_state_create(md, _cuda(d["f"], torch.float32), d["lambdas"], L0, c)
    P.ipiano_solve(st)
    _, u = P.ipiano_get_iterate(st)
    u = u.cpu().numpy()[0]
    tr = P.ipiano_get_trace(st)[0]
    assert rel_l2(u, ref["u"]) <= 1e-4
    clean = d["clean"][0]
    assert abs(oracle.psnr(u, clean) - oracle.psnr(ref["u"], clean)) <= 0.01
    np.testing.assert_array_equal(tr[1:, 3], ref["trace"][1:, 3])
    np.testing.assert_array_equal(tr[1:, 4], ref["trace"][1:, 4])
    np.testing.assert_allclose(tr[:, 2], ref["trace"][:, 2], rtol=1e-6)


def test_c4_bench_launch_config_full_trajectory_P3():
    """c4 in the launch configuration bench.py times (64 x 512^2, AUTO stencil -> K8, 300
    iterations, per-image L_init from the GPU estimate): images 5 and 42 free-running against
    the oracle run on each alone (final image rel L2 <= 1e-4, |dPSNR| <= 0.01 dB, identical
    decisions)."""
    cfg = S.config("c4")
    d = S.make_inputs(cfg)
    v0 = S.lipschitz_start_vector(cfg.B, cfg.H, cfg.W)
    md = _model(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]))
    _, L0 = P.foe_estimate_lipschitz(md, _cuda(d["f"], torch.float32), _cuda(v0, torch.float64), 25)
    c = P.ipiano_config_default(max_iters=cfg.iters)
    st = P.ipiano_state_create(md, _cuda(d["f"], torch.float32), d["lambdas"], L0, c)
    assert P.ipiano_state_stencil(st) == P.FOE_STENCIL_TENSOR
    P.ipiano_solve(st)
    _, u = P.ipiano_get_iterate(st)
    u = u.cpu().numpy()
    tr = P.ipiano_get_trace(st)
    for b in (5, 42):
        l1, l2 = d["lambdas"][b]
        ref = oracle.ipiano_run(d["f"][b], d["filters"], d["theta"], l1, l2, oracle.make_cfg(L0[b], cfg.iters))
        assert ref["status"] == 0
        assert rel_l2(u[b], ref["u"]) <= 1e-4, b
        clean = d["clean"][b]
        assert abs(oracle.psnr(u[b], clean) - oracle.psnr(ref["u"], clean)) <= 0.01
        np.testing.assert_array_equal(tr[b, 1:, 3], ref["trace"][1:, 3])
        np.testing.assert_array_equal(tr[b, 1:, 4], ref["trace"][1:, 4])


def test_c4_teacher_forced_P2_every_10():
    """P2 at the bench's launch configuration (k = 10 on c4): the full c4 batch
    (64 x 512^2, AUTO stencil -> K8 with packed tiles, K2 at 16 px/thread) advanced one accepted
    iteration at a time; at iterations 10, 20, 30 the oracle redoes the next iteration of images
    0 and 37 from the GPU's own state (w_n, w_{n-1}, L_n): update w+ - w within 1e-5 relative L2
    and the same trial count unless the margin is a near-tie."""
    cfg = S.config("c4")
    d = S.make_inputs(cfg)
    v0 = S.lipschitz_start_vector(cfg.B, cfg.H, cfg.W)
    md = _model(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]))
    _, L0 = P.foe_estimate_lipschitz(md, _cuda(d["f"], torch.float32), _cuda(v0, torch.float64), 25)
    st = P.ipiano_state_create(md, _cuda(d["f"], torch.float32), d["lambdas"], L0,
                               P.ipiano_config_default(max_iters=31))
    assert P.ipiano_state_stencil(st) == P.FOE_STENCIL_TENSOR
    imgs = (0, 37)
    w_prev = None
    w_cur = P.ipiano_get_iterate(st, want_u=False)[0].cpu().numpy()[list(imgs)]
    for n in range(31):
        if n in (10, 20, 30):
            L = P.ipiano_get_counters(st)["L"]
            P.ipiano_step(st)
            w_next = P.ipiano_get_iterate(st, want_u=False)[0].cpu().numpy()[list(imgs)]
            tr = P.ipiano_get_trace(st)
            for k, b in enumerate(imgs):
                f = d["f"][b]
                l1, l2 = d["lambdas"][b]
                F, g = oracle.energy_grad_w(w_cur[k], d["filters"], d["theta"])
                Lb, trials = L[b], 0
                while True:
                    trials += 1
                    r = oracle.ipiano_trial(w_cur[k], w_prev[k], g, F, Lb, f, d["filters"], d["theta"], l1, l2,
                                            oracle.make_cfg(Lb, 1))
                    if r["accepted"]:
                        break
                    Lb *= 2
                assert trials == tr[b, n + 1, 4] or abs(r["margin"]) < 1e-6 * abs(F), (n, b)
                assert rel_l2(w_next[k] - w_cur[k], r["wplus"] - w_cur[k]) <= 1e-5, (n, b)
        else:
            P.ipiano_step(st)
            w_next = P.ipiano_get_iterate(st, want_u=False)[0].cpu().numpy()[list(imgs)]
        w_prev, w_cur = w_cur, w_next
