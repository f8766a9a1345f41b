"""GPU parity of the variant model (6) in u (FOE_DATA_IDIV) against the
oracle's u-domain tier (tests/test_oracle_idiv.py pins it): gradient grad_u F (no W) on both
prior stencils, the I-divergence data energy, the u-domain Hessian-vector product and
Lipschitz estimate, a single iPiano step (P1) and free-running runs (P3), and the slab path.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import foe_synth as S  # noqa: E402
import oracle  # noqa: E402
import paper_1404_5344_b200 as P  # noqa: E402

STENCILS = [P.FOE_STENCIL_FFMA, P.FOE_STENCIL_TENSOR]


@pytest.fixture(scope="module", autouse=True)
def _require_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    P.lib()


def rel_l2(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _cuda(a, dtype):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def _model(k, th, lam):
    return P.foe_model_create(k, th, lam=(lam, 0.0), term=P.FOE_DATA_IDIV)


@pytest.mark.parametrize("stencil", STENCILS)
@pytest.mark.parametrize("m,nf,H,W", [(7, 48, 150, 260), (5, 24, 130, 129), (7, 48, 12, 12)])
def test_idiv_energy_grad_parity(stencil, m, nf, H, W):
    k, th = S.random_filter_bank(nf, m, 3000 + m + nf)
    f = S.add_speckle(S.piecewise_smooth_scene(H, W, 61), 3, 62)[None]
    u = np.maximum(f.astype(np.float64), 1.0) * (1 + 0.01 * np.random.default_rng(1).standard_normal(f.shape))
    lam = S.idiv_lambda(3)
    md = _model(k, th, lam)
    P.foe_model_set_stencil(md, stencil)
    Fg, Gg, g = P.foe_energy_grad(md, _cuda(u, torch.float64), f=_cuda(f, torch.float32), data=True,
                                  lam_per_image=[lam, 0.0])
    Fo, go = oracle.energy_grad_u(u[0], k, th)
    assert rel_l2(g.cpu().numpy()[0], go) <= 1e-5
    assert Fg[0] == pytest.approx(Fo, rel=1e-6)
    assert Gg[0] == pytest.approx(oracle.idiv_energy(u[0], oracle.ftilde(f[0]), lam), rel=1e-12)


def test_idiv_hvp_and_lipschitz():
    k, th = S.random_filter_bank(24, 7, 6)
    f = S.add_speckle(S.piecewise_smooth_scene(70, 90, 3), 1, 4)[None]
    u = np.maximum(f.astype(np.float64), 1.0)
    v = np.random.default_rng(0).standard_normal(u.shape)
    md = _model(k, th, S.idiv_lambda(1))
    hv = P.foe_hvp(md, _cuda(u, torch.float64), _cuda(v, torch.float64)).cpu().numpy()
    assert rel_l2(hv[0], oracle.hvp_u(u[0], v[0], k, th)) <= 1e-4
    v0 = S.lipschitz_start_vector(1, 70, 90)
    rho, L = P.foe_estimate_lipschitz(md, _cuda(f, torch.float32), _cuda(v0, torch.float64), 25)
    rho_o, L_o = oracle.estimate_lipschitz_u(f[0], k, th, v0[0], 25)
    assert rho[0] == pytest.approx(rho_o, rel=1e-4) and L[0] == L_o


def _case(name, **over):
    cfg = S.config(name, **over)
    d = S.make_inputs(cfg)
    lam = S.idiv_lambda(int(d["looks"][0]))
    v0 = S.lipschitz_start_vector(1, cfg.H, cfg.W)
    _, L0 = oracle.estimate_lipschitz_u(d["f"][0], d["filters"], d["theta"], v0[0])
    return cfg, d, lam, L0


def test_idiv_single_step_P1():
    cfg, d, lam, L0 = _case("c2", H=96, W=80)
    md = _model(d["filters"], d["theta"], lam)
    st = P.ipiano_state_create(md, _cuda(d["f"], torch.float32), [lam, 0.0], [L0], P.ipiano_config_default(max_iters=2))
    P.ipiano_step(st)
    ug, _ = P.ipiano_get_iterate(st, want_u=False)
    ug = ug.cpu().numpy()[0]
    f = d["f"][0]
    u0 = oracle.ftilde(f)
    F0, g0 = oracle.energy_grad_u(u0, d["filters"], d["theta"])
    r = oracle.ipiano_trial_u(u0, u0, g0, F0, L0, f, d["filters"], d["theta"], lam, oracle.make_cfg(L0, 1))
    tr = P.ipiano_get_trace(st)[0]
    assert r["accepted"] and tr[1, 4] == 1
    assert rel_l2(ug - u0, r["uplus"] - u0) <= 1e-5
    assert tr[1, 0] == pytest.approx(r["Fplus"], rel=1e-6)
    assert tr[1, 1] == pytest.approx(r["Gplus"], rel=1e-9)


@pytest.mark.parametrize("stencil", STENCILS)
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_idiv_free_running_P3(name, stencil):
    cfg, d, lam, L0 = _case(name)
    md = _model(d["filters"], d["theta"], lam)
    c = P.ipiano_config_default(max_iters=cfg.iters, stencil=stencil)
    u, tr = P.ipiano_run(md, _cuda(d["f"], torch.float32), [lam, 0.0], [L0], c)
    u = u.cpu().numpy()[0]
    ref = oracle.ipiano_run_u(d["f"][0], d["filters"], d["theta"], lam, oracle.make_cfg(L0, cfg.iters))
    assert ref["status"] == 0
    assert rel_l2(u, ref["u"]) <= 1e-4
    clean = d["clean"][0]
    assert abs(oracle.psnr(u, clean) - oracle.psnr(ref["u"], clean)) <= 0.01
    np.testing.assert_array_equal(tr[0, 1:, 3], ref["trace"][1:, 3])
    np.testing.assert_array_equal(tr[0, 1:, 4], ref["trace"][1:, 4])
    np.testing.assert_allclose(tr[0, :, 2], ref["trace"][:, 2], rtol=1e-6)


def test_idiv_slabs_g_invariant():
    H, W = 256, 96
    f = S.add_speckle(S.piecewise_smooth_scene(H, W, 71), 1, 72)
    k, th = S.random_filter_bank(48, 7, 603)
    lam = S.idiv_lambda(1)
    md = _model(k, th, lam)
    outs = []
    for G in (1, 4):
        sl = P.ipiano_slabs_create(md, _cuda(f, torch.float32), H, nslabs=G, lam=(lam, 0.0), lipschitz_init=512.0,
                                   cfg=P.ipiano_config_default(max_iters=12))
        P.ipiano_slabs_solve(sl)
        w, u = P.ipiano_slabs_get_iterate(sl)
        outs.append((w.cpu().numpy(), u.cpu().numpy()))
        sl.destroy()
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][0].astype(np.float32), outs[0][1])     # u_out = the iterate
    ref = oracle.ipiano_run_u(f, k, th, lam, oracle.make_cfg(512.0, 12))
    assert rel_l2(outs[0][1], ref["u"]) <= 1e-4
