"""GPU parity at scale and for model (8), against the fp64 oracle.

* c5 (BASELINE.json configs[4]: 8192^2 SAR-like scene, L=1, 48 x 7x7, 300 iterations) in the
  row-slab launch configuration of the bench (4 slabs, tensor-core stencil): P2 teacher forcing
  at iterations 10, 150 and 290 (k = 10 schedule of SURVEY 8(c), sampled) -- the oracle redoes
  the next accepted iteration of the WHOLE scene from the GPU's own (w_n, w_{n-1}, L_n): update
  w+ - w within 1e-5 relative L2 and the same trial count unless the oracle's margin is a
  near-tie (|margin| < 1e-6 |F|).
* A 1024^2 scene of the same SAR-like generator (wider dynamic range, point targets at 255)
  on 4 slabs with the tensor-core stencil, free-running for 300 iterations (P3): final image
  relative L2 <= 1e-4, |dPSNR| <= 0.01 dB, identical L_n and trial traces.
* Model (8) alone (FOE_DATA_NAKAGAMI: lambda_2 = 0, its Newton prox
  :185-192): P1 and P3 on the c1 / c2 shapes, both prior stencils.  The oracle's model (8) is
  its combined model with lambda_2 = 0 (pinned against the Lambert-W closed form of Eq. (8)'s
  prox in tests/test_oracle_pins.py).
"""
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
    P.lib()


def rel_l2(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _cuda(a, dtype):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def _slab_w(sl):
    w, _ = P.ipiano_slabs_get_iterate(sl, want_u=False)
    torch.cuda.synchronize()
    return w.cpu().numpy()


def _oracle_next(w_cur, w_prev, L, f, k, th, l1, l2):
    """One accepted iteration of algorithm C-0 from (w_n, w_{n-1}, L_n): (w+, trials, margin, F)."""
    F, g = oracle.energy_grad_w(w_cur, k, th)
    trials = 0
    while True:
        trials += 1
        r = oracle.ipiano_trial(w_cur, w_prev, g, F, L, f, k, th, l1, l2, oracle.make_cfg(L, 1), want_gplus=False)
        if r["accepted"]:
            return r["wplus"], trials, r["margin"], F
        L *= 2.0
        assert trials < 60


def test_c5_full_scene_teacher_forced_P2():
    cfg = S.config("c5")
    d = S.make_inputs(cfg)
    f = d["f"][0]
    k, th = d["filters"], d["theta"]
    l1, l2 = d["lambdas"][0]
    md = P.foe_model_create(k, th, lam=(l1, l2))
    v0 = S.lipschitz_start_vector(1, cfg.H, cfg.W)
    _, L0 = P.foe_estimate_lipschitz(md, _cuda(d["f"], torch.float32), _cuda(v0, torch.float64), 25)
    c = P.ipiano_config_default(max_iters=cfg.iters, stencil=P.FOE_STENCIL_TENSOR)
    sl = P.ipiano_slabs_create(md, _cuda(f, torch.float32), cfg.H, nslabs=4, lam=(l1, l2),
                               lipschitz_init=float(L0[0]), cfg=c)
    try:
        assert P.ipiano_state_stencil(P.ipiano_slabs_member(sl, 0)) == P.FOE_STENCIL_TENSOR
        for n in (10, 150, 290):
            P.ipiano_slabs_advance(sl, n - 1)
            w_prev = _slab_w(sl)
            P.ipiano_slabs_advance(sl, n)
            w_cur = _slab_w(sl)
            L = float(P.ipiano_get_counters(P.ipiano_slabs_member(sl, 0))["L"][0])
            P.ipiano_slabs_advance(sl, n + 1)
            w_next = _slab_w(sl)
            tr = P.ipiano_get_trace(P.ipiano_slabs_member(sl, 0))[0]
            assert P.ipiano_get_counters(P.ipiano_slabs_member(sl, 0))["iters"][0] == n + 1
            wplus, trials, margin, F = _oracle_next(w_cur, w_prev, L, f, k, th, l1, l2)
            assert trials == tr[n + 1, 4] or abs(margin) < 1e-6 * abs(F), (n, trials, tr[n + 1, 4], margin)
            err = rel_l2(w_next - w_cur, wplus - w_cur)
            assert err <= 1e-5, (n, err)
            del w_prev, w_cur, w_next, wplus
    finally:
        sl.destroy()


def test_sar_1024_slabs_tensor_P3():
    H = W = 1024
    clean = S.sar_like_scene(H, W, 611)
    f = S.add_speckle(clean, 1, 612)
    k, th = S.random_filter_bank(48, 7, 603)
    lam = (160.0, 0.004)
    md = P.foe_model_create(k, th, lam=lam)
    v0 = S.lipschitz_start_vector(1, H, W)
    _, L0 = P.foe_estimate_lipschitz(md, _cuda(f[None], torch.float32), _cuda(v0, torch.float64), 25)
    L0 = float(L0[0])
    c = P.ipiano_config_default(max_iters=300, stencil=P.FOE_STENCIL_TENSOR)
    sl = P.ipiano_slabs_create(md, _cuda(f, torch.float32), H, nslabs=4, lam=lam, lipschitz_init=L0, cfg=c)
    try:
        assert P.ipiano_state_stencil(P.ipiano_slabs_member(sl, 0)) == P.FOE_STENCIL_TENSOR
        P.ipiano_slabs_solve(sl)
        _, u = P.ipiano_slabs_get_iterate(sl)
        u = u.cpu().numpy()
        tr = P.ipiano_get_trace(P.ipiano_slabs_member(sl, 0))[0]
        cnt = P.ipiano_get_counters(P.ipiano_slabs_member(sl, 0))
    finally:
        sl.destroy()
    assert cnt["status"][0] == 0 and cnt["iters"][0] == 300
    ref = oracle.ipiano_run(f, k, th, lam[0], lam[1], oracle.make_cfg(L0, 300))
    assert ref["status"] == 0
    assert rel_l2(u, ref["u"]) <= 1e-4
    assert abs(oracle.psnr(u, clean) - oracle.psnr(ref["u"], clean)) <= 0.01
    np.testing.assert_array_equal(tr[1:, 3], ref["trace"][1:, 3])
    np.testing.assert_array_equal(tr[1:, 4], ref["trace"][1:, 4])
    np.testing.assert_allclose(tr[:, 2], ref["trace"][:, 2], rtol=1e-6)


# ------------------------------------------------------------------- model (8) alone

STENCILS = [P.FOE_STENCIL_FFMA, P.FOE_STENCIL_TENSOR]


def _nakagami_setup(name, **over):
    cfg = S.config(name, **over)
    d = S.make_inputs(cfg)
    v0 = S.lipschitz_start_vector(cfg.B, cfg.H, cfg.W)
    L0 = np.array([oracle.estimate_lipschitz(d["f"][b], d["filters"], d["theta"], v0[b])[1]
                   for b in range(cfg.B)])
    l1 = float(d["lambdas"][0][0])
    md = P.foe_model_create(d["filters"], d["theta"], lam=(l1, 0.0), term=P.FOE_DATA_NAKAGAMI)
    return cfg, d, L0, l1, md


@pytest.mark.parametrize("stencil", STENCILS)
def test_nakagami_single_step_P1(stencil):
    cfg, d, L0, l1, md = _nakagami_setup("c2", H=96, W=80, iters=3)
    lam = np.array([[l1, 0.0]])
    st = P.ipiano_state_create(md, _cuda(d["f"], torch.float32), lam, L0,
                               P.ipiano_config_default(max_iters=3, stencil=stencil))
    P.ipiano_step(st)
    wg = P.ipiano_get_iterate(st, want_u=False)[0].cpu().numpy()[0]
    tr = P.ipiano_get_trace(st)[0]
    f = d["f"][0]
    w0 = np.log(oracle.ftilde(f))
    F0, g0 = oracle.energy_grad_w(w0, d["filters"], d["theta"])
    r = oracle.ipiano_trial(w0, w0, g0, F0, L0[0], f, d["filters"], d["theta"], l1, 0.0, oracle.make_cfg(L0[0], 3))
    assert r["accepted"] and tr[1, 4] == 1
    assert rel_l2(wg - w0, r["wplus"] - w0) <= 1e-5
    assert tr[1, 0] == pytest.approx(r["Fplus"], rel=1e-6)
    assert tr[1, 1] == pytest.approx(r["Gplus"], rel=1e-9)
    # the data term is model (8): G = (lambda/2) sum (2w + f~^2 e^{-2w})
    ft = oracle.ftilde(f)
    G8 = 0.5 * l1 * np.sum(2.0 * wg + ft ** 2 * np.exp(-2.0 * wg))
    assert tr[1, 1] == pytest.approx(G8, rel=1e-9)


@pytest.mark.parametrize("stencil", STENCILS)
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_nakagami_free_running_P3(name, stencil):
    cfg, d, L0, l1, md = _nakagami_setup(name)
    lam = np.array([[l1, 0.0]])
    st = P.ipiano_state_create(md, _cuda(d["f"], torch.float32), lam, L0,
                               P.ipiano_config_default(max_iters=cfg.iters, stencil=stencil))
    P.ipiano_solve(st)
    _, u = P.ipiano_get_iterate(st)
    u = u.cpu().numpy()[0]
    tr = P.ipiano_get_trace(st)[0]
    assert P.ipiano_get_counters(st)["status"][0] == 0
    ref = oracle.ipiano_run(d["f"][0], d["filters"], d["theta"], l1, 0.0, oracle.make_cfg(L0[0], cfg.iters))
    assert ref["status"] == 0
    assert rel_l2(u, ref["u"]) <= 1e-4
    clean = d["clean"][0]
    assert abs(oracle.psnr(u, clean) - oracle.psnr(ref["u"], clean)) <= 0.01
    np.testing.assert_array_equal(tr[1:, 3], ref["trace"][1:, 3])
    np.testing.assert_array_equal(tr[1:, 4], ref["trace"][1:, 4])
