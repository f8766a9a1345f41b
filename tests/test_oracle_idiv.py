"""Pins of the oracle's variant model (6) in u (I-divergence data term).

PAPER.md:143-150 (Eq.(5), model (6)), :194-204 (grad_u F and the closed-form prox).  As
in test_oracle_pins.py, no test re-types the oracle's formula: the prox is checked against
bounded scalar minimisation and SPEC.md's worked values, the data term against the combined
model's independent implementation, the Hessian against finite differences
and a dense eigensolver, and the iPiano loop against its Lyapunov inequality, the
proximal-point special case and monotonicity for beta = 0.
"""
import math

import numpy as np
import pytest
import scipy.optimize as sopt

import foe_synth as S
import oracle
from oracle import brute

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


def _rng(seed=0):
    return np.random.default_rng(seed)


def _bank(n, m, seed):
    k, th = S.random_filter_bank(n, m, seed)
    return k.astype(np.float64), th.astype(np.float64)


def _problem(H=20, W=22, L=3, seed=0, nf=8, m=5):
    u = S.piecewise_smooth_scene(H, W, 900 + seed)
    f = S.add_speckle(u, L, 910 + seed)
    k, th = _bank(nf, m, 920 + seed)
    return u, f, k, th, S.idiv_lambda(L)


def test_idiv_prox_spec_values():
    # u^=0, f=1, tau lam=1 -> sqrt(2)/2; u^=f=c is a fixed point; tau lam -> 0 -> u^
    assert oracle.idiv_prox_pixel(0.0, 1.0, 1.0, 1.0) == pytest.approx(math.sqrt(2) / 2, rel=1e-15)
    for c in (0.5, 1.0, 100.0):
        assert oracle.idiv_prox_pixel(c, c, 0.7, 1.3) == pytest.approx(c, rel=1e-14)
    assert oracle.idiv_prox_pixel(37.0, 5.0, 1e-14, 1.0) == pytest.approx(37.0, rel=1e-12)


def test_idiv_prox_matches_scalar_minimisation():
    # the prox objective 1/2 (u - u^)^2 + tau lam/2 (u^2 - 2 f^2 log u) minimised numerically
    rng = _rng(3)
    for _ in range(300):
        uh = rng.uniform(-50, 300)
        f = rng.uniform(1, 255)
        tl = 10 ** rng.uniform(-4, 1)
        obj = lambda u: 0.5 * (u - uh) ** 2 + 0.5 * tl * (u * u - 2 * f * f * math.log(u))
        hi = max(abs(uh), f) * 4 + 10
        r = sopt.minimize_scalar(obj, bounds=(1e-9, hi), method="bounded",
                                 options={"xatol": 1e-12 * hi, "maxiter": 1000})
        u = oracle.idiv_prox_pixel(uh, f, tl, 1.0)
        assert u > 0
        assert u == pytest.approx(r.x, rel=1e-6, abs=1e-7)            # Brent's bounded search
        assert obj(u) <= obj(r.x) + 1e-12 * abs(obj(r.x))             # at least as good
        for d in (1e-6, -1e-6):                                         # a local minimum
            assert obj(u) <= obj(u * (1 + d))
        # the first-order condition, solved by bracketing root search on the derivative
        dobj = lambda x: (x - uh) + tl * (x - f * f / x)
        root = sopt.brentq(dobj, 1e-12, hi, xtol=1e-15, rtol=1e-15)
        assert u == pytest.approx(root, rel=1e-11)


def test_idiv_energy_values_and_minimiser():
    # f = u = 1, lam = 2, one pixel -> 1; per-pixel minimiser at u = f
    assert oracle.idiv_energy(np.ones((1, 1)), np.ones((1, 1)), 2.0) == pytest.approx(1.0, rel=1e-15)
    f = np.full((1, 1), 37.0)
    h = 1e-5
    d = (oracle.idiv_energy(f + h, f, 0.3) - oracle.idiv_energy(f - h, f, 0.3)) / (2 * h)
    assert abs(d) < 1e-6
    assert oracle.idiv_energy(f * 1.01, f, 0.3) > oracle.idiv_energy(f, f, 0.3)
    assert oracle.idiv_energy(f * 0.99, f, 0.3) > oracle.idiv_energy(f, f, 0.3)
    assert math.isnan(oracle.idiv_energy(np.zeros((1, 1)), f, 0.3))      # u > 0 required


def test_combined_with_lambda1_zero_is_idiv_at_exp_w():
    # Eq.(10) with l1 = 0 equals Eq.(5) at u = e^w with lam = l2 (two separate
    # implementations in the oracle: the w-domain combined term and the u-domain I-divergence)
    rng = _rng(4)
    w = rng.uniform(0.0, 5.5, (9, 11))
    ft = oracle.ftilde(rng.uniform(0, 255, (9, 11)).astype(np.float32))
    a = oracle.data_energy(w, ft, 0.0, 0.02)
    b = oracle.idiv_energy(np.exp(w), ft, 0.02)
    assert a == pytest.approx(b, rel=1e-12)


def test_hvp_u_matches_finite_difference_of_gradient():
    k, th = _bank(8, 5, 130)
    u = S.piecewise_smooth_scene(12, 13, 16).astype(np.float64)
    v = _rng(12).standard_normal(u.shape)
    h = 1e-4
    fd = (oracle.energy_grad_u(u + h * v, k, th)[1] - oracle.energy_grad_u(u - h * v, k, th)[1]) / (2 * h)
    hv = oracle.hvp_u(u, v, k, th)
    assert np.linalg.norm(hv - fd) <= 1e-6 * np.linalg.norm(fd)


def test_power_iteration_u_matches_dense_eigensolver():
    k, th = _bank(6, 3, 140)
    f = S.add_speckle(S.piecewise_smooth_scene(8, 8, 17), 3, 18)
    u0 = np.maximum(f.astype(np.float64), 1.0)
    Hm = brute.hessian_u(u0, k, th)
    top = np.abs(np.linalg.eigvalsh(0.5 * (Hm + Hm.T))).max()
    v0 = S.lipschitz_start_vector(1, 8, 8)[0]
    rho_hat, L0 = oracle.estimate_lipschitz_u(f, k, th, v0, iters=400)
    assert rho_hat == pytest.approx(top, rel=1e-4)
    assert L0 == 2.0 ** math.ceil(math.log2(rho_hat))


def test_ipiano_u_zero_prior_is_proximal_point_and_converges_to_f():
    # F = 0: one step = the closed-form prox; with beta = 0 the iterates go to
    # argmin D = f~ (D'(u) = lam (u - f^2/u) = 0 at u = f)
    u, f, k, th, lam = _problem()
    k = np.zeros_like(k)
    ft = oracle.ftilde(f)
    uh = ft * (1 + 0.2 * _rng(5).standard_normal(ft.shape))
    cfg = oracle.make_cfg(4.0, 1, beta=0.0)
    r = oracle.ipiano_trial_u(uh, uh, np.zeros_like(uh), 0.0, 4.0, f, k, th, lam, cfg)
    a = 0.95 * 2 / 4.0
    ref = np.array([[oracle.idiv_prox_pixel(uh[i, j], ft[i, j], a, lam) for j in range(uh.shape[1])]
                    for i in range(uh.shape[0])])
    np.testing.assert_array_equal(r["uplus"], ref)
    run = oracle.ipiano_run_u(f, k, th, lam, oracle.make_cfg(1.0, 5, beta=0.0))
    np.testing.assert_allclose(run["u"], ft, rtol=1e-12)


def _lyapunov_u(f, k, th, lam, cfg, steps):
    ft = oracle.ftilde(f)
    x = ft.copy(); xp = x.copy()
    F, g = oracle.energy_grad_u(x, k, th)
    L = cfg.lipschitz_init
    for _ in range(steps):
        while True:
            r = oracle.ipiano_trial_u(x, xp, g, F, L, f, k, th, lam, cfg)
            if r["accepted"]:
                break
            L *= cfg.backtrack_factor
        a = cfg.step_safety * 2 * (1 - cfg.beta) / L
        delta = 1 / a - L / 2 - cfg.beta / (2 * a)
        Hx = F + oracle.idiv_energy(x, ft, lam)
        lhs = r["Fplus"] + r["Gplus"] + delta * r["dd"]
        rhs = Hx + cfg.beta / (2 * a) * np.sum((x - xp) ** 2)
        assert lhs <= rhs + 1e-10 * abs(Hx), (lhs, rhs)
        assert np.all(r["uplus"] > 0)
        xp, x, g, F = x, r["uplus"], r["gplus"], r["Fplus"]
        L *= cfg.shrink


def test_ipiano_u_lyapunov_inequality():
    u, f, k, th, lam = _problem(seed=1)
    _, L0 = oracle.estimate_lipschitz_u(f, k, th, S.lipschitz_start_vector(1, *f.shape)[0])
    _lyapunov_u(f, k, th, lam, oracle.make_cfg(L0, 30), 30)
    _lyapunov_u(f, k, th, lam, oracle.make_cfg(L0 / 64, 20, beta=0.8, shrink=0.5), 20)   # SPEC policy


def test_ipiano_u_beta_zero_monotone_descent_and_consistency():
    u, f, k, th, lam = _problem(seed=2, L=1)
    _, L0 = oracle.estimate_lipschitz_u(f, k, th, S.lipschitz_start_vector(1, *f.shape)[0])
    run = oracle.ipiano_run_u(f, k, th, lam, oracle.make_cfg(L0, 40, beta=0.0))
    assert run["status"] == 0 and run["iters"] == 40
    H = run["trace"][:, 2]
    assert np.all(np.diff(H) <= 1e-9 * np.abs(H[:-1]))
    assert np.all(run["u"] > 0)
    run = oracle.ipiano_run_u(f, k, th, lam, oracle.make_cfg(L0, 40))
    tr = run["trace"]
    assert tr[-1, 2] < tr[0, 2] and np.all(tr[1:, 5] >= 0) and run["trials"] == int(tr[1:, 4].sum())
    # the first accepted step equals a direct trial from u^0
    ft = oracle.ftilde(f)
    F0, g0 = oracle.energy_grad_u(ft, k, th)
    short = oracle.ipiano_run_u(f, k, th, lam, oracle.make_cfg(L0, 1))
    r = oracle.ipiano_trial_u(ft, ft, g0, F0, short["trace"][1, 3], f, k, th, lam, oracle.make_cfg(L0, 1))
    np.testing.assert_array_equal(short["u"], r["uplus"])


def test_idiv_lambda_reading():
    # R-18: lam = l1 / u_rms^2 with the clean RMS 120.4 of Table II (C-14): equal curvature of
    # Eq.(5) and model (8)'s data term at u = f = u_rms
    for L in (1, 3, 8):
        l1 = S.LAMBDA_PRESETS[L][0]
        lam = S.idiv_lambda(L)
        u = 120.4
        d8 = l1 * (-1 / u ** 2 + 3 * u ** 2 / u ** 4)        # d^2/du^2 of l1/2 (2 log u + f^2/u^2) at f=u
        d6 = lam * (1 + u ** 2 / u ** 2)                     # d^2/du^2 of lam/2 (u^2 - 2 f^2 log u) at f=u
        assert d6 == pytest.approx(d8, rel=1e-12)
