"""GPU: the persistent small-image driver (FOE_SOLVER_PERSISTENT) against the
graph driver and the oracle.

Both drivers run the same per-pixel K2 and the same K1 tiles/filter groups; the persistent one
cuts K2 into smaller pixel blocks (so its test sums are added in a different order) and takes
each decision redundantly in every CTA.  So the two must take identical decisions (L_n and
trial counts) and agree on the iterate to fp64 rounding of the step arithmetic, and the
persistent driver must meet the oracle parity bar of configs c1-c3 itself (north_star:
final image rel L2 <= 1e-4, |dPSNR| <= 0.01 dB).  The oracle P3 runs of c1/c2/c3 in
test_gpu_parity.py go through FOE_SOLVER_AUTO, which resolves to this driver there (asserted
below).
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


def _inputs(name, **over):
    cfg = S.config(name, **over)
    d = S.make_inputs(cfg)
    md = P.foe_model_create(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]))
    v0 = S.lipschitz_start_vector(cfg.B, cfg.H, cfg.W)
    _, L0 = P.foe_estimate_lipschitz(md, _cuda(d["f"], torch.float32), _cuda(v0, torch.float64), 25)
    return cfg, d, md, L0


def _run(md, d, L0, iters, solver, model_lams=None, **cfg_over):
    c = P.ipiano_config_default(max_iters=iters, solver=solver, **cfg_over)
    lam = d["lambdas"] if model_lams is None else model_lams
    st = P.ipiano_state_create(md, _cuda(d["f"], torch.float32), lam, L0, c)
    P.ipiano_solve(st)
    w, u = P.ipiano_get_iterate(st)
    return (P.ipiano_state_solver(st), w.cpu().numpy(), u.cpu().numpy(), P.ipiano_get_trace(st),
            P.ipiano_get_counters(st))


def _same_trajectory(a, b, wtol=1e-12):
    _, wa, _, ta, ca = a
    _, wb, _, tb, cb = b
    np.testing.assert_array_equal(ca["iters"], cb["iters"])
    np.testing.assert_array_equal(ca["trials"], cb["trials"])
    np.testing.assert_array_equal(ca["status"], cb["status"])
    np.testing.assert_array_equal(ta[:, :, 3], tb[:, :, 3])   # L_n of every accepted iteration
    np.testing.assert_array_equal(ta[:, :, 4], tb[:, :, 4])   # trials of every iteration
    np.testing.assert_array_equal(ta[:, :, 0], tb[:, :, 0])   # F: same K1 partials, same order
    np.testing.assert_allclose(ta[:, :, 1], tb[:, :, 1], rtol=1e-12)   # G: K2 block sums reordered
    for b in range(wa.shape[0]):
        assert rel_l2(wa[b], wb[b]) <= wtol, b


@pytest.mark.parametrize("name,iters", [("c1", 100), ("c2", 60), ("c3", 20)])
def test_persistent_matches_graph(name, iters):
    cfg, d, md, L0 = _inputs(name)
    a = _run(md, d, L0, iters, P.FOE_SOLVER_GRAPH, stencil=P.FOE_STENCIL_FFMA)
    b = _run(md, d, L0, iters, P.FOE_SOLVER_PERSISTENT)
    assert a[0] == P.FOE_SOLVER_GRAPH and b[0] == P.FOE_SOLVER_PERSISTENT
    _same_trajectory(a, b)
    # AUTO resolves to the persistent FFMA driver for images below 2^16 pixels (c1), and to the
    # graph driver with the tensor-core stencil in short tiles from there (c2: 4-row, c3: 8-row)
    c = P.ipiano_config_default(max_iters=1)
    st = P.ipiano_state_create(md, _cuda(d["f"], torch.float32), d["lambdas"], L0, c)
    if name in ("c2", "c3"):
        assert P.ipiano_state_solver(st) == P.FOE_SOLVER_GRAPH
        assert P.ipiano_state_stencil(st) == P.FOE_STENCIL_TENSOR
    else:
        assert P.ipiano_state_solver(st) == P.FOE_SOLVER_PERSISTENT
        assert P.ipiano_state_stencil(st) == P.FOE_STENCIL_FFMA


def test_persistent_P3_c1_against_oracle():
    # the explicit persistent driver on BASELINE config 1 against the fp64 oracle (P3)
    cfg = S.config("c1")
    d = S.make_inputs(cfg)
    v0 = S.lipschitz_start_vector(1, cfg.H, cfg.W)
    L0 = np.array([oracle.estimate_lipschitz(d["f"][0], d["filters"], d["theta"], v0[0])[1]])
    md = P.foe_model_create(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]))
    solver, _, u, tr, cnt = _run(md, d, L0, cfg.iters, P.FOE_SOLVER_PERSISTENT)
    assert solver == P.FOE_SOLVER_PERSISTENT
    assert cnt["status"][0] == 0 and cnt["iters"][0] == cfg.iters
    l1, l2 = d["lambdas"][0]
    ref = oracle.ipiano_run(d["f"][0], d["filters"], d["theta"], l1, l2, oracle.make_cfg(L0[0], cfg.iters))
    assert rel_l2(u[0], ref["u"]) <= 1e-4
    clean = d["clean"][0]
    assert abs(oracle.psnr(u[0], clean) - oracle.psnr(ref["u"], clean)) <= 0.01
    np.testing.assert_array_equal(tr[0, 1:, 3], ref["trace"][1:, 3])
    np.testing.assert_array_equal(tr[0, 1:, 4], ref["trace"][1:, 4])
    np.testing.assert_allclose(tr[0, :, 2], ref["trace"][:, 2], rtol=1e-6)


def test_persistent_batch_mixed_looks_and_backtracking():
    # B = 3 images with their own lambdas (L = 1, 3, 8) under the SPEC policy (beta = 0.8, L_n
    # halved after every accept): about two trials per iteration, so images
    # backtrack and leave the trial loop at different rounds
    cfg, d, md, L0 = _inputs("c4", B=3, H=96, W=112, iters=15)
    pol = dict(beta=0.8, shrink=0.5)
    a = _run(md, d, L0, cfg.iters, P.FOE_SOLVER_GRAPH, **pol)
    b = _run(md, d, L0, cfg.iters, P.FOE_SOLVER_PERSISTENT, **pol)
    assert b[0] == P.FOE_SOLVER_PERSISTENT
    assert np.all(b[4]["trials"] > cfg.iters + 3)          # backtracked
    _same_trajectory(a, b)


def test_persistent_step_and_rel_change_stop():
    cfg, d, md, L0 = _inputs("c1", H=80, W=72, iters=8)
    c = P.ipiano_config_default(max_iters=8, solver=P.FOE_SOLVER_PERSISTENT)
    st = P.ipiano_state_create(md, _cuda(d["f"], torch.float32), d["lambdas"], L0, c)
    for n in range(8):
        assert P.ipiano_step(st)[0] == n + 1
    w_step = P.ipiano_get_iterate(st, want_u=False)[0].cpu().numpy()
    _, w_solve, _, _, _ = _run(md, d, L0, 8, P.FOE_SOLVER_PERSISTENT)
    np.testing.assert_array_equal(w_step, w_solve)
    # rel_change_tol: both drivers stop at the same iteration
    a = _run(md, d, L0, 200, P.FOE_SOLVER_GRAPH, rel_change_tol=2e-3)
    b = _run(md, d, L0, 200, P.FOE_SOLVER_PERSISTENT, rel_change_tol=2e-3)
    assert 0 < a[4]["iters"][0] < 200
    _same_trajectory(a, b)


def test_persistent_idiv_model():
    cfg = S.config("c1", H=96, W=96, iters=30)
    d = S.make_inputs(cfg)
    lam = S.idiv_lambda(int(d["looks"][0]))
    md = P.foe_model_create(d["filters"], d["theta"], lam=(lam, 0.0), term=P.FOE_DATA_IDIV)
    v0 = S.lipschitz_start_vector(1, cfg.H, cfg.W)
    _, L0 = P.foe_estimate_lipschitz(md, _cuda(d["f"], torch.float32), _cuda(v0, torch.float64), 25)
    a = _run(md, d, L0, cfg.iters, P.FOE_SOLVER_GRAPH, model_lams=[lam, 0.0])
    b = _run(md, d, L0, cfg.iters, P.FOE_SOLVER_PERSISTENT, model_lams=[lam, 0.0])
    assert b[0] == P.FOE_SOLVER_PERSISTENT
    _same_trajectory(a, b)


def test_persistent_contracts():
    cfg, d, md, L0 = _inputs("c1", H=64, W=64, iters=2)
    f = _cuda(d["f"], torch.float32)
    with pytest.raises(P.FoeError) as e:
        P.ipiano_state_create(md, f, d["lambdas"], L0, P.ipiano_config_default(solver=7))
    assert e.value.status == 1
    with pytest.raises(P.FoeError) as e:
        P.ipiano_state_create(md, f, d["lambdas"], L0,
                              P.ipiano_config_default(solver=P.FOE_SOLVER_PERSISTENT, stencil=P.FOE_STENCIL_TENSOR))
    assert e.value.status == 9
    # profiling (per-launch K1 events) runs the graph rounds on a persistent state: same result
    st = P.ipiano_state_create(md, f, d["lambdas"], L0, P.ipiano_config_default(max_iters=2))
    P.ipiano_profile(st, 1)
    P.ipiano_solve(st)
    w_prof = P.ipiano_get_iterate(st, want_u=False)[0].cpu().numpy()
    _, w_pers, _, _, _ = _run(md, d, L0, 2, P.FOE_SOLVER_PERSISTENT)
    assert rel_l2(w_prof, w_pers) <= 1e-12


def test_persistent_bitwise_deterministic_and_per_image_stops():
    # the redundant per-CTA decisions and fixed-order reductions: two solves are bitwise equal;
    # with rel_change_tol, images of a batch stop at different iterations and the others go on
    cfg, d, md, L0 = _inputs("c4", B=3, H=80, W=96, iters=60)
    free = _run(md, d, L0, 60, P.FOE_SOLVER_PERSISTENT)
    relchg = free[3][:, 1:, 7]                      # ||w_n - w_{n-1}|| / max(||w_{n-1}||, 1) per image
    tol = float(np.sort(relchg[:, 0])[1])           # the middle image's first change: the image with
                                                    # the smallest first step stops at once, the others run on
    runs = [_run(md, d, L0, 60, P.FOE_SOLVER_PERSISTENT, rel_change_tol=tol) for _ in range(2)]
    np.testing.assert_array_equal(runs[0][1], runs[1][1])
    np.testing.assert_array_equal(runs[0][3], runs[1][3])
    iters = runs[0][4]["iters"]
    assert len(set(iters.tolist())) > 1, (iters, relchg[:, :4])
    g = _run(md, d, L0, 60, P.FOE_SOLVER_GRAPH, rel_change_tol=tol)
    _same_trajectory(g, runs[0])
