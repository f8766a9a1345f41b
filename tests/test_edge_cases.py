"""GPU: degenerate and boundary inputs of the method against the fp64 oracle, on every driver
and stencil: zero and saturated pixels (the clamp f~ = max(f, 1) of R-4 on both sides), the
smallest image the filters allow (H = W = m), a one-column-wide K8 strip, images of one constant
value, and one-image batches next to much larger ones.  Tolerances as test_gpu_parity.py."""
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


def _clamped_scene(H, W, seed):
    """A speckled scene with ~10 % exact zeros, ~5 % values in (0, 1) and ~5 % saturated 255."""
    rng = np.random.default_rng(seed)
    f = S.add_speckle(S.piecewise_smooth_scene(H, W, seed), 1, seed + 1).astype(np.float32)
    r = rng.random((H, W))
    f[r < 0.10] = 0.0
    f[(r >= 0.10) & (r < 0.15)] = rng.random(int(((r >= 0.10) & (r < 0.15)).sum())).astype(np.float32)
    f[r > 0.95] = 255.0
    return f


@pytest.mark.parametrize("stencil,solver", [
    (P.FOE_STENCIL_FFMA, P.FOE_SOLVER_PERSISTENT),
    (P.FOE_STENCIL_FFMA, P.FOE_SOLVER_GRAPH),
    (P.FOE_STENCIL_TENSOR, P.FOE_SOLVER_GRAPH),
])
def test_zero_and_saturated_pixels_P3(stencil, solver):
    H, W, iters = 96, 130, 25
    f = _clamped_scene(H, W, 71)
    k, th = S.random_filter_bank(48, 7, 72)
    lam = (160.0, 0.004)
    v0 = S.lipschitz_start_vector(1, H, W)
    L0 = oracle.estimate_lipschitz(f, k, th, v0[0])[1]
    md = P.foe_model_create(k, th, lam=lam)
    st = P.ipiano_state_create(md, _cuda(f[None], torch.float32), None, [L0],
                               P.ipiano_config_default(max_iters=iters, stencil=stencil, solver=solver))
    assert P.ipiano_state_solver(st) == solver
    P.ipiano_solve(st)
    u = P.ipiano_get_iterate(st)[1].cpu().numpy()[0]
    tr = P.ipiano_get_trace(st)[0]
    ref = oracle.ipiano_run(f, k, th, lam[0], lam[1], oracle.make_cfg(L0, iters))
    assert ref["status"] == 0 and P.ipiano_get_counters(st)["status"][0] == 0
    assert rel_l2(u, ref["u"]) <= 1e-4
    np.testing.assert_array_equal(tr[1:, 4], ref["trace"][1:, 4])
    # the input is not modified and the clamp applies on the GPU as in the oracle
    assert np.all(u > 0) and np.isfinite(u).all()


@pytest.mark.parametrize("stencil", [P.FOE_STENCIL_FFMA, P.FOE_STENCIL_TENSOR])
def test_smallest_image_equals_filter_size(stencil):
    # H = W = m: every response wraps around the whole image several times
    k, th = S.random_filter_bank(48, 7, 81)
    rng = np.random.default_rng(82)
    w = np.log(rng.uniform(20.0, 220.0, (2, 7, 7)))
    md = P.foe_model_create(k, th, lam=(160.0, 0.004))
    P.foe_model_set_stencil(md, stencil)
    F, _, g = P.foe_energy_grad(md, _cuda(w, torch.float64))
    g = g.cpu().numpy()
    for b in range(2):
        Fo, go = oracle.energy_grad_w(w[b], k, th)
        assert rel_l2(g[b], go) <= 1e-5
        assert F[b] == pytest.approx(Fo, rel=1e-6)


def test_constant_images_stay_at_the_data_minimiser():
    # a constant observation: the prior gradient vanishes (zero-mean filters), so iPiano is the
    # plain prox iteration and every pixel converges to the same value on both sides
    H, W = 64, 80
    f = np.full((2, H, W), 97.0, np.float32)
    k, th = S.random_filter_bank(24, 5, 91)
    lam = (160.0, 0.004)
    md = P.foe_model_create(k, th, lam=lam)
    st = P.ipiano_state_create(md, _cuda(f, torch.float32), None, [2.0 ** 10] * 2, P.ipiano_config_default(max_iters=10))
    P.ipiano_solve(st)
    u = P.ipiano_get_iterate(st)[1].cpu().numpy()
    ref = oracle.ipiano_run(f[0], k, th, lam[0], lam[1], oracle.make_cfg(2.0 ** 10, 10))
    assert np.ptp(u) <= 1e-5 * u.max()
    assert rel_l2(u[0], ref["u"]) <= 1e-6


def test_one_column_strip_k8():
    # W = 1 column beyond full K8 tiles (122 + 1): the remainder packs into strips of 1 + 4C lanes
    k, th = S.random_filter_bank(48, 7, 101)
    rng = np.random.default_rng(102)
    w = np.log(rng.uniform(20.0, 220.0, (1, 200, 123)))
    md = P.foe_model_create(k, th, lam=(160.0, 0.004))
    P.foe_model_set_stencil(md, P.FOE_STENCIL_TENSOR)
    F, _, g = P.foe_energy_grad(md, _cuda(w, torch.float64))
    Fo, go = oracle.energy_grad_w(w[0], k, th)
    assert rel_l2(g.cpu().numpy()[0], go) <= 1e-5
    assert F[0] == pytest.approx(Fo, rel=1e-6)
