"""GPU parity of K8, the tensor-core (tcgen05, 3xTF32) prior energy + gradient stencil.

The same bars as K1 (BASELINE.json north_star): gradient relative L2 <= 1e-5 and energy to
1e-6 against the fp64 oracle; free-running final image relative L2 <= 1e-4, |dPSNR| <= 0.01 dB,
identical L_n / trial decisions (P3); K8 forced with FOE_STENCIL_TENSOR on shapes that span
several 64 x (128 - 2C) tiles, ragged tails, images smaller than a tile, padded filter
counts, both instantiated banks (m = 7, N_f <= 48; m = 5, N_f <= 32), and the slab path.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import foe_synth as S  # noqa: E402
import oracle  # noqa: E402
import paper_1404_5344_b200 as P  # noqa: E402

TENSOR, FFMA = P.FOE_STENCIL_TENSOR, P.FOE_STENCIL_FFMA


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


@pytest.mark.parametrize("m,nf,B,H,W", [
    (7, 48, 1, 64, 122),    # exactly one K8 tile
    (7, 48, 2, 150, 260),   # ragged in both axes (3 x 3 tiles), 2 images
    (7, 48, 1, 12, 12),     # image smaller than a tile: rows and columns wrap inside the tile
    (7, 40, 1, 130, 200),   # N_f padded to 48
    (7, 48, 1, 256, 256),   # c2 geometry
    (5, 24, 1, 130, 129),   # c1 bank, m = 5 (N_f padded to 32)
    (5, 32, 2, 70, 300),
    # column packing: the remainder columns of several 64-row bands share one tile
    (7, 48, 2, 209, 512),   # c4 width (4 full tiles + 24 columns), 4 bands -> 2 packed tiles, last with 1 strip
    (7, 48, 1, 64, 1000),   # one band: a packed tile with a single valid strip
])
def test_tc_energy_grad_parity(m, nf, B, H, W):
    k, th = S.random_filter_bank(nf, m, 2000 + m + nf)
    rng = np.random.default_rng(H * W + B + 7)
    f = np.stack([S.add_speckle(S.piecewise_smooth_scene(H, W, 30 + b), 3, 40 + b) for b in range(B)])
    w = np.log(np.maximum(f.astype(np.float64), 1.0)) + 0.01 * rng.standard_normal(f.shape)
    md = P.foe_model_create(k, th, lam=(310.0, 0.008))
    P.foe_model_set_stencil(md, TENSOR)
    Fg, _, g = P.foe_energy_grad(md, _cuda(w, torch.float64))
    g = g.cpu().numpy()
    for b in range(B):
        Fo, go = oracle.energy_grad_w(w[b], k, th)
        assert rel_l2(g[b], go) <= 1e-5, (b, rel_l2(g[b], go))
        assert Fg[b] == pytest.approx(Fo, rel=1e-6)


def test_tc_matches_ffma_stencil_512():
    """K8 and K1 on a c4-size image: both within the fp32 error of the exact gradient."""
    k, th = S.random_filter_bank(48, 7, 403)
    f = S.add_speckle(S.piecewise_smooth_scene(512, 512, 400), 8, 500)[None]
    w = _cuda(np.log(np.maximum(f.astype(np.float64), 1.0)), torch.float64)
    md = P.foe_model_create(k, th, lam=(550.0, 0.02))
    P.foe_model_set_stencil(md, TENSOR)
    Ft, _, gt = P.foe_energy_grad(md, w)
    P.foe_model_set_stencil(md, FFMA)
    Ff, _, gf = P.foe_energy_grad(md, w)
    assert rel_l2(gt.cpu().numpy(), gf.cpu().numpy()) <= 1e-5
    assert Ft[0] == pytest.approx(Ff[0], rel=1e-6)


def test_tc_constant_image_zero_gradient():
    k, th = S.random_filter_bank(48, 7, 5)
    md = P.foe_model_create(k, th, lam=(310.0, 0.008))
    P.foe_model_set_stencil(md, TENSOR)
    F, _, g = P.foe_energy_grad(md, _cuda(np.full((1, 96, 300), np.log(120.0)), torch.float64))
    assert np.abs(g.cpu().numpy()).max() < 1e-4
    assert F[0] < 1e-6


def test_tc_unsupported_bank():
    k, th = S.random_filter_bank(8, 3, 1)
    md = P.foe_model_create(k, th, lam=(310.0, 0.008))
    with pytest.raises(P.FoeError) as e:
        P.foe_model_set_stencil(md, TENSOR)
    assert e.value.status == 9


def _setup(name, **over):
    cfg = S.config(name, **over)
    d = S.make_inputs(cfg)
    v0 = S.lipschitz_start_vector(cfg.B, cfg.H, cfg.W)
    L0 = np.array([oracle.estimate_lipschitz(d["f"][b], d["filters"], d["theta"], v0[b])[1]
                   for b in range(cfg.B)])
    return cfg, d, L0


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_tc_free_running_P3(name):
    """P3 with K8 on the full BASELINE configs 1 and 2."""
    cfg, d, L0 = _setup(name)
    md = P.foe_model_create(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]))
    c = P.ipiano_config_default(max_iters=cfg.iters, stencil=TENSOR)
    st = P.ipiano_state_create(md, _cuda(d["f"], torch.float32), d["lambdas"], L0, c)
    P.ipiano_solve(st)
    _, u = P.ipiano_get_iterate(st)
    u = u.cpu().numpy()
    tr = P.ipiano_get_trace(st)
    cnt = P.ipiano_get_counters(st)
    assert cnt["status"][0] == 0 and cnt["iters"][0] == cfg.iters
    l1, l2 = d["lambdas"][0]
    ref = oracle.ipiano_run(d["f"][0], d["filters"], d["theta"], l1, l2, oracle.make_cfg(L0[0], cfg.iters))
    assert rel_l2(u[0], ref["u"]) <= 1e-4
    clean = d["clean"][0]
    assert abs(oracle.psnr(u[0], clean) - oracle.psnr(ref["u"], clean)) <= 0.01
    np.testing.assert_array_equal(tr[0, 1:, 3], ref["trace"][1:, 3])
    np.testing.assert_array_equal(tr[0, 1:, 4], ref["trace"][1:, 4])
    np.testing.assert_allclose(tr[0, :, 2], ref["trace"][:, 2], rtol=1e-6)


def test_tc_c4_bench_launch_config_sampled():
    """c4 in the bench's launch configuration (64 x 512^2, AUTO -> K8), 2 iterations: images 0
    and 37 against the oracle run on each alone."""
    cfg = S.config("c4", iters=2)
    d = S.make_inputs(cfg)
    v0 = S.lipschitz_start_vector(cfg.B, cfg.H, cfg.W)
    md = P.foe_model_create(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]))
    _, L0 = P.foe_estimate_lipschitz(md, _cuda(d["f"], torch.float32), _cuda(v0, torch.float64), 25)
    c = P.ipiano_config_default(max_iters=2)
    st = P.ipiano_state_create(md, _cuda(d["f"], torch.float32), d["lambdas"], L0, c)
    P.ipiano_solve(st)
    _, u = P.ipiano_get_iterate(st)
    u = u.cpu().numpy()
    tr = P.ipiano_get_trace(st)
    for b in (0, 37):
        l1, l2 = d["lambdas"][b]
        ref = oracle.ipiano_run(d["f"][b], d["filters"], d["theta"], l1, l2, oracle.make_cfg(L0[b], 2))
        assert rel_l2(u[b], ref["u"]) <= 1e-5
        np.testing.assert_array_equal(tr[b, 1:, 4], ref["trace"][1:, 4])


def test_tc_slabs_bitwise_g_invariant():
    H, W = 256, 96
    u0 = S.piecewise_smooth_scene(H, W, 11)
    f = S.add_speckle(u0, 1, 12)
    k, th = S.random_filter_bank(48, 7, 603)
    md = P.foe_model_create(k, th, lam=(160.0, 0.004))
    ft = _cuda(f, torch.float32)
    outs = []
    for G in (1, 2, 4):
        c = P.ipiano_config_default(max_iters=15, stencil=TENSOR)
        sl = P.ipiano_slabs_create(md, ft, H, nslabs=G, lam=(160.0, 0.004), lipschitz_init=2.0 ** 18, cfg=c)
        P.ipiano_slabs_solve(sl)
        w, _ = P.ipiano_slabs_get_iterate(sl, want_u=False)
        outs.append((w.cpu().numpy(), P.ipiano_get_trace(P.ipiano_slabs_member(sl, 0))[0]))
        sl.destroy()
    for w, tr in outs[1:]:
        np.testing.assert_array_equal(w, outs[0][0])
        np.testing.assert_array_equal(tr, outs[0][1])
    ref = oracle.ipiano_run(f, k, th, 160.0, 0.004, oracle.make_cfg(2.0 ** 18, 15))
    assert rel_l2(np.exp(outs[0][0]), ref["u"]) <= 1e-4


@pytest.mark.parametrize("rows", [8, 32])
@pytest.mark.parametrize("B,H,W", [(2, 300, 260), (1, 520, 512), (2, 256, 260), (1, 8, 300), (2, 256, 256),
                                   (1, 64, 128), (1, 8, 128)])
def test_tc_tile_rows_P3(rows, B, H, W):
    """K8 with forced tile heights (ipiano_config.tile_rows) against the oracle on batch shapes.
    Bands that tile H (and are >= 2C = 6 rows tall) run without row halos, and without column halos
    too when 128-column tiles tile W (the partial sums of the rows / columns near tile edges and the
    four-tile corners, incl. the periodic wrap, a single band H = 8, a single column tile W = 128 and
    a single tile, are added by the last tile to finish); the others (300 rows; 520 in 32-row
    bands; 8 rows in 32-row tiles) with halos and a short last band.
    Ragged and packed remainder columns (W = 512: the 24 remainder columns of several bands share
    one tile), every image of a batch.  P3 bars (final image rel L2 <= 1e-4, |dPSNR| <= 0.01 dB,
    identical L_n / trials, H trace to 1e-6) over 30 iterations."""
    cfg, d, L0 = _setup("c4", B=B, H=H, W=W, iters=30)
    md = P.foe_model_create(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]))
    c = P.ipiano_config_default(max_iters=cfg.iters, stencil=TENSOR, tile_rows=rows)
    st = P.ipiano_state_create(md, _cuda(d["f"], torch.float32), d["lambdas"], L0, c)
    P.ipiano_solve(st)
    _, u = P.ipiano_get_iterate(st)
    u = u.cpu().numpy()
    tr = P.ipiano_get_trace(st)
    cnt = P.ipiano_get_counters(st)
    for b in range(B):
        assert cnt["status"][b] == 0 and cnt["iters"][b] == cfg.iters
        l1, l2 = d["lambdas"][b]
        ref = oracle.ipiano_run(d["f"][b], d["filters"], d["theta"], l1, l2, oracle.make_cfg(L0[b], cfg.iters))
        assert ref["status"] == 0
        assert rel_l2(u[b], ref["u"]) <= 1e-4, (b, rel_l2(u[b], ref["u"]))
        clean = d["clean"][b]
        assert abs(oracle.psnr(u[b], clean) - oracle.psnr(ref["u"], clean)) <= 0.01
        np.testing.assert_array_equal(tr[b, 1:, 3], ref["trace"][1:, 3])
        np.testing.assert_array_equal(tr[b, 1:, 4], ref["trace"][1:, 4])
        np.testing.assert_allclose(tr[b, :, 2], ref["trace"][:, 2], rtol=1e-6)


def test_tc_tile_rows_invalid():
    k, th = S.random_filter_bank(48, 7, 5)
    md = P.foe_model_create(k, th, lam=(310.0, 0.008))
    f = _cuda(np.full((1, 64, 64), 50.0), torch.float32)
    with pytest.raises(P.FoeError) as e:
        P.ipiano_state_create(md, f, None, np.array([1.0]), P.ipiano_config_default(tile_rows=48))
    assert e.value.status == 1
