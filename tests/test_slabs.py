"""Row-slab decomposition of one scene (BASELINE.json configs[4]) on the GPU.

* G-invariance: the scene cut into 1, 2 or 4 row slabs (in-process slabs on one GPU, ghost
  rows moved by device copies) gives a bitwise identical iterate and trace.
* The NCCL transport (this rank's own communicator, nranks = 1: the ring exchanges with
  itself through ncclSend/ncclRecv) gives the same bits as the in-process path.
* Parity: the slab path against the fp64 oracle's whole-scene periodic run (final image
  relative L2 <= 1e-4, |dPSNR| <= 0.01 dB, identical L_n / trial decisions).
* c5 at full size (8192^2) in the slab launch configuration: 1 vs 4 slabs bitwise, and the
  slab path against the batch path for the first iterations.
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


def _scene(H, W, L=1, seed=7, sar=False):
    u = S.sar_like_scene(H, W, seed) if sar else S.piecewise_smooth_scene(H, W, seed)
    return u, S.add_speckle(u, L, seed + 1)


def _run_slabs(md, f, nslabs, L0, iters, comm=None, lam=(160.0, 0.004)):
    cfg = P.ipiano_config_default(max_iters=iters)
    H, W = f.shape
    ft = torch.as_tensor(f, device="cuda")
    sl = P.ipiano_slabs_create(md, ft, H, nslabs=nslabs, lam=lam, lipschitz_init=L0, cfg=cfg, comm=comm)
    P.ipiano_slabs_solve(sl)
    w, u = P.ipiano_slabs_get_iterate(sl)
    tr = P.ipiano_get_trace(P.ipiano_slabs_member(sl, 0))[0]
    cnt = P.ipiano_get_counters(P.ipiano_slabs_member(sl, 0))
    torch.cuda.synchronize()
    out = (w.cpu().numpy(), u.cpu().numpy(), tr, cnt)
    sl.destroy()
    return out


@pytest.fixture(scope="module")
def small_case():
    H, W = 256, 96
    clean, f = _scene(H, W, L=1, seed=11)
    k, th = S.random_filter_bank(48, 7, 603)
    md = P.foe_model_create(k, th, lam=(160.0, 0.004))
    v0 = S.lipschitz_start_vector(1, H, W)
    _, L0 = P.foe_estimate_lipschitz(md, torch.as_tensor(f[None], device="cuda"),
                                     torch.as_tensor(v0, device="cuda"), 25)
    return dict(H=H, W=W, clean=clean, f=f, k=k, th=th, md=md, L0=float(L0[0]))


def test_slab_g_invariance_bitwise(small_case):
    c = small_case
    runs = {G: _run_slabs(c["md"], c["f"], G, c["L0"], 25) for G in (1, 2, 4)}
    w1, u1, tr1, cnt1 = runs[1]
    assert cnt1["status"][0] == 0 and cnt1["iters"][0] == 25
    for G in (2, 4):
        w, u, tr, cnt = runs[G]
        np.testing.assert_array_equal(w, w1)
        np.testing.assert_array_equal(tr, tr1)
        assert cnt["trials"][0] == cnt1["trials"][0]


def test_slab_nccl_self_ring_matches_in_process(small_case):
    c = small_case
    comm = P.foe_comm_create(P.foe_comm_unique_id(), 1, 0, 0)
    try:
        w_n, u_n, tr_n, _ = _run_slabs(c["md"], c["f"], 1, c["L0"], 12, comm=comm)
    finally:
        comm.destroy()
    w_l, u_l, tr_l, _ = _run_slabs(c["md"], c["f"], 1, c["L0"], 12)
    np.testing.assert_array_equal(w_n, w_l)
    np.testing.assert_array_equal(tr_n, tr_l)


def test_slab_nccl_fused_p2p_self_ring(small_case):
    """The fused exchange (K2 stores its boundary rows straight into the ring neighbours' ghost
    buffers; here the 1-rank ring's neighbour is the slab itself) gives the same bits as the
    ncclSend/ncclRecv path and the in-process path."""
    c = small_case
    comm = P.foe_comm_create(P.foe_comm_unique_id(), 1, 0, 0)
    try:
        ft = torch.as_tensor(c["f"], device="cuda")
        sl = P.ipiano_slabs_create(c["md"], ft, c["H"], lam=(160.0, 0.004), lipschitz_init=c["L0"],
                                   cfg=P.ipiano_config_default(max_iters=12), comm=comm)
        h = P.ipiano_slabs_halo_handle(sl)
        assert len(h) == 64
        P.ipiano_slabs_connect_peers(sl, h, h)
        with pytest.raises(P.FoeError):
            P.ipiano_slabs_connect_peers(sl, h, h)           # only once
        P.ipiano_slabs_reset(sl, ft, c["L0"])                # re-init on the fused path
        P.ipiano_slabs_solve(sl)
        w_p, _ = P.ipiano_slabs_get_iterate(sl, want_u=False)
        tr_p = P.ipiano_get_trace(P.ipiano_slabs_member(sl, 0))[0]
        w_p = w_p.cpu().numpy()
        sl.destroy()
    finally:
        comm.destroy()
    w_l, _, tr_l, _ = _run_slabs(c["md"], c["f"], 1, c["L0"], 12)
    np.testing.assert_array_equal(w_p, w_l)
    np.testing.assert_array_equal(tr_p, tr_l)


def test_slab_parity_vs_oracle(small_case):
    """P3 on the slab path (2 slabs): free-running final image against the whole-scene oracle."""
    c = small_case
    iters = 40
    w, u, tr, cnt = _run_slabs(c["md"], c["f"], 2, c["L0"], iters)
    ref = oracle.ipiano_run(c["f"], c["k"], c["th"], 160.0, 0.004, oracle.make_cfg(c["L0"], iters))
    assert ref["status"] == 0
    assert rel_l2(u, ref["u"]) <= 1e-4
    assert abs(oracle.psnr(u, c["clean"]) - oracle.psnr(ref["u"], c["clean"])) <= 0.01
    np.testing.assert_array_equal(tr[1:, 3], ref["trace"][1:, 3])     # L_n
    np.testing.assert_array_equal(tr[1:, 4], ref["trace"][1:, 4])     # trials
    np.testing.assert_allclose(tr[:, 0], ref["trace"][:, 0], rtol=1e-6)  # F


def test_slab_matches_batch_path(small_case):
    """The slab path and the single-scene batch path solve the same problem (not bitwise:
    their reductions are grouped differently)."""
    c = small_case
    w, u, tr, _ = _run_slabs(c["md"], c["f"], 4, c["L0"], 20)
    ub, trb = P.ipiano_run(c["md"], torch.as_tensor(c["f"][None], device="cuda"), np.array([[160.0, 0.004]]),
                           np.array([c["L0"]]), P.ipiano_config_default(max_iters=20))
    assert rel_l2(u, ub.cpu().numpy()[0]) <= 1e-5
    np.testing.assert_array_equal(tr[1:, 4], trb[0, 1:, 4])


def test_slab_argument_errors(small_case):
    c = small_case
    ft = torch.as_tensor(c["f"], device="cuda")
    with pytest.raises(P.FoeError) as e:   # 256 rows cannot make 3 slabs of whole 64-row bands
        P.ipiano_slabs_create(c["md"], ft, c["H"], nslabs=3, lipschitz_init=c["L0"])
    assert e.value.status == 1
    with pytest.raises(P.FoeError) as e:
        P.ipiano_slabs_create(c["md"], ft[:, :90].contiguous(), c["H"], nslabs=1, lipschitz_init=c["L0"])
    assert e.value.status == 1 and "multiple of 32" in e.value.message
    with pytest.raises(P.FoeError) as e:
        P.ipiano_slabs_create(c["md"], ft, c["H"], nslabs=1, lipschitz_init=0.0)
    assert e.value.status == 1


def test_c5_full_size_slab_vs_batch_path():
    """c5 (8192^2 SAR-like, 48 x 7x7, L=1) at full size in the slab launch configuration the
    bench times (the whole scene as slabs on one GPU): 3 iterations of the slab path against
    the batch path (whose gradient is checked against the oracle on sampled pixels of this
    scene in test_gpu_parity.py), and bitwise equality of 1 vs 4 slabs."""
    cfg = S.config("c5")
    d = S.make_inputs(cfg)
    f = d["f"][0]
    lam = tuple(d["lambdas"][0])
    md = P.foe_model_create(d["filters"], d["theta"], lam=lam)
    ft = torch.as_tensor(f, device="cuda")
    L0 = 2.0 ** 18
    c3 = P.ipiano_config_default(max_iters=3)
    outs = {}
    for G in (1, 4):
        sl = P.ipiano_slabs_create(md, ft, cfg.H, nslabs=G, lam=lam, lipschitz_init=L0, cfg=c3)
        P.ipiano_slabs_solve(sl)
        _, u = P.ipiano_slabs_get_iterate(sl, want_w=False)
        cnt = P.ipiano_get_counters(P.ipiano_slabs_member(sl, 0))
        tr = P.ipiano_get_trace(P.ipiano_slabs_member(sl, 0))[0]
        assert cnt["status"][0] == 0 and cnt["iters"][0] == 3
        outs[G] = (u.cpu().numpy(), tr)
        sl.destroy()
    np.testing.assert_array_equal(outs[1][0], outs[4][0])
    np.testing.assert_array_equal(outs[1][1], outs[4][1])
    ub, trb = P.ipiano_run(md, ft[None].contiguous(), np.array([lam]), np.array([L0]), c3)
    assert rel_l2(outs[1][0], ub.cpu().numpy()[0]) <= 1e-6
    np.testing.assert_array_equal(outs[1][1][1:, 4], trb[0, 1:, 4])
    np.testing.assert_allclose(outs[1][1][:, 0], trb[0, :, 0], rtol=1e-9)
