"""Small cases for compute-sanitizer (profiles/r02_sanitizers.md):
  k8      one K8 tile (64 x 122, 48 x 7x7, tensor-core stencil) energy + gradient, and one HVP
  persist the persistent cooperative driver on a c1-shaped image, 5 iterations
  slabs   4 in-process row slabs of a 256 x 244 scene (K8, interior/boundary split), 3 iterations"""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import foe_synth as S  # noqa: E402
import paper_1404_5344_b200 as P  # noqa: E402

case = sys.argv[1]
if case == "k8":
    k, th = S.random_filter_bank(48, 7, 1)
    f = S.add_speckle(S.piecewise_smooth_scene(64, 122, 2), 3, 3)[None]
    w = torch.as_tensor(np.log(np.maximum(f.astype(np.float64), 1.0)), device="cuda")
    md = P.foe_model_create(k, th, lam=(310.0, 0.008))
    P.foe_model_set_stencil(md, P.FOE_STENCIL_TENSOR)
    F, _, g = P.foe_energy_grad(md, w)
    hv = P.foe_hvp(md, w, torch.randn_like(w))
    torch.cuda.synchronize()
    print("k8 ok", F[0], float(g.abs().max()), float(hv.abs().max()))
elif case == "persist":
    cfg = S.config("c1", iters=5)
    d = S.make_inputs(cfg)
    md = P.foe_model_create(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]))
    st = P.ipiano_state_create(md, torch.as_tensor(d["f"], device="cuda"), d["lambdas"], [2.0 ** 18],
                               P.ipiano_config_default(max_iters=5, solver=P.FOE_SOLVER_PERSISTENT))
    P.ipiano_solve(st)
    torch.cuda.synchronize()
    print("persistent ok", P.ipiano_get_counters(st)["iters"])
elif case == "slabs":
    k, th = S.random_filter_bank(48, 7, 603)
    f = S.add_speckle(S.sar_like_scene(256, 244, 5), 1, 6)
    md = P.foe_model_create(k, th, lam=(160.0, 0.004))
    sl = P.ipiano_slabs_create(md, torch.as_tensor(f, device="cuda"), 256, nslabs=4, lam=(160.0, 0.004),
                               lipschitz_init=2.0 ** 18,
                               cfg=P.ipiano_config_default(max_iters=3, stencil=P.FOE_STENCIL_TENSOR))
    P.ipiano_slabs_solve(sl)
    torch.cuda.synchronize()
    print("slabs ok", P.ipiano_get_counters(P.ipiano_slabs_member(sl, 0))["iters"])
