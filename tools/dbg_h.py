import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import foe_synth as S, oracle
import paper_1404_5344_b200 as P
k, th = S.random_filter_bank(48, 7, 2100)
H, W = 64, 122
rng = np.random.default_rng(1)
f = S.add_speckle(S.piecewise_smooth_scene(H, W, 60), 3, 70)
w = np.log(np.maximum(f.astype(np.float64), 1.0))
for name, wv in [("const", np.full((H, W), 3.0)), ("scene", w), ("ramp", 3.0 + 0.001 * np.arange(W)[None, :] + 0 * w)]:
    res = {}
    for tf in ("0", "1"):
        os.environ["FOE_K8_TF32"] = tf
        md = P.foe_model_create(k, th, lam=(310.0, 0.008))
        P.foe_model_set_stencil(md, P.FOE_STENCIL_TENSOR)
        Fg, _, g = P.foe_energy_grad(md, torch.as_tensor(wv[None], device="cuda"))
        res[tf] = (Fg[0], g.cpu().numpy()[0])
    Fo, go = oracle.energy_grad_w(wv, k, th)
    for tf in ("0", "1"):
        F, g = res[tf]
        print(name, "tf32" if tf == "1" else "fp16", "F", F, "Fo", Fo, "grad relL2", np.linalg.norm(g - go) / max(np.linalg.norm(go), 1e-30),
              "gmax", np.abs(g).max(), "gomax", np.abs(go).max())
    g = res["0"][1]
    err = np.abs(g - go)
    print("  worst rows", np.argsort(err.max(1))[-5:], "worst cols", np.argsort(err.max(0))[-5:])
    print("  row err", np.round(err.max(1)[:12], 3))
    print("  col err", np.round(err.max(0)[:20], 3))
