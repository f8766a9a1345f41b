import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import foe_synth as S, oracle, paper_1404_5344_b200 as P
H, W, nf = 70, 90, 24
k, th = S.random_filter_bank(nf, 7, 6)
f = S.add_speckle(S.piecewise_smooth_scene(H, W, 3), 1, 4)[None]
w = np.log(np.maximum(f.astype(np.float64), 1.0))
md = P.foe_model_create(k, th, lam=(310.0, 0.008))
for name, v in [("zero", np.zeros_like(w)), ("ones", np.ones_like(w)), ("randn", np.random.default_rng(0).standard_normal(w.shape))]:
    hv = P.foe_hvp(md, torch.as_tensor(w, device="cuda"), torch.as_tensor(v, device="cuda")).cpu().numpy()[0]
    ho = oracle.hvp_w(w[0], v[0], k, th)
    bad = ~np.isfinite(hv)
    fin = np.argwhere(~bad)
    print(name, "nan", bad.sum(), "finite at", fin[:8].tolist(), "rel", np.linalg.norm((hv-ho)[~bad]) / max(np.linalg.norm(ho[~bad]), 1e-30))
    print("   sample hv", hv[0, :5], "ho", ho[0, :5])
mdu = P.foe_model_create(k, th, lam=(0.01, 0.0), term=P.FOE_DATA_IDIV)
u = np.maximum(f.astype(np.float64), 1.0)
v = np.random.default_rng(0).standard_normal(w.shape)
hv = P.foe_hvp(mdu, torch.as_tensor(u, device="cuda"), torch.as_tensor(v, device="cuda")).cpu().numpy()[0]
print("udom nan", (~np.isfinite(hv)).sum())
