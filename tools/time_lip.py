import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import foe_synth as S, paper_1404_5344_b200 as P
cfg = S.config("c4"); d = S.make_inputs(cfg)
md = P.foe_model_create(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]))
f = torch.as_tensor(d["f"], device="cuda"); v0 = torch.as_tensor(S.lipschitz_start_vector(cfg.B, cfg.H, cfg.W), device="cuda")
w = torch.log(torch.clamp(f.double(), min=1.0)); v = torch.randn_like(w)
for it in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    rho, L = P.foe_estimate_lipschitz(md, f, v0, 25)
    torch.cuda.synchronize(); print("lipschitz", it, (time.perf_counter() - t) * 1e3, "ms")
for it in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    hv = P.foe_hvp(md, w, v)
    torch.cuda.synchronize(); print("hvp", it, (time.perf_counter() - t) * 1e3, "ms")
for it in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    F, _, g = P.foe_energy_grad(md, w)
    torch.cuda.synchronize(); print("grad", it, (time.perf_counter() - t) * 1e3, "ms")
