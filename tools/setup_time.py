"""Where the e2e-with-setup leg's time goes on c4: foe_estimate_lipschitz alone, ipiano_run
(host buffers) alone, and the two back to back, wall clock around device syncs."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import foe_synth as S
import paper_1404_5344_b200 as P

cfg = S.config("c4")
d = S.make_inputs(cfg)
B, H, W = d["f"].shape
md = P.foe_model_create(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]))
f_dev = torch.as_tensor(d["f"], device="cuda")
v0 = torch.as_tensor(S.lipschitz_start_vector(B, H, W), device="cuda")
c = P.ipiano_config_default(max_iters=cfg.iters, record_trace=0)
f_pin = torch.empty((B, H, W), dtype=torch.float32, pin_memory=True); f_pin.copy_(torch.as_tensor(d["f"]))
u_pin = torch.empty((B, H, W), dtype=torch.float32, pin_memory=True)
f_np, u_np = f_pin.numpy(), u_pin.numpy()


def t(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    return r, 1e3 * (time.perf_counter() - t0)


for rep in range(3):
    (_, L0), a = t(lambda: P.foe_estimate_lipschitz(md, f_dev, v0, 25))
    _, b = t(lambda: P.ipiano_run(md, f_np, d["lambdas"], L0, c, u_out=u_np, want_trace=False))
    def both():
        _, L = P.foe_estimate_lipschitz(md, f_dev, v0, 25)
        P.ipiano_run(md, f_np, d["lambdas"], L, c, u_out=u_np, want_trace=False)
    _, e = t(both)
    print(f"lipschitz {a:.1f} ms, ipiano_run {b:.1f} ms, both {e:.1f} ms", flush=True)
