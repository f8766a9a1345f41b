"""c4 Lipschitz setup (R-10) alone: warm call + timed calls (run under ncu --metrics
gpu__time_duration.sum for the per-kernel breakdown of foe_estimate_lipschitz)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import foe_synth as S
import paper_1404_5344_b200 as P

cfg = S.config("c4")
d = S.make_inputs(cfg)
B, H, W = d["f"].shape
md = P.foe_model_create(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]), device=0)
f = torch.as_tensor(d["f"], device="cuda:0")
v0 = torch.as_tensor(S.lipschitz_start_vector(B, H, W), device="cuda:0")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
s = torch.cuda.current_stream()
ts = []
for k in range(n):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    rho, L0 = P.foe_estimate_lipschitz(md, f, v0, 25)
    e1.record(s); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
print("lipschitz ms", [round(t, 2) for t in ts], "L0[:4]", list(L0[:4]))
