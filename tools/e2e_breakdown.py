#!/usr/bin/env python
"""Where the end-to-end ipiano_run time goes (c4 shape): state creation, init, solve, output,
destroy, host copies -- each bracketed by device synchronisation, wall-clock."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import foe_synth as S  # noqa: E402
import paper_1404_5344_b200 as P  # noqa: E402

cfg = S.config("c4")
d = S.make_inputs(cfg)
B, H, W = d["f"].shape
md = P.foe_model_create(d["filters"], d["theta"], lam=tuple(d["lambdas"][0]))
f_dev = torch.as_tensor(d["f"], device="cuda")
v0 = torch.as_tensor(S.lipschitz_start_vector(B, H, W), device="cuda")
_, L0 = P.foe_estimate_lipschitz(md, f_dev, v0, 25)
c = P.ipiano_config_default(max_iters=cfg.iters, record_trace=0)
f_pin = torch.empty((B, H, W), dtype=torch.float32, pin_memory=True); f_pin.copy_(torch.as_tensor(d["f"]))
u_pin = torch.empty((B, H, W), dtype=torch.float32, pin_memory=True)


def t(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    return r, 1e3 * (time.perf_counter() - t0)


for rep in range(3):
    _, t_run = t(lambda: P.ipiano_run(md, f_pin.numpy(), d["lambdas"], L0, c, u_out=u_pin.numpy(), want_trace=False))
    st, t_create = t(lambda: P.ipiano_state_create(md, f_dev, d["lambdas"], L0, c))
    _, t_solve = t(lambda: P.ipiano_solve(st))
    _, t_reset = t(lambda: P.ipiano_state_reset(st, f_dev, L0))
    _, t_solve2 = t(lambda: P.ipiano_solve(st))
    _, t_out = t(lambda: P.ipiano_get_iterate(st, want_w=False))
    _, t_destroy = t(lambda: st.destroy())
    print(f"rep {rep}: ipiano_run(host) {t_run:.1f} ms | create {t_create:.1f} solve {t_solve:.1f} reset {t_reset:.1f} "
          f"solve(again) {t_solve2:.1f} out {t_out:.1f} destroy {t_destroy:.1f} ms", flush=True)
