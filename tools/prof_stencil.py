#!/usr/bin/env python
"""Time one prior energy+gradient evaluation (K1 or K8) on a c4-size batch with CUDA events,
and check the two stencils against each other.  Small enough to run under ncu:

    python tools/prof_stencil.py [--stencil tensor|ffma|both] [--batch 64] [--reps 5]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import foe_synth as S  # noqa: E402
import paper_1404_5344_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--stencil", default="both", choices=["tensor", "ffma", "both"])
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--size", type=int, default=512)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()

k, th = S.random_filter_bank(48, 7, 403)
B, n = a.batch, a.size
f = np.stack([S.add_speckle(S.piecewise_smooth_scene(n, n, 400 + i), 8, 500 + i) for i in range(min(B, 4))])
f = np.concatenate([f] * ((B + 3) // 4))[:B]
w = torch.as_tensor(np.log(np.maximum(f.astype(np.float64), 1.0)), device="cuda")
md = P.foe_model_create(k, th, lam=(550.0, 0.02))
out = {}
for name, sid in (("ffma", P.FOE_STENCIL_FFMA), ("tensor", P.FOE_STENCIL_TENSOR)):
    if a.stencil not in (name, "both"):
        continue
    P.foe_model_set_stencil(md, sid)
    F, _, g = P.foe_energy_grad(md, w)
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); P.foe_energy_grad(md, w, prior=False); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    tf = 4.0 * 48 * 49 * B * n * n / (ms / 1e3) / 1e12
    print(f"{name}: {ms:.3f} ms per evaluation (incl. alloc), {tf:.1f} TFLOP/s algorithmic, "
          f"{tf / 74.45:.3f} of FP32 peak; F[0]={F[0]:.10e}")
    out[name] = (F, g.cpu().numpy())
if len(out) == 2:
    gt, gf = out["tensor"][1], out["ffma"][1]
    print("rel L2(K8 - K1) =", float(np.linalg.norm(gt - gf) / np.linalg.norm(gf)))
