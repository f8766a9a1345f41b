#!/usr/bin/env python
"""A/B of the two K8 variants in one process: device time of one prior evaluation (64 x 512^2,
48 x 7x7), CUDA events around the kernel-only foe_energy_grad call, interleaved, min and median."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import foe_synth as S  # noqa: E402
import paper_1404_5344_b200 as P  # noqa: E402

k, th = S.random_filter_bank(48, 7, 403)
B, n = 64, 512
f = np.stack([S.add_speckle(S.piecewise_smooth_scene(n, n, 400 + i), 8, 500 + i) for i in range(4)])
f = np.concatenate([f] * 16)[:B]
w = torch.as_tensor(np.log(np.maximum(f.astype(np.float64), 1.0)), device="cuda")
md = P.foe_model_create(k, th, lam=(550.0, 0.02))
P.foe_model_set_stencil(md, P.FOE_STENCIL_TENSOR)
VARS = sys.argv[1].split(",") if len(sys.argv) > 1 else ["3", "4"]
res = {v: [] for v in VARS}
g = {}
for it in range(12):
    for v in VARS:
        os.environ["FOE_K8_VARIANT"] = v
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); _, _, gg = P.foe_energy_grad(md, w); e1.record(); e1.synchronize()
        if it > 1:
            res[v].append(e0.elapsed_time(e1))
        g[v] = gg
for v in VARS:
    print(f"K8 v{v}: min {min(res[v]):.3f} ms, median {statistics.median(res[v]):.3f} ms")
if "3" in g and "4" in g:
    a, b = g["3"].cpu().numpy(), g["4"].cpu().numpy()
    print("v3 vs v4 gradient max |diff|", float(np.abs(a - b).max()), "bitwise" if np.array_equal(a, b) else "")
