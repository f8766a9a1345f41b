"""The data-term protocol of the paper's Fig. 2 (Sec. III-A) on seeded synthetic
data, on the GPU: one image corrupted with L = 8 speckle, restored by

  model (8)   Nakagami data term, lambda_2 = 0         (FOE_DATA_NAKAGAMI)
  model (6)   I-divergence data term, iterate in u     (FOE_DATA_IDIV)
  model (10)  the combined model                       (FOE_DATA_COMBINED)

each with its lambda picked from a small grid by the best PSNR against the clean scene ("We
carefully tuned the parameter lambda"; the paper prints none for (6) and
hand-tuned (lambda_1, lambda_2) for (10)), and PSNR / SSIM measured by the
library's own kernels (foe_psnr / foe_ssim).  The paper's learned filter bank and test image are
not available: the bank is the seeded 48 x 7x7 random bank of the configs, so the
numbers are this build's, not the paper's 29.30 / 28.40 / 29.62 dB.  GPU only: the oracle
comparison of the chosen runs is tests/test_fig2_protocol.py.
"""
from __future__ import annotations

import numpy as np

import foe_synth as S

from . import foe as P

LOOKS = 8
SCALES = (0.25, 0.5, 1.0, 2.0, 4.0)


def inputs(H: int = 512, W: int = 512, seed: int = 901):
    """Clean piecewise-smooth scene, L = 8 speckle, the 48 x 7x7 bank of c2-c5 (seed 403)."""
    clean = S.piecewise_smooth_scene(H, W, seed)
    f = S.add_speckle(clean, LOOKS, seed + 1)
    k, th = S.random_filter_bank(48, 7, 403)
    return clean.astype(np.float32), f.astype(np.float32), k, th


def grid(model: str):
    """lambda candidates per model: (lambda_1, lambda_2) pairs; the presets of L = 8 scaled."""
    l1, l2 = S.LAMBDA_PRESETS[LOOKS]
    if model == "(8)":
        return [(l1 * s, 0.0) for s in SCALES]
    if model == "(6)":   # reading R-18's lambda sits at the grid's top: (6) wants more smoothing here
        return [(S.idiv_lambda(LOOKS) * s, 0.0) for s in (1 / 256, 1 / 64, 1 / 16, 1 / 4, 1.0)]
    return [(l1 * a, l2 * b) for a in (0.5, 1.0, 2.0) for b in (0.25, 1.0, 4.0)]


TERMS = {"(8)": P.FOE_DATA_NAKAGAMI, "(6)": P.FOE_DATA_IDIV, "(10)": P.FOE_DATA_COMBINED}


def run(iters: int = 300, H: int = 512, W: int = 512, device: int = 0):
    """Returns dict(noisy=(psnr, ssim), models={name: dict(lam, L0, psnr, ssim, u, grid)})."""
    import torch
    clean, f, k, th = inputs(H, W)
    dev = torch.device("cuda", device)
    fd = torch.as_tensor(f[None], device=dev)
    cd = torch.as_tensor(clean[None], device=dev)
    v0 = torch.as_tensor(S.lipschitz_start_vector(1, H, W), device=dev)
    out = {"noisy": (float(P.foe_psnr(fd, cd)[0]), float(P.foe_ssim(fd, cd)[0])), "models": {},
           "image": f"{H}x{W} piecewise-smooth (seed 901), L = {LOOKS}, 48 x 7x7 random bank (seed 403), "
                    f"{iters} iPiano iterations"}
    for name, term in TERMS.items():
        best = None
        rows = []
        for lam in grid(name):
            md = P.foe_model_create(k, th, lam=lam, term=term, device=device)
            _, L0 = P.foe_estimate_lipschitz(md, fd, v0, 25)
            cfg = P.ipiano_config_default(max_iters=iters)
            u, _ = P.ipiano_run(md, fd, np.array([lam]), L0, cfg, want_trace=False)
            ps, ss = float(P.foe_psnr(u, cd)[0]), float(P.foe_ssim(u, cd)[0])
            rows.append((lam, ps, ss))
            if best is None or ps > best["psnr"]:
                best = dict(lam=lam, L0=float(L0[0]), psnr=ps, ssim=ss, u=u.cpu().numpy()[0])
            md.destroy()
        best["grid"] = rows
        out["models"][name] = best
    return out
