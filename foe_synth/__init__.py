"""Seeded synthetic inputs for the FoE/iPiano despeckling hot path.

This module is the ONLY code shared by the CPU oracle (`oracle/`) and the CUDA
path (`paper_1404_5344_b200/`).  It holds no arithmetic of the method itself
(no convolution, potential, prox, or iPiano step): only

  * the seeded scene generators that stand in for the paper's missing test
    images (Couple/Lenna/Peppers 256x256, Berkeley-68 481x321, the JSTARS SAR
    scene -- PAPER.md:262, :314-315, :388),
  * the speckle simulator that produces the observation f (amplitude model,
    PAPER.md:113-121 Nakagami likelihood),
  * the seeded zero-mean unit-norm filter bank and weights theta_i > 0 that
    stand in for the learned 48 x 7x7 bank (which is not
    published),
  * the lambda presets per number of looks,
  * the five BASELINE.json configurations and the iPiano policy constants
    (DESIGN.md "Readings"), and
  * the random start vector of the Lipschitz power iteration (a random draw the
    method makes, so it is passed to both sides as an input).

Every generator uses numpy ``Generator(PCG64(seed))`` so the oracle and the GPU
path see bit-identical fp32 inputs.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "LAMBDA_PRESETS", "IDIV_U_RMS", "idiv_lambda", "POLICY", "Config", "CONFIGS", "config", "rng",
    "piecewise_smooth_scene", "sar_like_scene", "add_speckle",
    "random_filter_bank", "dct_filter_bank", "lipschitz_start_vector",
    "make_inputs",
]

# PAPER.md:272-274 (Sec. III-B): "if L = 8, lambda_1 = 550, lambda_2 = 0.02; if L = 3,
# lambda_1 = 310, lambda_2 = 0.008; and if L = 1, lambda_1 = 160, lambda_2 = 0.004".
# PAPER.md:389 (Sec. III-C, real SAR, L = 5): "lambda_1 = 50, lambda_2 = 0.15".
LAMBDA_PRESETS: Dict[int, Tuple[float, float]] = {
    1: (160.0, 0.004),
    3: (310.0, 0.008),
    5: (50.0, 0.15),
    8: (550.0, 0.02),
}

# Variant model (6) (I-divergence): the paper tuned lambda by hand and
# prints none.  Reading R-18: lambda = lambda_1 / u_rms^2, which gives Eq.(5)
# the curvature of model (8)'s data term at u = f = u_rms; u_rms = 120.4 is the clean RMS that
# reproduces Table II's noisy PSNR row (reading R-14).
IDIV_U_RMS = 120.4


def idiv_lambda(L: int) -> float:
    return LAMBDA_PRESETS[L][0] / (IDIV_U_RMS * IDIV_U_RMS)


# iPiano step policy used for every graded configuration (reading R-9):
# doubling backtracking, L never shrinks, beta = 0.4, safety 0.95
# ("alpha = 0.95 * 2(1-beta)/L_n"), L_init = 2^ceil(log2 rho_hat) from
# 25 power-iteration steps on the prior Hessian at w^0 (reading R-10).
POLICY = dict(
    beta=0.4,
    step_safety=0.95,
    backtrack_factor=2.0,
    shrink=1.0,
    max_backtracks=60,
    newton_max_iters=30,
    rel_change_tol=0.0,         # benchmarks run exactly max_iters (reading R-12)
    power_iters=25,
    power_seed=3,
)


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(int(seed)))


# --------------------------------------------------------------------------------------
# Scenes
# --------------------------------------------------------------------------------------

def piecewise_smooth_scene(H: int, W: int, seed: int, n_shapes: int = 30) -> np.ndarray:
    """Piecewise-smooth clean amplitude scene in [1, 255] (fp32, [H][W]).

    Recipe: a background level U[40,200] with a linear
    ramp, then ``n_shapes`` axis-aligned rectangles or ellipses (50/50), each with
    a base value U[1,255] plus a linear ramp of slope U[-2,2] per pixel (scaled by
    128/max(H,W) so that larger images keep the same look), clipped to [1,255].
    The value range follows SPEC.md:151 (native 8-bit amplitude scale).
    """
    g = rng(seed)
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    s = 128.0 / max(H, W)
    base = g.uniform(40.0, 200.0)
    gy, gx = g.uniform(-0.5, 0.5, 2) * s
    img = base + gy * (yy - H / 2.0) + gx * (xx - W / 2.0)
    for _ in range(n_shapes):
        kind = g.integers(0, 2)
        cy, cx = g.uniform(0, H), g.uniform(0, W)
        hy, hx = g.uniform(0.04, 0.25) * H, g.uniform(0.04, 0.25) * W
        val = g.uniform(1.0, 255.0)
        sy, sx = g.uniform(-2.0, 2.0, 2) * s
        if kind == 0:
            mask = (np.abs(yy - cy) <= hy) & (np.abs(xx - cx) <= hx)
        else:
            mask = ((yy - cy) / hy) ** 2 + ((xx - cx) / hx) ** 2 <= 1.0
        img = np.where(mask, val + sy * (yy - cy) + sx * (xx - cx), img)
    return np.clip(img, 1.0, 255.0).astype(np.float32)


def _gaussian_blur_periodic(x: np.ndarray, sigma: float) -> np.ndarray:
    """Periodic Gaussian blur via FFT (input synthesis only, not the method)."""
    H, W = x.shape
    fy = np.fft.fftfreq(H)[:, None]
    fx = np.fft.rfftfreq(W)[None, :]
    kern = np.exp(-2.0 * (np.pi * sigma) ** 2 * (fy ** 2 + fx ** 2))
    return np.fft.irfft2(np.fft.rfft2(x) * kern, s=(H, W))


def sar_like_scene(H: int, W: int, seed: int, n_regions: int = 400,
                   target_density: float = 1e-5) -> np.ndarray:
    """SAR-like clean amplitude scene (stand-in for the JSTARS image).

    Recipe: a jittered-grid Voronoi partition with about ``n_regions`` cells (sharp
    edges); per region a log-normal texture exp(mu_r + sigma_r * S) with
    mu_r ~ U[log 20, log 150], sigma_r ~ U[0.1, 0.5], S a unit-variance Gaussian
    field blurred with sigma = 3 px; sparse 3x3 point targets set to 255 at density
    ``target_density``; clipped to [1, 255].  Returns fp32 [H][W].
    """
    g = rng(seed)
    ng = max(1, int(round(np.sqrt(n_regions * H / W))))
    nx = max(1, int(round(n_regions / ng)))
    cell_h, cell_w = H / ng, W / nx
    sy = (np.arange(ng)[:, None] + g.uniform(0.1, 0.9, (ng, nx))) * cell_h
    sx = (np.arange(nx)[None, :] + g.uniform(0.1, 0.9, (ng, nx))) * cell_w
    n_cells = ng * nx
    mu = g.uniform(np.log(20.0), np.log(150.0), n_cells)
    sig = g.uniform(0.1, 0.5, n_cells)
    S = g.standard_normal((H, W))
    S = _gaussian_blur_periodic(S, 3.0)
    S /= S.std()
    out = np.empty((H, W), np.float32)
    xs = np.arange(W, dtype=np.float64)
    block = max(1, int(4_000_000 // max(W, 1)))
    for y0 in range(0, H, block):
        y1 = min(H, y0 + block)
        yy = np.arange(y0, y1, dtype=np.float64)[:, None] + 0.5
        xx = xs[None, :] + 0.5
        cy = np.clip((yy // cell_h).astype(np.int64), 0, ng - 1)
        cx = np.clip((xx // cell_w).astype(np.int64), 0, nx - 1)
        best = np.full((y1 - y0, W), np.inf)
        lab = np.zeros((y1 - y0, W), np.int64)
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                ny = np.clip(cy + dy, 0, ng - 1)
                nxx = np.clip(cx + dx, 0, nx - 1)
                d = (sy[ny, nxx] - yy) ** 2 + (sx[ny, nxx] - xx) ** 2
                better = d < best
                best = np.where(better, d, best)
                lab = np.where(better, ny * nx + nxx, lab)
        out[y0:y1] = np.exp(mu[lab] + sig[lab] * S[y0:y1])
    n_t = int(round(target_density * H * W))
    ty = g.integers(1, max(2, H - 1), n_t)
    tx = g.integers(1, max(2, W - 1), n_t)
    for y, x in zip(ty, tx):
        out[max(0, y - 1):y + 2, max(0, x - 1):x + 2] = 255.0
    return np.clip(out, 1.0, 255.0).astype(np.float32)


# --------------------------------------------------------------------------------------
# Speckle (observation model)
# --------------------------------------------------------------------------------------

def add_speckle(u: np.ndarray, looks: float, seed: int) -> np.ndarray:
    """Amplitude speckle f = u * sqrt(s), s ~ Gamma(shape L, scale 1/L) (mean 1).

    PAPER.md:113-121 (Sec. II-B): f given u is Nakagami with L looks; f/u then is
    Nakagami(L, 1), i.e. (f/u)^2 ~ Gamma(L, 1/L) ("number of independent values
    averaged").  SPEC.md:343 states the same construction.  DESIGN.md reading R-14
    pins the amplitude reading against Table II's noisy PSNR row.
    """
    s = rng(seed).gamma(float(looks), 1.0 / float(looks), size=np.shape(u))
    return (np.asarray(u, np.float64) * np.sqrt(s)).astype(np.float32)


# --------------------------------------------------------------------------------------
# Filter banks
# --------------------------------------------------------------------------------------

def random_filter_bank(n_filters: int, m: int, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    """Seeded stand-in for the learned FoE bank (Fig. 1).

    Gaussian m x m taps, mean removed and scaled to unit Frobenius norm in fp64,
    then rounded to fp32 (so sum(k) is ~1e-8, not exactly 0 -- reading R-15).
    Weights theta_i ~ U[0.1, 1] (> 0 as PAPER.md:92 requires).
    Returns (filters fp32 [n][m][m], theta fp32 [n]).
    """
    g = rng(seed)
    k = g.standard_normal((n_filters, m, m))
    k -= k.mean(axis=(1, 2), keepdims=True)
    k /= np.sqrt((k ** 2).sum(axis=(1, 2), keepdims=True))
    theta = g.uniform(0.1, 1.0, n_filters)
    return k.astype(np.float32), theta.astype(np.float32)


def dct_filter_bank(m: int, count: int) -> Tuple[np.ndarray, np.ndarray]:
    """Non-DC 2-D DCT-II basis, unit norm, unit weights (SPEC.md:44-52 substitute bank)."""
    if m < 3 or m % 2 == 0:
        raise ValueError("m must be odd and >= 3")
    if count > m * m - 1:
        raise ValueError(f"only {m*m-1} non-constant kernels exist for m={m}")
    n = np.arange(m)
    C = np.cos(np.pi * (n[None, :] + 0.5) * n[:, None] / m)  # C[freq][pos]
    out = []
    for s in range(2 * m - 1):  # order by total frequency, then by row frequency
        for p in range(m):
            q = s - p
            if 0 <= q < m and (p, q) != (0, 0):
                k = np.outer(C[p], C[q])
                out.append(k / np.sqrt((k ** 2).sum()))
    bank = np.stack(out[:count]).astype(np.float32)
    return bank, np.ones(count, np.float32)


def lipschitz_start_vector(B: int, H: int, W: int, seed: int = 3) -> np.ndarray:
    """Random start v_0 ~ N(0, I) for the power iteration (reading R-10); fp64 [B][H][W].

    The method draws this vector, so it is an input passed to both sides.
    """
    return rng(seed).standard_normal((B, H, W))


# --------------------------------------------------------------------------------------
# BASELINE.json configurations
# --------------------------------------------------------------------------------------

@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    H: int
    W: int
    B: int
    n_filters: int
    m: int
    iters: int
    scene: str                  # "piecewise" | "sar"
    scene_seeds: Tuple[int, ...]
    speckle_seeds: Tuple[int, ...]
    looks: Tuple[int, ...]
    bank_seed: int
    description: str = ""

    @property
    def pixels(self) -> int:
        return self.B * self.H * self.W


def _c4_looks() -> Tuple[int, ...]:
    return tuple(int(v) for v in rng(499).choice(np.array([1, 3, 8]), 64))


CONFIGS: Dict[str, Config] = {
    "c1": Config("c1", 128, 128, 1, 24, 5, 100, "piecewise", (101,), (102,), (1,), 103,
                 "BASELINE.json configs[0]: 128^2, L=1, 24 x 5x5, 100 it"),
    "c2": Config("c2", 256, 256, 1, 48, 7, 200, "piecewise", (201,), (202,), (3,), 203,
                 "BASELINE.json configs[1]: 256^2, L=3, 48 x 7x7, 200 it"),
    "c3": Config("c3", 512, 512, 1, 48, 7, 300, "piecewise", (301,), (302,), (8,), 303,
                 "BASELINE.json configs[2]: 512^2, L=8, 48 x 7x7, 300 it"),
    "c4": Config("c4", 512, 512, 64, 48, 7, 300, "piecewise",
                 tuple(400 + i for i in range(64)), tuple(500 + i for i in range(64)),
                 _c4_looks(), 403,
                 "BASELINE.json configs[3]: 64 x 512^2, L in {1,3,8}, 48 x 7x7, 300 it"),
    "c5": Config("c5", 8192, 8192, 1, 48, 7, 300, "sar", (601,), (602,), (1,), 603,
                 "BASELINE.json configs[4]: 8192^2 SAR-like, L=1, 48 x 7x7, 300 it"),
}


def config(name: str, **overrides) -> Config:
    return dataclasses.replace(CONFIGS[name], **overrides)


def make_inputs(cfg: Config, images: Optional[Sequence[int]] = None) -> dict:
    """Materialise the seeded inputs of ``cfg``.

    ``images`` selects a subset of image indices (for c4 shards / samples); image i
    always gets the same scene/speckle seeds regardless of the subset, so an
    image's inputs do not depend on how the batch is sharded.  For indices beyond
    the configured batch (weak-scaling replicas) the seeds continue the pattern
    (scene seed 400+i, speckle 500+i... for c4) and looks cycle through the list.
    """
    idx = list(range(cfg.B)) if images is None else list(images)
    clean, noisy, looks, lam = [], [], [], []
    for i in idx:
        j = i % len(cfg.scene_seeds)
        extra = (i // len(cfg.scene_seeds)) * 1000
        sseed = cfg.scene_seeds[j] + extra
        nseed = cfg.speckle_seeds[j] + extra
        L = cfg.looks[i % len(cfg.looks)]
        if cfg.scene == "piecewise":
            u = piecewise_smooth_scene(cfg.H, cfg.W, sseed)
        else:
            u = sar_like_scene(cfg.H, cfg.W, sseed)
        clean.append(u)
        noisy.append(add_speckle(u, L, nseed))
        looks.append(L)
        lam.append(LAMBDA_PRESETS[L])
    filters, theta = random_filter_bank(cfg.n_filters, cfg.m, cfg.bank_seed)
    return dict(
        clean=np.stack(clean), f=np.stack(noisy), filters=filters, theta=theta,
        looks=np.array(looks, np.int64), lambdas=np.array(lam, np.float64),
        images=np.array(idx, np.int64), cfg=cfg,
    )
