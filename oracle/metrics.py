"""Oracle tier for SURVEY.md 8(f) f4's evaluation and synthesis kernels (TEST INFRASTRUCTURE ONLY;
only tests/, __graft_entry__.smoke() and bench.py's oracle legs may import this module).

* PSNR and SSIM as SPEC.md:394-420 defines them (PSNR 10 log10(peak^2 / MSE); SSIM = mean local
  SSIM with an 11 x 11 Gaussian window, sigma 1.5, K1 = 0.01, K2 = 0.03, on the valid region,
  Wang et al. as cited by PAPER.md Sec. III).  fp64, plain numpy.
* Counter-based speckle synthesis: the amplitude model f = u sqrt(s), s ~ Gamma(L, 1/L) (reading
  R-14), with the Gamma variate drawn by Marsaglia-Tsang's method from a
  Philox4x32-10 counter-based stream (Salmon et al. 2011): pixel p, attempt k uses the counter
  (p mod 2^32, p div 2^32, k, 0) under the key (seed mod 2^32, seed div 2^32).  The CUDA side
  implements the same generator independently (paper_1404_5344_b200/csrc), so both sides draw
  the same numbers without sharing code.
"""
from __future__ import annotations

import math

import numpy as np

# ------------------------------------------------------------------------------- metrics


def psnr(x, ref, peak: float = 255.0) -> float:
    """10 log10(peak^2 / MSE), +inf when MSE = 0."""
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    mse = float(np.mean((x - ref) ** 2))
    return math.inf if mse == 0.0 else 10.0 * math.log10(peak * peak / mse)


def gaussian_window(size: int = 11, sigma: float = 1.5) -> np.ndarray:
    """Normalised 1-D Gaussian of the SSIM window (the 2-D window is its outer product)."""
    r = np.arange(size, dtype=np.float64) - (size - 1) / 2.0
    g = np.exp(-(r * r) / (2.0 * sigma * sigma))
    return g / g.sum()


def ssim(x, ref, peak: float = 255.0, size: int = 11, sigma: float = 1.5, k1: float = 0.01,
         k2: float = 0.03) -> float:
    """mean of the local SSIM map over the valid region (every full window).

    Local statistics by explicit windowed sums (the 2-D Gaussian window w, sum w = 1):
      mu_x = sum w x, sigma_x^2 = sum w x^2 - mu_x^2, sigma_xy = sum w x y - mu_x mu_y,
      SSIM = (2 mu_x mu_y + C1)(2 sigma_xy + C2) / ((mu_x^2 + mu_y^2 + C1)(sigma_x^2 + sigma_y^2 + C2)).
    """
    x = np.asarray(x, np.float64)
    y = np.asarray(ref, np.float64)
    H, W = x.shape
    if H < size or W < size:
        raise ValueError("image smaller than the SSIM window")
    g = gaussian_window(size, sigma)
    w2 = np.outer(g, g)
    c1 = (k1 * peak) ** 2
    c2 = (k2 * peak) ** 2
    oh, ow = H - size + 1, W - size + 1
    # windows as a strided view: [oh][ow][size][size]
    sx = np.lib.stride_tricks.sliding_window_view(x, (size, size))
    sy = np.lib.stride_tricks.sliding_window_view(y, (size, size))
    mx = np.einsum("ijab,ab->ij", sx, w2)
    my = np.einsum("ijab,ab->ij", sy, w2)
    vx = np.einsum("ijab,ab->ij", sx * sx, w2) - mx * mx
    vy = np.einsum("ijab,ab->ij", sy * sy, w2) - my * my
    cxy = np.einsum("ijab,ab->ij", sx * sy, w2) - mx * my
    smap = (2 * mx * my + c1) * (2 * cxy + c2) / ((mx * mx + my * my + c1) * (vx + vy + c2))
    assert smap.shape == (oh, ow)
    return float(smap.mean())


# ------------------------------------------------------------------- Philox4x32-10 + Gamma

PHILOX_M0, PHILOX_M1 = 0xD2511F53, 0xCD9E8D57
PHILOX_W0, PHILOX_W1 = 0x9E3779B9, 0xBB67AE85
MASK32 = 0xFFFFFFFF


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32 with 10 rounds on uint32 numpy arrays (broadcast), Salmon et al. (SC'11):
    round: (hi0, lo0) = M0 * c0, (hi1, lo1) = M1 * c2,
           (c0, c1, c2, c3) <- (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0);  key += (W0, W1)."""
    c0, c1, c2, c3 = (np.asarray(v, np.uint64) for v in (c0, c1, c2, c3))
    k0 = np.asarray(k0, np.uint64)
    k1 = np.asarray(k1, np.uint64)
    for r in range(10):
        p0 = np.uint64(PHILOX_M0) * c0
        p1 = np.uint64(PHILOX_M1) * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & np.uint64(MASK32)
        hi1, lo1 = p1 >> np.uint64(32), p1 & np.uint64(MASK32)
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        if r < 9:
            k0 = (k0 + np.uint64(PHILOX_W0)) & np.uint64(MASK32)
            k1 = (k1 + np.uint64(PHILOX_W1)) & np.uint64(MASK32)
    return tuple(v.astype(np.uint32) for v in (c0, c1, c2, c3))


def _u01(w):
    """(w + 0.5) 2^-32: a uniform in (0, 1) from 32 random bits."""
    return (w.astype(np.float64) + 0.5) * (1.0 / 4294967296.0)


def gamma_philox(shape_L, seed: int, n: int, offset: int = 0, max_attempts: int = 64):
    """Gamma(L, scale 1/L) variates for pixels offset .. offset+n-1 (Marsaglia-Tsang, L >= 1).

    Attempt k of pixel p: Philox counter (p lo, p hi, k, 0), key (seed lo, seed hi) ->
      x = sqrt(-2 ln u1) cos(2 pi u2)   (Box-Muller, u1, u2 from words 0, 1)
      v = (1 + c x)^3, accept if v > 0 and ln u3 < x^2/2 + d - d v + d ln v   (u3 from word 2)
    with d = L - 1/3, c = 1/sqrt(9 d); the variate is d v / L.  Returns (s, attempts)."""
    L = float(shape_L)
    if not L >= 1.0:
        raise ValueError("this generator needs L >= 1")
    d = L - 1.0 / 3.0
    c = 1.0 / math.sqrt(9.0 * d)
    p = np.arange(offset, offset + n, dtype=np.uint64)
    plo = p & np.uint64(MASK32)
    phi = p >> np.uint64(32)
    k0 = np.uint64(seed & MASK32)
    k1 = np.uint64((seed >> 32) & MASK32)
    out = np.full(n, np.nan)
    attempts = np.zeros(n, np.int64)
    todo = np.ones(n, bool)
    for k in range(max_attempts):
        if not todo.any():
            break
        idx = np.nonzero(todo)[0]
        w0, w1, w2, _ = philox4x32_10(plo[idx], phi[idx], np.full(idx.size, k, np.uint64), np.zeros(idx.size, np.uint64),
                                      k0, k1)
        u1, u2, u3 = _u01(w0), _u01(w1), _u01(w2)
        x = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)
        t = 1.0 + c * x
        v = t * t * t
        ok = v > 0
        acc = np.zeros(idx.size, bool)
        acc[ok] = np.log(u3[ok]) < 0.5 * x[ok] * x[ok] + d - d * v[ok] + d * np.log(v[ok])
        attempts[idx] += 1
        out[idx[acc]] = d * v[acc] / L
        todo[idx[acc]] = False
    return out, attempts


def add_speckle_philox(u, looks, seed: int):
    """f = u sqrt(s) per image b (looks[b]), pixel counter p = b H W + y W + x; fp32 result."""
    u = np.asarray(u, np.float64)
    if u.ndim == 2:
        u = u[None]
    B, H, W = u.shape
    looks = np.broadcast_to(np.asarray(looks, np.float64), (B,))
    f = np.empty((B, H, W), np.float32)
    for b in range(B):
        s, _ = gamma_philox(looks[b], seed, H * W, offset=b * H * W)
        f[b] = (u[b] * np.sqrt(s.reshape(H, W))).astype(np.float32)
    return f
