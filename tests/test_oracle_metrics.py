"""Pins of the oracle's f4 tier (oracle/metrics.py): PSNR / SSIM and the
counter-based speckle generator (Philox4x32-10 + Marsaglia-Tsang, reading R-14).

PSNR/SSIM against SPEC.md's worked values and closed forms (identical images, constant images,
symmetry, inversion, a noise ladder); Philox against its published known-answer vectors
(tests/golden/philox4x32_10_kat.txt); the Gamma variates against the Gamma(L, 1/L) law (moments,
Kolmogorov-Smirnov against scipy.stats.gamma) and the speckled images against Table II's noisy-PSNR
closed form (reading R-14).
"""
import math
import os

import numpy as np
import pytest
import scipy.stats as sst

import foe_synth as S
from oracle import metrics as M

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_psnr_spec_values():
    ref = np.full((8, 8), 100.0)
    assert M.psnr(ref, ref) == math.inf
    assert M.psnr(np.full((4, 4), 255.0), np.zeros((4, 4))) == pytest.approx(0.0, abs=1e-12)
    assert M.psnr(np.full((4, 4), 110.0), ref[:4, :4]) == pytest.approx(10 * math.log10(255 ** 2 / 100), rel=1e-14)
    rng = np.random.default_rng(0)
    x, y = rng.uniform(0, 255, (2, 16, 16))
    assert M.psnr(x, y) == M.psnr(y, x)
    prev = math.inf
    for a in (0.5, 1, 2, 4, 8):                       # strictly decreasing on a noise ladder
        p = M.psnr(y + a * np.sign(rng.standard_normal(y.shape)), y)
        assert p < prev
        prev = p


def test_ssim_closed_forms_and_properties():
    rng = np.random.default_rng(1)
    x = rng.uniform(0, 255, (20, 23))
    assert M.ssim(x, x) == pytest.approx(1.0, abs=1e-14)
    y = x + rng.normal(0, 20, x.shape)
    assert M.ssim(x, y) == pytest.approx(M.ssim(y, x), rel=1e-14)      # symmetric
    assert M.ssim(255 - x, x) < 1.0                                     # inversion
    assert -1.0 <= M.ssim(255 - x, x) <= 1.0
    # two constant images a, b: sigma = 0, so SSIM = (2ab + C1)/(a^2 + b^2 + C1) exactly
    a, b = 90.0, 130.0
    c1 = (0.01 * 255) ** 2
    assert M.ssim(np.full((15, 15), a), np.full((15, 15), b)) == pytest.approx((2 * a * b + c1) / (a * a + b * b + c1),
                                                                            rel=1e-12)
    g = M.gaussian_window()
    assert g.sum() == pytest.approx(1.0) and g[5] == g.max() and np.allclose(g, g[::-1])
    with pytest.raises(ValueError):
        M.ssim(np.zeros((10, 30)), np.zeros((10, 30)))


def test_ssim_brute_force_single_window():
    # an 11x11 image has exactly one window: SSIM from plain weighted moments written out
    rng = np.random.default_rng(2)
    x, y = rng.uniform(0, 255, (2, 11, 11))
    w = np.outer(M.gaussian_window(), M.gaussian_window())
    mx, my = (w * x).sum(), (w * y).sum()
    vx = (w * (x - mx) ** 2).sum()
    vy = (w * (y - my) ** 2).sum()
    cxy = (w * (x - mx) * (y - my)).sum()
    c1, c2 = (0.01 * 255) ** 2, (0.03 * 255) ** 2
    ref = (2 * mx * my + c1) * (2 * cxy + c2) / ((mx * mx + my * my + c1) * (vx + vy + c2))
    assert M.ssim(x, y) == pytest.approx(ref, rel=1e-12)


def test_philox_known_answer_vectors():
    for line in open(os.path.join(GOLD, "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(t, 16) for t in line.split()]
        out = M.philox4x32_10([v[0]], [v[1]], [v[2]], [v[3]], v[4], v[5])
        assert [int(o[0]) for o in out] == v[6:10]


def test_philox_uniform_bits():
    n = 200000
    w = M.philox4x32_10(np.arange(n, dtype=np.uint64), 0, 0, 0, 12345, 678)
    u = M._u01(np.concatenate(w))
    assert sst.kstest(u, "uniform").pvalue > 0.001
    bits = np.unpackbits(np.concatenate(w).view(np.uint8))
    assert abs(bits.mean() - 0.5) < 2e-3


@pytest.mark.parametrize("L", [1, 3, 8])
def test_gamma_philox_law(L):
    s, att = M.gamma_philox(L, seed=99 + L, n=200000)
    assert np.isfinite(s).all() and att.max() < 64
    assert s.mean() == pytest.approx(1.0, rel=0.01)
    assert s.var() == pytest.approx(1.0 / L, rel=0.03)
    assert sst.kstest(s, sst.gamma(a=L, scale=1.0 / L).cdf).pvalue > 0.001
    assert att.mean() < 1.1                               # Marsaglia-Tsang acceptance > 0.9


@pytest.mark.parametrize("L", [1, 3, 8])
def test_speckle_philox_table2_noisy_psnr(L):
    # R-14: E[(f-u)^2]/E[u^2] = 2 - 2 Gamma(L+1/2)/(Gamma(L) sqrt(L)) for f = u sqrt(s)
    u = np.full((256, 256), 120.4)
    f = M.add_speckle_philox(u, [L], seed=7)[0].astype(np.float64)
    ratio = np.mean((f - u) ** 2) / np.mean(u ** 2)
    closed = 2 - 2 * math.exp(math.lgamma(L + 0.5) - math.lgamma(L)) / math.sqrt(L)
    assert ratio == pytest.approx(closed, rel=0.02)
    # scale equivariance: the same draws scale with u
    f2 = M.add_speckle_philox(2 * u, [L], seed=7)[0]
    np.testing.assert_allclose(f2, 2 * M.add_speckle_philox(u, [L], seed=7)[0], rtol=1e-6)
