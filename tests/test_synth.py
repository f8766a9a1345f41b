"""Pins of the seeded input generators (foe_synth) -- CPU only.

The speckle simulator is pinned to the paper through Table II's noisy-input PSNR
row, which fixes the amplitude reading f = u * sqrt(s),
s ~ Gamma(L, 1/L) (reading R-14).
"""
import math
import os

import numpy as np
import pytest
import scipy.special as ssp
import scipy.stats as sst

import foe_synth as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _table2():
    rows = [l.split() for l in open(os.path.join(GOLD, "table2_noisy_psnr.txt")) if l[0] != "#"]
    return {int(L): float(p) for L, p, _ in rows}


def _noise_ratio_closed_form(L):
    # E[(f-u)^2]/E[u^2] for f = u sqrt(s), s ~ Gamma(L,1/L): 2 - 2 E[sqrt(s)],
    # E[sqrt(s)] = Gamma(L+1/2) / (Gamma(L) sqrt(L))
    return 2.0 - 2.0 * math.exp(ssp.gammaln(L + 0.5) - ssp.gammaln(L)) / math.sqrt(L)


@pytest.mark.parametrize("L", [1, 3, 8])
def test_speckle_moments(L):
    # mean of (f/u)^2 = 1 +- 0.5 %, variance 1/L +- 5 %
    u = np.full((1000, 1000), 100.0, np.float32)
    f = S.add_speckle(u, L, 1234 + L).astype(np.float64)
    s = (f / 100.0) ** 2
    assert abs(s.mean() - 1.0) < 0.005
    assert abs(s.var() - 1.0 / L) < 0.05 / L


@pytest.mark.parametrize("L", [1, 3, 8])
def test_speckle_ks_against_gamma(L):
    # KS statistic below the 1 % critical value
    u = np.full((100000,), 50.0, np.float32)
    s = (S.add_speckle(u, L, 77 + L).astype(np.float64) / 50.0) ** 2
    assert sst.kstest(s, sst.gamma(a=L, scale=1.0 / L).cdf).pvalue > 0.01


def test_speckle_amplitude_reading_reproduces_table2_noisy_row():
    # PAPER.md:333 prints noisy PSNR 21.61 / 17.42 / 12.95 dB at L = 8 / 3 / 1 over the
    # same 68 images; with a common clean power the PSNR differences depend only on the
    # noise model.  Amplitude speckle reproduces both printed differences to the print
    # rounding; the literal intensity reading f = u * s (ratio 1/L) misses by > 0.25 dB.
    gold = _table2()
    r = {L: _noise_ratio_closed_form(L) for L in (1, 3, 8)}
    d31 = 10 * math.log10(r[1] / r[3])
    d83 = 10 * math.log10(r[3] / r[8])
    assert abs(d31 - (gold[3] - gold[1])) < 0.015
    assert abs(d83 - (gold[8] - gold[3])) < 0.015
    assert abs(10 * math.log10(3.0) - (gold[3] - gold[1])) > 0.25
    # and the generator matches the closed form empirically (1 % relative)
    u = S.piecewise_smooth_scene(512, 512, 9).astype(np.float64)
    for L in (1, 3, 8):
        f = S.add_speckle(u, L, 90 + L).astype(np.float64)
        emp = np.mean((f - u) ** 2) / np.mean(u ** 2)
        assert emp == pytest.approx(r[L], rel=0.01)


def test_speckle_reproducible_and_scale_equivariant():
    u = S.piecewise_smooth_scene(64, 48, 1)
    a = S.add_speckle(u, 3, 5)
    np.testing.assert_array_equal(a, S.add_speckle(u, 3, 5))
    np.testing.assert_array_equal(S.add_speckle(4 * u, 3, 5), 4 * a)  # SPEC.md:362 (c = 4 exact)
    assert np.all(S.add_speckle(np.zeros((5, 5), np.float32), 1, 1) == 0)


def test_scenes_range_and_determinism():
    for gen, args in [(S.piecewise_smooth_scene, (100, 77, 3)), (S.sar_like_scene, (128, 160, 4))]:
        a = gen(*args)
        assert a.dtype == np.float32 and a.shape == args[:2]
        assert a.min() >= 1.0 and a.max() <= 255.0
        np.testing.assert_array_equal(a, gen(*args))
    sar = S.sar_like_scene(512, 512, 601)
    assert (sar == 255.0).sum() >= 9  # point targets present


def test_random_bank_properties():
    k, th = S.random_filter_bank(48, 7, 203)
    assert k.dtype == np.float32 and k.shape == (48, 7, 7)
    k64 = k.astype(np.float64)
    assert np.abs(k64.sum(axis=(1, 2))).max() < 1e-6        # zero-mean up to fp32 rounding (R-15)
    np.testing.assert_allclose(np.sqrt((k64 ** 2).sum(axis=(1, 2))), 1.0, atol=1e-6)
    assert th.min() >= 0.1 and th.max() <= 1.0


def test_dct_bank_orthonormal():
    # SPEC.md:50-52, :56
    k, th = S.dct_filter_bank(3, 8)
    G = np.einsum("iab,jab->ij", k.astype(np.float64), k.astype(np.float64))
    np.testing.assert_allclose(G, np.eye(8), atol=1e-6)
    assert np.abs(k.astype(np.float64).sum(axis=(1, 2))).max() < 1e-6
    with pytest.raises(ValueError):
        S.dct_filter_bank(3, 9)


def test_config_registry_matches_baseline():
    c = S.CONFIGS
    assert (c["c1"].H, c["c1"].n_filters, c["c1"].m, c["c1"].iters, c["c1"].looks) == (128, 24, 5, 100, (1,))
    assert (c["c2"].H, c["c2"].n_filters, c["c2"].m, c["c2"].iters, c["c2"].looks) == (256, 48, 7, 200, (3,))
    assert (c["c3"].H, c["c3"].iters, c["c3"].looks) == (512, 300, (8,))
    assert c["c4"].B == 64 and set(c["c4"].looks) == {1, 3, 8}
    assert (c["c5"].H, c["c5"].W, c["c5"].scene) == (8192, 8192, "sar")
    d = S.make_inputs(S.config("c4"), images=[5, 17])
    d2 = S.make_inputs(S.config("c4"))
    np.testing.assert_array_equal(d["f"][1], d2["f"][17])     # shard-independent inputs
