"""Pins for oracle/filt.py and oracle/conventions.py (CPU only)."""

import json
import math
import os

import numpy as np
import pytest

from dsft_synth import planted
from oracle.conventions import band_B, centered_dft_bruteforce, grid_y, trig_poly_eval
from oracle.filt import g_periodized, ghat, lemma1_majorant

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_values.json")))


@pytest.mark.parametrize("c1", [0.05, 0.1, 0.3])
def test_lemma2_closed_form_vs_quadrature(c1):
    """Lemma 2 against (1/2pi) int g(x) e^{-i omega x} dx of eq. (4),
    by the trapezoid rule (spectrally accurate for smooth periodic integrands)."""
    M = 4096
    x = -math.pi + 2 * math.pi * np.arange(M) / M
    gx = g_periodized(x, c1, n_images=4)
    for om in (0, 1, -1, 7, -7, 20, 64):
        quad = np.mean(gx * np.exp(-1j * om * x))
        assert abs(quad - ghat(om, c1)) < 1e-10


def test_ghat_worked_values():
    g = GOLD["ghat_c1_0p1_omega10"]
    assert abs(float(ghat(10, 0.1)) - g["value"]) < g["tol"]
    assert abs(float(ghat(0, 0.37)) - GOLD["ghat_omega0"]["value"]) < GOLD["ghat_omega0"]["tol"]
    assert abs(float(g_periodized(0.0, 0.1)) - GOLD["g0_c1_0p1"]["value"]) < GOLD["g0_c1_0p1"]["tol"]


def test_ghat_monotone_and_below_half():
    om = np.arange(0, 5000)
    gh = ghat(om, 1e-3)
    assert np.all(np.diff(gh) < 0) and gh.max() < 0.5


def test_lemma1_majorant():
    rng = np.random.default_rng(1)
    for _ in range(200):
        c1 = float(rng.uniform(0.01, 0.5))
        x = rng.uniform(-math.pi, math.pi, 50)
        assert np.all(g_periodized(x, c1) <= lemma1_majorant(x, c1) * (1 + 1e-14))


@pytest.mark.parametrize("N", [16, 15, 37, 64])
def test_centered_dft_convention(N):
    """F f = fhat for f_j = sum fhat_omega e^{i omega y_j}."""
    rng = np.random.default_rng(N)
    B = band_B(N)
    assert len(B) == N and B[0] == -((N + 1) // 2) + 1 and B[-1] == N // 2
    fhat = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    f = trig_poly_eval(B, fhat, grid_y(N))
    om, got = centered_dft_bruteforce(f)
    assert np.array_equal(om, B)
    assert np.max(np.abs(got - fhat)) < 1e-12
    # Parseval: N ||fhat||^2 = ||f||^2
    assert abs(N * np.sum(np.abs(got) ** 2) - np.sum(np.abs(f) ** 2)) < 1e-9 * np.sum(np.abs(f) ** 2)


def test_synth_matches_paper_convention():
    """dsft_synth plants fhat_omega = (-1)^omega c_omega in the PAPER.md:82 convention."""
    for N, s in ((64, 5), (97, 7), (128, 9)):
        pl = planted(N, s, cfg=9, trial=N)
        om, fh = centered_dft_bruteforce(pl.f)
        dense = np.zeros(N, dtype=np.complex128)
        dense[pl.freqs - om[0]] = pl.fhat
        assert np.max(np.abs(fh - dense)) < 1e-12
        assert np.allclose(np.abs(pl.fhat), 1.0)


def test_synth_snr_exact():
    pl0 = planted(4096, 10, cfg=3, trial=1)
    for snr in (0.0, 10.0, 20.0, 60.0):
        pl = planted(4096, 10, cfg=3, trial=1, snr_db=snr)
        n = pl.f - pl0.f
        got = 20 * math.log10(np.linalg.norm(pl0.f) / np.linalg.norm(n))
        assert abs(got - snr) < 1e-9
