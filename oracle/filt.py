"""Periodized Gaussian filter (test infrastructure only).

PAPER.md:121-127 eq. (Def_Periodic_Gaussian):
    g(x) = (1/c1) * sum_n exp(-(x - 2 n pi)^2 / (2 c1^2))
Lemma 2:  ghat_omega = exp(-c1^2 omega^2 / 2) / sqrt(2 pi).
Lemma 1:  g(x) <= (3/c1 + 1/sqrt(2 pi)) exp(-x^2/(2 c1^2)).
"""

from __future__ import annotations

import math

import numpy as np


def g_periodized(x, c1: float, n_images: int = 3):
    """eq. (4) with the image sum truncated to |n| <= n_images (reading R5:
    for c1 < 0.5 the |n| >= 1 images are below e^-(pi^2/(2 c1^2)) ~ e^-19)."""
    x = np.asarray(x, dtype=np.float64)
    acc = np.zeros_like(x)
    for n in range(-n_images, n_images + 1):
        acc = acc + np.exp(-((x - 2.0 * n * math.pi) ** 2) / (2.0 * c1 * c1))
    return acc / c1


def ghat(omega, c1: float):
    """Lemma 2: Fourier coefficient of g at integer omega."""
    om = np.asarray(omega, dtype=np.float64)
    return np.exp(-(c1 * c1) * om * om / 2.0) / math.sqrt(2.0 * math.pi)


def lemma1_majorant(x, c1: float):
    """Lemma 1 upper bound for g(x), x in [-pi, pi]."""
    x = np.asarray(x, dtype=np.float64)
    return (3.0 / c1 + 1.0 / math.sqrt(2.0 * math.pi)) * np.exp(-(x * x) / (2.0 * c1 * c1))
