"""Centered-DFT conventions (test infrastructure only).

PAPER.md:79-98: F_{omega,j} = ((-1)^omega / N) exp(-2 pi i omega j / N),
B = (-ceil(N/2), floor(N/2)] cap Z, f_j = f(-pi + 2 pi j / N), fhat = F f.
"""

from __future__ import annotations

import math

import numpy as np


def band_B(N: int) -> np.ndarray:
    """B as an increasing int64 array."""
    return np.arange(-((N + 1) // 2) + 1, N // 2 + 1, dtype=np.int64)


def grid_y(N: int) -> np.ndarray:
    """y_j = -pi + 2 pi j / N, j = 0..N-1."""
    return -math.pi + 2.0 * math.pi * np.arange(N, dtype=np.float64) / N


def parity_sign(omega):
    """(-1)^omega for integer omega of either sign."""
    om = np.asarray(omega, dtype=np.int64)
    return np.where(om % 2 == 0, 1.0, -1.0)


def centered_dft_bruteforce(f: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """fhat = F f by the O(N^2) matrix of PAPER.md:82.  Returns (B, fhat)."""
    f = np.asarray(f, dtype=np.complex128)
    N = f.shape[0]
    om = band_B(N)
    j = np.arange(N, dtype=np.int64)
    # reduce omega*j mod N exactly before forming the angle
    ang = 2.0 * math.pi * ((om[:, None] * j[None, :]) % N) / N
    Fm = parity_sign(om)[:, None] * np.exp(-1j * ang) / N
    return om, Fm @ f


def trig_poly_eval(freqs, coeffs, x) -> np.ndarray:
    """f(x) = sum_omega fhat_omega exp(i omega x)."""
    freqs = np.asarray(freqs, dtype=np.float64)
    coeffs = np.asarray(coeffs, dtype=np.complex128)
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    return np.exp(1j * x[:, None] * freqs[None, :]) @ coeffs
