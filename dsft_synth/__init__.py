"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic: it only plants sparse
spectra and adds noise, following the paper's trial protocol (PAPER.md:659:
s frequencies, unit magnitude, uniform random phase, inverse DFT; PAPER.md:686
footnote: SNR = 20 log10(||f||_2 / ||n||_2), i.i.d. complex Gaussian noise) as
restated by BASELINE.json's configs (frequencies drawn without replacement from
B, reading R12 in DESIGN.md).

Recipe: Generator(PCG64(SeedSequence([0xD5F7, cfg, trial, vector])));
freqs = rng.choice(N, s, replace=False) - ceil(N/2) + 1; theta = 2 pi rng.random(s);
c = exp(i theta); f_j = sum_omega c_omega exp(2 pi i omega j / N) via N*ifft.
In the paper's convention the planted DFT is fhat_omega = (-1)^omega c_omega.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass
class Planted:
    f: np.ndarray            # complex128[N] (noisy if snr_db given)
    freqs: np.ndarray        # int64[s], ascending
    fhat: np.ndarray         # complex128[s]: paper-convention truth at freqs
    noise_inf: float = 0.0   # ||n||_inf (0 if noiseless)


def rng_for(cfg: int, trial: int, vector: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([0xD5F7, cfg, trial, vector])))


def planted(N: int, s: int, cfg: int = 0, trial: int = 0, vector: int = 0,
            snr_db: float | None = None, magnitudes: np.ndarray | None = None) -> Planted:
    """Exactly s-sparse planted spectrum on B, optional noise at an exact SNR."""
    rng = rng_for(cfg, trial, vector)
    lo = -((N + 1) // 2) + 1
    idx = rng.choice(N, s, replace=False).astype(np.int64)
    freqs = idx + lo
    theta = 2.0 * math.pi * rng.random(s)
    c = np.exp(1j * theta)
    if magnitudes is not None:
        c = c * np.asarray(magnitudes, dtype=np.float64)
    chat = np.zeros(N, dtype=np.complex128)
    chat[freqs % N] = c
    f = N * np.fft.ifft(chat)
    sign = np.where(freqs % 2 == 0, 1.0, -1.0)
    order = np.argsort(freqs)
    out = Planted(f=f, freqs=freqs[order], fhat=(sign * c)[order])
    if snr_db is not None:
        n = rng.standard_normal(N) + 1j * rng.standard_normal(N)
        scale = np.linalg.norm(f) / (np.linalg.norm(n) * 10.0 ** (snr_db / 20.0))
        n *= scale
        out.f = f + n
        out.noise_inf = float(np.max(np.abs(n)))
    return out


def planted_with_tail(N: int, s: int, tail: int, tail_mag: float, cfg: int = 0,
                      trial: int = 0) -> Planted:
    """s unit-magnitude heads plus `tail` smaller entries (SPEC.md:462 style)."""
    mags = np.concatenate([np.ones(s), np.full(tail, tail_mag)])
    rng = rng_for(cfg, trial, 1)
    mags = mags[rng.permutation(s + tail)]
    return planted(N, s + tail, cfg=cfg, trial=trial, magnitudes=mags)


def planted_at(N: int, freqs, coeffs) -> Planted:
    """f_j = sum_omega c_omega exp(2 pi i omega j / N) for GIVEN frequencies on B and
    coefficients c (test fixtures with tones placed on band edges etc.)."""
    freqs = np.asarray(freqs, dtype=np.int64)
    c = np.asarray(coeffs, dtype=np.complex128)
    chat = np.zeros(N, dtype=np.complex128)
    chat[freqs % N] = c
    f = N * np.fft.ifft(chat)
    sign = np.where(freqs % 2 == 0, 1.0, -1.0)
    order = np.argsort(freqs)
    return Planted(f=f, freqs=freqs[order], fhat=(sign * c)[order])
