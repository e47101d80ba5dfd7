"""Pins for the CLW-style inner SFT of the oracle (reading R14; SURVEY §8(f) 4,
PAPER.md:653 "CLW-DSFT ... uses the SFT developed in [clw] in its line 9";
SPEC.md's phase-encoding engine).  CPU only: closed forms (the aliasing identity on
shifted grids), exhaustive decoding on tiny N, brute-force DFT end to end."""

import math

import numpy as np
import pytest

from dsft_synth import planted, planted_at
from oracle.conventions import centered_dft_bruteforce
from oracle.dsft import (SENTINEL, alias_dft, clw_decode, dsft, filtered_samples, identify_clw,
                         nearest_grid_index)
from oracle.filt import ghat
from oracle.params import OracleParams, clw_shifts, derive_plan


def wrap_B(x, N):
    lo = -((N + 1) // 2) + 1
    return lo + (np.asarray(x) - lo) % N


@pytest.mark.parametrize("P,N", [(7, 64), (37, 4096), (4051, 2**26), (211, 2**22), (13, 13 * 64), (17, 17 * 64 + 1)])
def test_clw_shifts_are_the_fewest_dyadic_scales(P, N):
    """0, then 1, 2, ..., 2^(L-1) with L the smallest count for which 2^(L-1) P >= N."""
    sh = clw_shifts(P, N)
    L = len(sh) - 1
    assert sh == [0] + [2 ** l for l in range(L)]
    assert 2 ** (L - 1) * P >= N and (L == 1 or 2 ** (L - 2) * P < N)


@pytest.mark.parametrize("N,P", [(64, 7), (97, 11), (100, 13), (255, 17), (1000, 31)])
def test_clw_decode_exhaustive(N, P):
    """Every omega' of the window q + B is decoded from exact shifted measurements
    E_sigma = c exp(2 pi i omega' m_sigma / N) in its bucket b = omega' mod P (the
    aliasing identity of a single frequency), for several band centres,
    including both edges of the window (the circular lift), and with phase errors of
    0.02 rad per scale; with errors up to pi/4 per scale for every omega' at least P
    from the window edges (a frequency near an edge is only distinguished from its
    wrap by N mod P, PAPER.md:84 / reading R14)."""
    rng = np.random.default_rng(N + P)
    sh = clw_shifts(P, N)
    for q in (-N // 2 + 3, -5, 0, 7, N // 2 - 2):
        lo = q - (N + 1) // 2 + 1
        for om in range(lo, lo + N):
            c = complex(*rng.standard_normal(2))
            inner = lo + P <= om < lo + N - P
            for noise in ((0.0, 0.02, math.pi / 4) if inner else (0.0, 0.02)):
                E = [c * np.exp(2j * math.pi * om * m / N + 1j * (noise * rng.uniform(-1, 1) if i else 0.0))
                     for i, m in enumerate(sh)]
                got, _ = clw_decode(E, sh, om % P, P, q, N)
                assert got == om, (q, om, noise)


def test_clw_decode_rejects_empty_bucket_and_wraps_foreign_frequencies():
    """An empty bucket yields no candidate; a frequency outside q + B is decoded as its
    representative in the window (the phases are N-periodic; G4's wrapped copy, which
    line 10's "cap B" / passband then rejects)."""
    N, P = 64, 7
    sh = clw_shifts(P, N)
    assert clw_decode([0j] * len(sh), sh, 3, P, 0, N)[0] == SENTINEL
    q, om = 0, 40  # q + B = (-32, 32]: 40 wraps to -24
    E = [np.exp(2j * math.pi * om * m / N) for m in sh]
    got, _ = clw_decode(E, sh, (om - N) % P, P, q, N)
    assert got == om - N


def closed_form_h(pl, plan, q, x):
    N = plan.N
    om = pl.freqs
    omp = q + wrap_B(om - q, N)
    ell = (om - omp) // N
    sgn = np.where((N * ell) % 2 == 0, 1.0, -1.0)
    amp = pl.fhat * sgn * ghat(omp - q, plan.c1)
    return np.exp(1j * np.outer(x, omp)) @ amp


@pytest.mark.parametrize("N,m", [(4096, 1), (4096, 64), (4095, 5), (6007, 512)])
def test_shifted_filtered_samples_closed_form(N, m):
    """O2 on a grid shifted by m steps of f: the closed form at x_k + 2 pi m / N within
    Theorem 4's bound 3 ||f||_inf N^-r (THM4, r = 2), and the window
    centre moves by exactly m (nearest_grid_index + m)."""
    plan = derive_plan(N, 8, OracleParams(preset="thm4", r=2.0))
    pl = planted(N, 12, cfg=61, trial=m)
    L = 37 * 3
    x = -math.pi + 2 * math.pi * np.arange(L) / L + 2 * math.pi * m / N
    bound = 3 * np.max(np.abs(pl.f)) * N ** -2.0
    for q in (plan.q[0], plan.q[len(plan.q) // 2], plan.q[-1]):
        err = np.max(np.abs(filtered_samples(pl.f, plan, q, L, m) - closed_form_h(pl, plan, q, x)))
        assert err <= bound, (q, err, bound)
    # impulse response: the shifted node's window is the unshifted one moved by m
    f = np.zeros(N, dtype=np.complex128)
    j0 = N // 3
    f[j0] = 1.0
    h = filtered_samples(f, plan, plan.q[1], L, m)
    jp = nearest_grid_index(np.arange(L), N, L) + m
    for k in range(L):
        inside = any((jp[k] + u) % N == j0 for u in range(-plan.kappa, plan.kappa + 1))
        assert (h[k] != 0) == inside


def test_clw_identifies_isolated_tones_in_every_prime():
    """Noiseless, well separated tones (kappa = 12 as CLW-DSFT): every
    bucket prime decodes each tone in its bucket."""
    N, s = 4096, 8
    plan = derive_plan(N, s, OracleParams(inner="clw", kappa=12, seed=1))
    assert all(r == [1] for r in plan.residues)
    pl = planted(N, 6, cfg=62, trial=0)
    r = dsft(pl.f, s, plan=plan, keep_bands=True)
    for om in pl.freqs:
        j = [jj for jj in range(plan.J) if plan.q[jj] - plan.w <= om < plan.q[jj] + plan.w][0]
        for t in range(plan.T):
            assert r.bands[j].ids[t].cand[om % plan.primes[t]] == om
    # 6 tones with s = 8: the 6 lead the output; any further entry is filter leakage
    assert sorted(r.freqs[:6].tolist()) == pl.freqs.tolist()
    assert np.all(np.abs(r.coeffs[6:]) < 1e-6)


@pytest.mark.parametrize("N,s", [(64, 4), (97, 4), (128, 6), (255, 6), (512, 8)])
def test_clw_end_to_end_vs_bruteforce_dft(N, s):
    """The CLW-style inner SFT in Algorithm 1 on exactly s-sparse inputs: the output set
    is R_s^opt of the O(N^2) brute-force DFT."""
    for trial in range(3):
        pl = planted(N, s, cfg=63, trial=trial)
        B, fh = centered_dft_bruteforce(pl.f)
        order = sorted(range(N), key=lambda k: (-abs(fh[k]), B[k]))[:s]
        res = dsft(pl.f, s, OracleParams(inner="clw", kappa=12, seed=trial))
        assert sorted(res.freqs.tolist()) == sorted(B[k] for k in order)
        d = dict(zip(res.freqs.tolist(), res.coeffs))
        assert max(abs(d[int(B[k])] - fh[k]) for k in order) < 1e-4


def test_clw_band_edges():
    """Passband edges and the extremes of B with the CLW identification (line 10)."""
    N, s = 4096, 8
    plan = derive_plan(N, s, OracleParams(inner="clw", kappa=12, seed=3))
    w, q = plan.w, plan.q
    freqs = sorted({q[2] - w, q[2] + w, plan.B_lo, plan.B_hi, q[9]})
    pl = planted_at(N, freqs, np.exp(1j * np.arange(len(freqs))))
    res = dsft(pl.f, s, plan=plan)
    n = len(freqs)
    assert sorted(res.freqs[:n].tolist()) == freqs and np.all(np.abs(res.coeffs[n:]) < 1e-6)


@pytest.mark.parametrize("j,t", [(4, 1), (0, 0), (7, 3), (14, 4)])
def test_identify_clw_matches_decode_per_bucket(j, t):
    """identify_clw = clw_decode in every bucket followed by the passband and B (line 10);
    the decision margins agree too (they cover the buckets whose circular estimate sits at
    the ends of q + B, where only the lifts by -N / +N find the nearest representative:
    those candidates fall outside the passband, so only the margin shows the lift)."""
    N, s = 4096, 8
    plan = derive_plan(N, s, OracleParams(inner="clw", seed=2))
    pl = planted(N, s, cfg=64, trial=1)
    q = plan.q[j]
    P = plan.primes[t]
    Et = [alias_dft(filtered_samples(pl.f, plan, q, P, m)) for m in plan.shifts[t]]
    ids = identify_clw(plan, j, t, Et)
    for b in range(P):
        om, margin = clw_decode([E[b] for E in Et], plan.shifts[t], b, P, q, N)
        keep = om != SENTINEL and q - plan.w <= om < q + plan.w and plan.B_lo <= om <= plan.B_hi
        assert ids.cand[b] == (om if keep else SENTINEL)
        assert abs(ids.gap[b] - margin) <= 1e-9 or ids.gap[b] == margin  # (inf == inf: empty bucket)
