"""Mutation-sensitive pins for the parts of oracle/dsft.py that the end-to-end
tests cannot see ("What's weak" 1): the vote threshold, the
band budget of line 9, the window centre j' = argmin |x - y_j| of Lemma 10, the
window q + B of the identification, the passband edges of line 10 and the
estimator's measurement set (reading R10).  Each test is built so that a
plausible mistake in that step (a threshold off by one, a dropped cut, floor for
round, an open window edge, all grids instead of the identifying ones) fails it.
CPU only."""

import math
from fractions import Fraction

import numpy as np
import pytest

from dsft_synth import planted_at
from oracle.dsft import (SENTINEL, Identification, dsft, estimate, filtered_samples, nearest_grid_index,
                         vote, window_representative)
from oracle.filt import ghat
from oracle.params import OracleParams, derive_plan


# ------------------------------------------------------------ vote (reading R9)
def _ids_with(plan, producers):
    """Identification sets in which bucket prime t produced exactly the omegas
    {omega: t in producers[omega]} (each in its own bucket omega mod P_t)."""
    ids = [Identification(cand=np.full(P, SENTINEL, dtype=np.int64), gap=np.full(P, np.inf))
           for P in plan.primes]
    for om, ts in producers.items():
        for t in ts:
            assert ids[t].cand[om % plan.primes[t]] == SENTINEL
            ids[t].cand[om % plan.primes[t]] = om
    return ids


def test_vote_threshold_is_exactly_v_min():
    """"more than half": with T = 5 and v_min = 3, an omega produced by
    2 distinct bucket primes is rejected, by 3 accepted, by all 5 accepted."""
    plan = derive_plan(4096, 8, OracleParams(seed=0))
    assert plan.T == 5 and plan.vote_min == 3
    ids = _ids_with(plan, {100: [0, 1], 201: [0, 2, 4], -300: [0, 1, 2, 3, 4], 7: [3]})
    assert vote(plan, ids) == [-300, 201]


@pytest.mark.parametrize("T,vmin", [(4, 3), (6, 4), (7, 4)])
def test_vote_majority_default(T, vmin):
    """vote_min = 0 resolves to floor(T/2) + 1, the smallest count that is more than
    half of T; one vote fewer is rejected."""
    plan = derive_plan(2**16, 50, OracleParams(n_bucket_primes=T, vote_min=0, seed=1))
    assert plan.T == T and plan.vote_min == vmin and 2 * vmin > T >= 2 * (vmin - 1)
    ids = _ids_with(plan, {5: list(range(vmin - 1)), 9: list(range(T - vmin, T))})
    assert vote(plan, ids) == [9]


# ------------------------------------------------------ band budget (line 9, R11)
def test_band_budget_keeps_the_largest_per_band():
    """Algorithm 1 line 9: A returns an s-sparse (here band_budget = 1) approximation
    of each band, so of two tones in one passband only the larger survives, while
    a tone alone in another band is kept (reading R11)."""
    N, s = 4096, 4
    base = derive_plan(N, s, OracleParams(seed=2))
    q3, q8 = base.q[3], base.q[8]
    freqs = [q3 - 10, q3 + 20, q8]
    pl = planted_at(N, freqs, [1.0, 2.0j, -1.5])
    full = dsft(pl.f, s, OracleParams(seed=2))
    assert sorted(full.freqs.tolist()) == sorted(freqs)
    cut = dsft(pl.f, s, OracleParams(seed=2, band_budget=1))
    assert sorted(cut.freqs.tolist()) == sorted([q3 + 20, q8])
    d = dict(zip(cut.freqs.tolist(), cut.coeffs))
    assert abs(d[q3 + 20] - pl.fhat[list(pl.freqs).index(q3 + 20)]) < 1e-4


# ------------------------------------------------ passband edges (line 10) and B
def test_passband_edges_and_B_extremes():
    """Line 10 keeps omega in [q - w, q + w) cap B: a tone at q_j - w
    belongs to band j, one at q_j + w = q_{j+1} - w to band j + 1 only (the
    passbands partition B: no duplicate), and the extremes of B = (-ceil(N/2),
    floor(N/2)] are recovered."""
    for N in (4096, 4095):
        s = 8
        plan = derive_plan(N, s, OracleParams(seed=3))
        w, q = plan.w, plan.q
        freqs = sorted({q[2] - w, q[2] + w, q[5] + w - 1, plan.B_lo, plan.B_hi, q[9]})
        assert len(freqs) == 6 and all(plan.B_lo <= x <= plan.B_hi for x in freqs)
        pl = planted_at(N, freqs, np.exp(1j * np.arange(len(freqs))))
        res = dsft(pl.f, s, plan=plan, keep_bands=True)
        assert sorted(res.freqs.tolist()) == freqs
        owners = {om: [j for j, br in enumerate(res.bands) if om in br.omegas] for om in freqs}
        assert owners[q[2] - w] == [2] and owners[q[2] + w] == [3] and owners[q[5] + w - 1] == [5]
        assert owners[plan.B_lo] == [0] and owners[plan.B_hi] == [plan.J - 1]
        d = dict(zip(res.freqs.tolist(), res.coeffs))
        assert max(abs(d[int(x)] - v) for x, v in zip(pl.freqs, pl.fhat)) < 1e-4


# ------------------------------------------ window centre j' (Lemma 10, R3)
@pytest.mark.parametrize("N", [64, 97, 100, 255])
@pytest.mark.parametrize("L", [15, 77, 111, 205, 393])
def test_window_centre_is_the_nearest_grid_point(N, L):
    """j' = argmin_j |x_k - y_j| by brute force over j in [0, N] with
    exact rationals, and |x_k - y_j'| <= pi / N."""
    jp = nearest_grid_index(np.arange(L), N, L)
    for k in range(L):
        dist = [abs(Fraction(k, L) - Fraction(j, N)) for j in range(N + 1)]  # (x_k - y_j) / (2 pi)
        best = min(range(N + 1), key=lambda j: dist[j])
        assert jp[k] == best
        assert dist[best] <= Fraction(1, 2 * N)


@pytest.mark.parametrize("N,L,j0", [(64, 111, 0), (97, 77, 50), (100, 393, 99), (255, 205, 128)])
def test_filtered_samples_window_support(N, L, j0):
    """Closed form for a unit impulse f = e_{j0}: h_q(x_k) != 0 exactly at the nodes
    whose window j' - kappa .. j' + kappa (mod N) contains j0,
    with j' the brute-force nearest grid index (the Gaussian taps never vanish)."""
    plan = derive_plan(N, 4, OracleParams(seed=0))
    f = np.zeros(N, dtype=np.complex128)
    f[j0] = 1.0
    h = filtered_samples(f, plan, plan.q[1], L)
    for k in range(L):
        best = min(range(N + 1), key=lambda j: abs(Fraction(k, L) - Fraction(j, N)))
        inside = any((best + u) % N == j0 for u in range(-plan.kappa, plan.kappa + 1))
        assert (h[k] != 0) == inside, (k, best)


# ------------------------------------------------- window q + B (reading R7, G4)
@pytest.mark.parametrize("N", [10, 11, 36])
def test_window_representative_bruteforce(N):
    """omega' = the unique integer = R (mod M) in q + B = (q - ceil(N/2), q + floor(N/2)],
    or none: brute force over the N integers of the window, both edges included."""
    for M in (N, N + 1, 2 * N - 1, 3 * N + 2):
        for q in range(-N, N + 1):
            window = range(q - (N + 1) // 2 + 1, q + N // 2 + 1)
            assert len(window) == N
            R = np.arange(M)
            got = window_representative(R, M, q, N)
            for r in range(M):
                hits = [x for x in window if (x - r) % M == 0]
                assert len(hits) <= 1
                assert got[r] == (hits[0] if hits else SENTINEL)


# ------------------------------------------------- estimator (reading R10, line 11)
@pytest.mark.parametrize("voting,odd", [((0, 1), False), ((0, 1, 2), False), ((1, 3), True)])
def test_estimate_uses_the_identifying_grids_only(voting, odd):
    """Reading R10: z_omega = median Re + i median Im of
    (-1)^omega E_{t,i}[omega mod L_{t,i}] over the grids of the bucket primes that
    produced omega; whatever the other grids hold does not enter.  The values are
    a shuffled 1..n (Re) and 10..10+n-1 (Im), so the median is known in closed form
    ((n+1)/2, mean of the two middle ones for even n).  vote_min = 2 leaves the
    non-voting grids in the majority, so an estimator over all T K grids fails.
    Line 11: at omega = q, c = z / ghat_0 = sqrt(2 pi) z."""
    plan = derive_plan(4096, 8, OracleParams(seed=4, vote_min=2))
    j = 6
    om = plan.q[j] + (1 if odd else 0)
    sgn = -1.0 if om % 2 else 1.0
    ids = _ids_with(plan, {om: list(voting)})
    n = sum(len(plan.residues[t]) for t in voting)
    rng = np.random.default_rng(7)
    re = rng.permutation(np.arange(1, n + 1)).astype(float)
    im = rng.permutation(np.arange(10, 10 + n)).astype(float)
    Y, k = [], 0
    for t in range(plan.T):
        row = []
        for L in plan.grid_lengths(t):
            y = np.full(L, 1e3 + 7e2j)  # non-identifying grids: far from every voter value
            if t in voting:
                y[om % L] = sgn * complex(re[k], im[k])
                k += 1
            row.append(y)
        Y.append(row)
    assert vote(plan, ids) == [om]
    oms, cs, zs, _ = estimate(plan, j, Y, ids, [om])
    z_exp = complex((n + 1) / 2, 10 + (n - 1) / 2)
    assert oms == [om] and zs[0] == z_exp
    assert abs(cs[0] - z_exp / float(ghat(om - plan.q[j], plan.c1))) <= 1e-15 * abs(cs[0])
    if not odd:
        assert abs(cs[0] - math.sqrt(2 * math.pi) * z_exp) <= 1e-14 * abs(cs[0])
