"""Pins for oracle/dsft.py (CPU only): each step against a closed form, brute
force, or the paper's error bounds (DESIGN.md §4 lists which pin covers what)."""

import math

import numpy as np
import pytest

from dsft_synth import planted, planted_with_tail
from oracle.conventions import centered_dft_bruteforce
from oracle.dsft import (SENTINEL, alias_dft, dsft, filtered_samples, identify, merge,
                         process_band, residue_bin)
from oracle.filt import ghat
from oracle.params import OracleParams, derive_plan


def wrap_B(x, N):
    """Representative of x mod N in B = (-ceil(N/2), floor(N/2)]."""
    lo = -((N + 1) // 2) + 1
    return lo + (np.asarray(x) - lo) % N


def closed_form_h(pl, plan, q, x):
    """(g~_q * f)(x) for a planted sparse f (G4 / reading R1): every omega appears
    at omega' = q + wrap_B(omega - q) with weight (-1)^{N l} ghat_{omega'-q}."""
    N = plan.N
    om = pl.freqs
    omp = q + wrap_B(om - q, N)
    ell = (om - omp) // N
    sgn = np.where((N * ell) % 2 == 0, 1.0, -1.0)
    amp = pl.fhat * sgn * ghat(omp - q, plan.c1)
    return np.exp(1j * np.outer(x, omp)) @ amp


@pytest.mark.parametrize("N,r", [(4096, 1.0), (4096, 2.0), (4095, 1.0), (6007, 2.0)])
def test_filtered_samples_theorem4_bound(N, r):
    """Theorem 4: |(g*f)(x) - truncated sum| <= 3 ||f||_inf N^-r,
    applied to every band centre q (incl. the edge bands, reading R1/G4)."""
    plan = derive_plan(N, 8, OracleParams(preset="thm4", r=r))
    pl = planted(N, 20, cfg=11, trial=int(r * 10) + N % 7)
    bound = 3 * np.max(np.abs(pl.f)) * N ** (-r)
    L = 37 * 5
    x = -math.pi + 2 * math.pi * np.arange(L) / L
    for q in plan.q + [0]:
        h = filtered_samples(pl.f, plan, q, L)
        err = np.max(np.abs(h - closed_form_h(pl, plan, q, x)))
        assert err <= bound, (q, err, bound)


def test_filtered_samples_dmsft_accuracy_and_window():
    """DMSFT presets: error far below the unit coefficients (reading R4); kappa
    large enough to cover all of f equals the untruncated sum (eq. UntruncatedFiniteSum)."""
    N = 4096
    pl = planted(N, 20, cfg=12, trial=0)
    for preset, tol in (("dmsft6", 2e-4), ("dmsft4", 5e-3)):  # 20 unit tones; survey measured 4-7e-5 / 1.2-1.8e-3
        plan = derive_plan(N, 8, OracleParams(preset=preset))
        L = 41 * 3
        x = -math.pi + 2 * math.pi * np.arange(L) / L
        for q in (plan.q[0], plan.q[7], plan.q[-1]):
            err = np.max(np.abs(filtered_samples(pl.f, plan, q, L) - closed_form_h(pl, plan, q, x)))
            assert err < tol, (preset, q, err)
    # full window vs the dense semi-discrete sum (1/N) sum_j f_j g~(x - y_j)
    Nt = 64
    plt = planted(Nt, 4, cfg=12, trial=1)
    plan = derive_plan(Nt, 4, OracleParams(kappa=31))
    L = 17 * 3
    q = plan.q[3]
    h = filtered_samples(plt.f, plan, q, L)
    x = -math.pi + 2 * math.pi * np.arange(L) / L
    y = -math.pi + 2 * math.pi * np.arange(Nt) / Nt
    dense = np.zeros(L, dtype=np.complex128)
    for jj in range(Nt):
        d = (x - y[jj] + math.pi) % (2 * math.pi) - math.pi  # nearest image
        gg = sum(np.exp(-(d + 2 * math.pi * n) ** 2 / (2 * plan.c1 ** 2)) for n in (-1, 0, 1)) / plan.c1
        dense += plt.f[jj] * gg * np.exp(1j * q * d)
    dense /= Nt
    # kappa = 31 covers 63 of 64 entries; the missing one sits at distance ~pi (weight e^-500)
    assert np.max(np.abs(h - dense)) < 1e-12


def test_alias_dft_bruteforce_and_aliasing_identity():
    """O3 vs the O(L^2) DFT; aliasing identity E[b] = sum_{omega'=b (L)} (-1)^omega' hhat_omega'
    within the filter error."""
    N = 4096
    plan = derive_plan(N, 8, OracleParams(preset="thm4", r=2.0))
    pl = planted(N, 12, cfg=13, trial=0)
    q = plan.q[5]
    L = 43 * 7
    h = filtered_samples(pl.f, plan, q, L)
    Y = alias_dft(h)
    k = np.arange(L)
    brute = np.array([np.sum(h * np.exp(-2j * math.pi * ((k * b) % L) / L)) / L for b in range(L)])
    assert np.max(np.abs(Y - brute)) < 1e-13 * max(1.0, np.max(np.abs(h)))
    omp = q + wrap_B(pl.freqs - q, N)
    ell = (pl.freqs - omp) // N
    amp = pl.fhat * np.where((N * ell) % 2 == 0, 1, -1) * ghat(omp - q, plan.c1)
    ref = np.zeros(L, dtype=np.complex128)
    np.add.at(ref, omp % L, np.where(omp % 2 == 0, 1, -1) * amp)
    assert np.max(np.abs(Y - ref)) <= 3 * np.max(np.abs(pl.f)) * N ** -2.0


def test_residue_bin_bruteforce():
    for P, r in ((37, 3), (41, 11), (17, 5)):
        for a in range(P):
            for c in range(r):
                n = int(residue_bin(a, c, P, r))
                assert n == [m for m in range(P * r) if m % P == a and m % r == c][0]


def test_identify_bruteforce_crt():
    """O4 against a brute-force scan of the window q + B and the passband."""
    N = 200
    plan = derive_plan(N, 4, OracleParams(seed=4))
    pl = planted(N, 4, cfg=14, trial=2)
    for j in (0, plan.J // 2, plan.J - 1):
        q = plan.q[j]
        for t in range(plan.T):
            P, rs = plan.primes[t], plan.residues[t]
            Yt = [alias_dft(filtered_samples(pl.f, plan, q, P * r)) for r in rs]
            ids = identify(plan, j, t, Yt)
            window = range(q - (N + 1) // 2 + 1, q + N // 2 + 1)
            for a in range(P):
                bs = []
                for i, r in enumerate(rs):
                    vals = []
                    for c in range(r):
                        n = [m for m in range(P * r) if m % P == a and m % r == c][0]
                        y = Yt[i][n]
                        vals.append(y.real * y.real + y.imag * y.imag)
                    bs.append(int(np.argmax(vals)))
                hits = [om for om in window if om % P == a and all(om % r == b for r, b in zip(rs, bs))]
                assert len(hits) <= 1
                exp = hits[0] if hits and q - plan.w <= hits[0] < q + plan.w and plan.B_lo <= hits[0] <= plan.B_hi else SENTINEL
                assert ids.cand[a] == exp


def test_isolated_tone_identified_in_every_prime():
    """Noiseless single tone: every bucket prime reconstructs exactly omega (P5/P6)."""
    N = 4096
    plan = derive_plan(N, 8, OracleParams(seed=2))
    pl = planted(N, 1 + 1, cfg=15, trial=3)
    r = dsft(pl.f, 8, plan=plan, keep_bands=True)
    for om in pl.freqs:
        j = [jj for jj in range(plan.J) if plan.q[jj] - plan.w <= om < plan.q[jj] + plan.w][0]
        br = r.bands[j]
        for t in range(plan.T):
            assert br.ids[t].cand[om % plan.primes[t]] == om
        assert om in br.accepted


@pytest.mark.parametrize("N,s", [(64, 4), (97, 4), (128, 6), (255, 6), (512, 8)])
def test_end_to_end_vs_bruteforce_dft(N, s):
    """North-star oracle check 1: O(N^2) brute-force DFT on tiny N, exactly s-sparse:
    the output set is R_s^opt and coefficients match."""
    for trial in range(3):
        pl = planted(N, s, cfg=16, trial=trial)
        B, fh = centered_dft_bruteforce(pl.f)
        order = sorted(range(N), key=lambda k: (-abs(fh[k]), B[k]))[:s]
        ropt = sorted(B[k] for k in order)
        res = dsft(pl.f, s, OracleParams(seed=trial))
        assert sorted(res.freqs.tolist()) == ropt
        d = dict(zip(res.freqs.tolist(), res.coeffs))
        err = max(abs(d[int(B[k])] - fh[k]) for k in order)
        assert err < 1e-4


def test_exact_recovery_thm4_coefficient_bound():
    """Noiseless exactly-sparse input, THM4 preset: |c - fhat| <= sqrt2 * 3||f||_inf N^-r / tau
    (Theorem 4 + PAPER.md:592; the tail term vanishes)."""
    N, s = 4096, 8
    for r_exp in (1.0, 2.0):
        plan = derive_plan(N, s, OracleParams(preset="thm4", r=r_exp, seed=1))
        for trial in range(2):
            pl = planted(N, s, cfg=17, trial=trial)
            res = dsft(pl.f, s, plan=plan)
            assert sorted(res.freqs.tolist()) == pl.freqs.tolist()
            d = dict(zip(res.freqs.tolist(), res.coeffs))
            bound = math.sqrt(2) * 3 * np.max(np.abs(pl.f)) * N ** (-r_exp) / plan.tau
            err = max(abs(d[int(w)] - c) for w, c in zip(pl.freqs, pl.fhat))
            assert err <= bound, (err, bound)


def test_theorem5_bound_with_tails():
    """Theorem 5: ||fhat - v||_2 <= ||fhat - fhat_s^opt||_2
    + 33/sqrt(s) ||fhat - fhat_s^opt||_1 + 198 sqrt(s) ||f||_inf N^-r (SPEC.md:462 setup)."""
    N, s, tail = 4096, 16, 48
    plan = derive_plan(N, s, OracleParams(preset="thm4", r=2.0, seed=3))
    for trial in range(3):
        pl = planted_with_tail(N, s, tail, 0.01, cfg=18, trial=trial)
        res = dsft(pl.f, s, plan=plan)
        dense = dict(zip(pl.freqs.tolist(), pl.fhat))
        mags = sorted(((abs(v), w) for w, v in dense.items()), key=lambda p: (-p[0], p[1]))
        head = {w for _, w in mags[:s]}
        tail_v = np.array([dense[w] for w in dense if w not in head])
        v = dict(zip(res.freqs.tolist(), res.coeffs))
        diff = [dense.get(w, 0) - v.get(w, 0) for w in set(dense) | set(v)]
        lhs = np.linalg.norm(diff)
        rhs = (np.linalg.norm(tail_v) + 33 / math.sqrt(s) * np.sum(np.abs(tail_v))
               + 198 * math.sqrt(s) * np.max(np.abs(pl.f)) * N ** -2.0)
        assert lhs <= rhs


def test_merge_bruteforce():
    plan = derive_plan(4096, 6, OracleParams())
    rng = np.random.default_rng(3)
    oms = rng.choice(np.arange(-2047, 2049), 40, replace=False).tolist()
    cs = [complex(x, y) for x, y in rng.integers(-3, 4, (40, 2))]  # many ties
    f, c, _ = merge(plan, oms, cs)
    ref = sorted([(abs(z) ** 2, w, z) for w, z in zip(oms, cs) if z != 0], key=lambda p: (-p[0], p[1]))[:6]
    assert f.tolist() == [w for _, w, _ in ref] and list(c) == [z for _, _, z in ref]


def test_zero_input_and_determinism_and_scaling():
    N, s = 4096, 8
    plan = derive_plan(N, s, OracleParams(seed=9))
    res0 = dsft(np.zeros(N, dtype=np.complex128), s, plan=plan)
    assert res0.freqs.size == 0
    pl = planted(N, s, cfg=20, trial=0)
    a = dsft(pl.f, s, plan=plan)
    b = dsft(pl.f.copy(), s, plan=plan)
    assert np.array_equal(a.freqs, b.freqs) and np.array_equal(a.coeffs, b.coeffs)
    c = dsft(2.0 * pl.f, s, plan=plan)  # exact power-of-two scaling is exact in every stage
    assert np.array_equal(c.freqs, a.freqs) and np.array_equal(c.coeffs, 2.0 * a.coeffs)


@pytest.mark.parametrize("N,s", [(1024, 12), (4096, 16), (4096, 30)])
def test_deterministic_variant_vs_bruteforce_dft(N, s):
    """Reading R13, the deterministic variant (n_bucket_primes = 0: every pool prime,
    PAPER.md:40-44, 604-610; vote_min = 0: more than half): exactly
    s-sparse input, the output set is R_s^opt of the O(N^2) brute-force DFT."""
    prm = OracleParams(n_bucket_primes=0, vote_min=0, pool_rule="smooth")
    plan = derive_plan(N, s, prm)
    assert len(plan.primes) > 5 and plan.vote_min == len(plan.primes) // 2 + 1
    for trial in range(2):
        pl = planted(N, s, cfg=19, trial=trial)
        B, fh = centered_dft_bruteforce(pl.f)
        order = sorted(range(N), key=lambda k: (-abs(fh[k]), B[k]))[:s]
        res = dsft(pl.f, s, plan=plan)
        assert sorted(res.freqs.tolist()) == sorted(B[k] for k in order)
        d = dict(zip(res.freqs.tolist(), res.coeffs))
        assert max(abs(d[int(B[k])] - fh[k]) for k in order) < 1e-4
