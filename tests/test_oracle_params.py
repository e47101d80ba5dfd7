"""Pins for oracle/params.py and oracle/numtheory.py (CPU only)."""

import json
import math
import os

import numpy as np
import pytest

from oracle.filt import ghat
from oracle.numtheory import SplitMix64, crt, draw_distinct, largest_prime_factor, primes_below
from oracle.params import (ConfigError, OracleParams, bucket_pool, derive_plan, passband_plan)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_values.json")))


def test_kappa_thm4_worked_value():
    p = derive_plan(4096, 8, OracleParams(preset="thm4", r=1.0))
    assert p.kappa == GOLD["kappa_thm4_N4096_r1"]["value"]
    assert p.beta == 6.0


def test_passband_worked_value():
    w, J, q = passband_plan(4096, 2.0)
    g = GOLD["passband_N4096_alpha2"]
    assert (w, J, q[0]) == (g["w"], g["J"], g["q1"])


@pytest.mark.parametrize("row", GOLD["appendixB_dmsft6"])
def test_appendix_b_dmsft6(row):
    p = derive_plan(row["N"], 8 if row["N"] < 10**5 else 50)
    assert abs(p.beta - row["beta"]) < 1e-3
    assert abs(p.alpha - row["alpha"]) < 1e-2
    assert (p.w, p.J, p.kappa) == (row["w"], row["J"], 6)


@pytest.mark.parametrize("row", GOLD["appendixB_thm4"])
def test_appendix_b_thm4(row):
    p = derive_plan(row["N"], 8 if row["N"] < 10**5 else 50, OracleParams(preset="thm4"))
    assert (p.kappa, p.w, p.J) == (row["kappa"], row["w"], row["J"])
    if "J_literal" in row:
        pl = derive_plan(row["N"], 50, OracleParams(preset="thm4", alpha_rule="literal"))
        assert pl.J == row["J_literal"]


@pytest.mark.parametrize("N", [64, 97, 1000, 4096, 2**14, 6000011])
@pytest.mark.parametrize("preset", ["dmsft6", "dmsft4", "thm4"])
def test_lemma3_passband_and_partition(N, preset):
    """Lemma 3: ghat in [tau, 1/sqrt(2pi)] on |omega| <= w, exhaustively;
    the passbands [q_j - w, q_j + w) partition B (Algorithm 1 line 10)."""
    p = derive_plan(N, 8, OracleParams(preset=preset))
    om = np.arange(-p.w, p.w + 1)
    gh = ghat(om, p.c1)
    assert gh.min() >= p.tau and gh.max() <= 1 / math.sqrt(2 * math.pi) + 1e-16
    # Lemma 3's exact constraint on beta
    assert p.beta <= p.alpha * math.sqrt(math.log(1 / (p.tau * math.sqrt(2 * math.pi))) / 2) + 1e-12
    # partition of B
    assert p.q[0] - p.w == p.B_lo
    for a, b in zip(p.q, p.q[1:]):
        assert a + p.w == b - p.w
    assert p.q[-1] + p.w > p.B_hi
    assert 2 * p.J * p.w >= N


def test_lemma3_literal_alpha_also_admissible():
    p = derive_plan(4096, 8, OracleParams(preset="thm4", alpha_rule="literal"))
    gh = ghat(np.arange(-p.w, p.w + 1), p.c1)
    assert gh.min() >= p.tau


def test_splitmix64_reference_vectors():
    for key, seed in (("splitmix64_seed0", 0), ("splitmix64_seed1234567", 1234567)):
        g = SplitMix64(seed)
        assert [g.next() for _ in GOLD[key]["values"]] == [int(v, 16) for v in GOLD[key]["values"]]


def _is_prime_naive(n):
    return n >= 2 and all(n % d for d in range(2, int(n ** 0.5) + 1))


def test_sieve_and_factor_bruteforce():
    assert primes_below(200) == [n for n in range(200) if _is_prime_naive(n)]
    for n in range(2, 3000):
        f = [d for d in range(2, n + 1) if n % d == 0 and _is_prime_naive(d)]
        assert largest_prime_factor(n) == max(f)


def test_crt_bruteforce():
    rng = np.random.default_rng(5)
    moduli = [7, 3, 5, 11]
    M = 7 * 3 * 5 * 11
    for _ in range(200):
        x = int(rng.integers(0, M))
        assert crt([x % m for m in moduli], moduli) == x


def test_pool_rule_bruteforce():
    for s in (4, 8, 50, 100):
        pool = bucket_pool(s, 4.0)
        ref = [p for p in range(4 * s, 8 * s) if _is_prime_naive(p)
               and max(d for d in range(2, p) if (p - 1) % d == 0 and _is_prime_naive(d)) <= 13]
        assert pool == ref


@pytest.mark.parametrize("s", [4, 8, 50, 1000])
def test_full_pool_is_every_prime_in_range(s):
    """Reading R6, DSFT_POOL_FULL: every prime in [ceil(c_b s), 2 ceil(c_b s))
    by trial division (a random subset of the deterministic
    measurements); the smooth pool is its subset with 13-smooth P - 1."""
    ref = [p for p in range(4 * s, 8 * s) if _is_prime_naive(p)]
    assert bucket_pool(s, 4.0, "full") == ref
    assert set(bucket_pool(s, 4.0, "smooth")) <= set(ref)
    assert derive_plan(2**20, max(s, 8), OracleParams(pool_rule="full")).pool == bucket_pool(max(s, 8), 4.0, "full")


def test_draw_is_distinct_sorted_seeded():
    pool = bucket_pool(1000, 4.0)
    a = draw_distinct(pool, 5, 7)
    assert a == sorted(set(a)) and len(a) == 5 and set(a) <= set(pool)
    assert a == draw_distinct(pool, 5, 7)
    assert any(draw_distinct(pool, 5, sd) != a for sd in range(8, 20))
    # partial Fisher-Yates spelled out independently
    g = SplitMix64(7)
    work = list(pool)
    for i in range(5):
        j = i + g.next() % (len(work) - i)
        work[i], work[j] = work[j], work[i]
    assert a == sorted(work[:5])


def _brute_residues(P, N):
    """Independent brute force of reading R8: depth-first over ascending subsets of
    the odd primes below min(P, 32); minimise (sum(r - 1), count, lexicographic)."""
    ps = [r for r in range(3, 32) if all(r % d for d in range(2, r)) and r < P]
    best = []

    def dfs(i, chosen, prod):
        if prod * P >= N and chosen:
            key = (sum(r - 1 for r in chosen), len(chosen), tuple(chosen))
            if not best or key < best[0]:
                best[:] = [key]
        for k in range(i, len(ps)):
            dfs(k + 1, chosen + [ps[k]], prod * ps[k])

    dfs(0, [], 1)
    return list(best[0][2]) if best else None


@pytest.mark.parametrize("N,s,seed", [(2**26, 1000, 3), (2**26, 1000, 0), (2**22, 50, 1), (4096, 8, 0),
                                      (6000011, 100, 2), (2**24, 256, 5), (2**21, 4000, 1), (64, 4, 0)])
def test_residue_rule(N, s, seed):
    """Reading R8: the CRT window is unique (P prod r >= N) with the fewest extra
    measurement rows sum (r - 1); checked against an independent brute force."""
    p = derive_plan(N, s, OracleParams(seed=seed))
    for P, rs in zip(p.primes, p.residues):
        assert math.prod(rs) * P >= N
        assert rs == sorted(rs) and all(r < P for r in rs) and len(set(rs)) == len(rs)
        assert rs == _brute_residues(P, N)


def test_residue_rule_headline_values():
    """BASELINE config 2 (N = 2^26, s = 1000, seed 0): P = 4051, 4057, 4357 need
    prod r >= 16567, 16542, 15403 -> {3,5,7,11,17} (38 extra rows) rather than the
    consecutive {3,...,17} (50); P = 4951, 7561 -> {3,5,7,11,13} (13-smooth pool)."""
    p = derive_plan(2**26, 1000, OracleParams(seed=0, pool_rule="smooth"))
    assert p.primes == [4051, 4057, 4357, 4951, 7561]
    assert p.residues == [[3, 5, 7, 11, 17]] * 3 + [[3, 5, 7, 11, 13]] * 2


@pytest.mark.parametrize("bad", [
    dict(N=30, s=4), dict(N=4096, s=1), dict(N=4096, s=4097),
    dict(N=4096, s=8, params=OracleParams(tau=0.5)),
    dict(N=4096, s=8, params=OracleParams(preset="thm4", r=0.5)),
    dict(N=4096, s=3),  # pool [12, 24) has < 5 smooth primes
    dict(N=4096, s=8, params=OracleParams(vote_min=6)),
])
def test_config_errors(bad):
    with pytest.raises(ConfigError):
        derive_plan(bad["N"], bad["s"], bad.get("params"))


@pytest.mark.parametrize("s", [8, 50, 300, 1000])
def test_deterministic_variant_plan(s):
    """Reading R13: n_bucket_primes = 0 takes every prime of the pool (brute-force pool
    rule, no draw, independent of the seed); vote_min = 0 is floor(T/2) + 1."""
    ref = [p for p in range(4 * s, 8 * s) if _is_prime_naive(p)
           and max(d for d in range(2, p) if (p - 1) % d == 0 and _is_prime_naive(d)) <= 13]
    for seed in (0, 7):
        p = derive_plan(2**20, s, OracleParams(n_bucket_primes=0, vote_min=0, seed=seed, pool_rule="smooth"))
        assert p.primes == ref and p.vote_min == len(ref) // 2 + 1
    assert derive_plan(2**20, s, OracleParams(n_bucket_primes=0, vote_min=2, pool_rule="smooth")).vote_min == 2
