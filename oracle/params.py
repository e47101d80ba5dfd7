"""Parameter derivation for Algorithm 1 (test infrastructure only).

Follows PAPER.md:
  * Lemma 3: tau in (0, 1/sqrt(2 pi)), alpha in [1, N/sqrt(ln N)],
    beta <= alpha*sqrt(ln(1/(tau sqrt(2 pi)))/2), c1 = beta sqrt(ln N)/N.
  * Algorithm 1 line 2: c2 = alpha sqrt(ln N)/2; lines 3-4
    (PAPER.md:233-234): q_j = -ceil(N/2) + 1 + (2j-1) ceil(N/(alpha sqrt(ln N))),
    j = 1..ceil(c2).
  * Theorem 4: beta = 6 sqrt(r),
    kappa = ceil(6 r ln N/(sqrt(2) pi)) + 1  (preset THM4).
  * Section 5: DMSFT-4 / DMSFT-6 use kappa = 4 / 6 (presets).
  * Section 4: tau = 1/3 default; alpha from beta (reading R2).
Readings R1..R12 are listed in DESIGN.md §3.
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field

from .numtheory import draw_distinct, largest_prime_factor, primes_below

PRESET_DMSFT6 = "dmsft6"
PRESET_DMSFT4 = "dmsft4"
PRESET_THM4 = "thm4"

# Largest prime factor allowed in P-1 for a bucket prime P (reading R6: every
# bucket DFT is evaluated by the GPU as a Rader convolution over a mixed-radix
# FFT of length P-1; the oracle mirrors only the pool rule, not the algorithm).
RADER_SMOOTH = 13


class ConfigError(ValueError):
    """Invalid (N, s, params) combination (the C-ABI's DSFT_ERR_CONFIG)."""


@dataclass
class OracleParams:
    preset: str = PRESET_DMSFT6
    r: float = 1.0            # THM4 decay exponent
    kappa: int = 0            # 0 = preset value
    tau: float = 1.0 / 3.0
    alpha_rule: str = "corrected"  # reading R2; "literal" = PAPER.md:597 as printed
    bucket_factor: float = 4.0     # c_b (reading R6)
    n_bucket_primes: int = 5       # T   (reading R6); 0 = deterministic variant (reading R13)
    vote_min: int = 3              # v_min (reading R9: > T/2); 0 = floor(T/2) + 1
    band_budget: int = 0           # 0 = s (reading R11)
    seed: int = 0
    pool_rule: str = "smooth"      # reading R6: "full" = every prime of the range, "smooth" = 13-smooth P-1
    inner: str = "gfft"            # inner SFT of line 9: "gfft" (readings R7-R10) or "clw" (reading R14)


@dataclass
class Plan:
    N: int
    s: int
    preset: str
    kappa: int
    beta: float
    c1: float
    tau: float
    alpha: float
    w: int
    J: int
    q: list[int]
    B_lo: int            # smallest element of B = (-ceil(N/2), floor(N/2)]
    B_hi: int            # largest element of B
    pool: list[int]
    primes: list[int]    # P_t, t = 0..T-1, ascending
    residues: list[list[int]] = field(default_factory=list)  # r_{t,i}
    vote_min: int = 3
    band_budget: int = 0
    seed: int = 0
    inner: str = "gfft"
    shifts: list[list[int]] = field(default_factory=list)  # CLW (R14): grid shifts m_sigma per prime

    @property
    def T(self) -> int:
        return len(self.primes)

    def grid_lengths(self, t: int) -> list[int]:
        """Aliasing grid lengths L_{t,i} = P_t * r_{t,i} (s_j)."""
        return [self.primes[t] * r for r in self.residues[t]]


def odd_primes(count_hint: int = 64) -> list[int]:
    return [p for p in primes_below(512) if p > 2][:count_hint]


def bucket_pool(s: int, bucket_factor: float, rule: str = "smooth") -> list[int]:
    """Reading R6: the primes P in [ceil(c_b s), 2 ceil(c_b s)) ("full"), or only those
    whose P-1 has no prime factor above 13 ("smooth").  PAPER.md:175-177 / 845-850 fix
    only that the moduli are primes and that the randomized variant reads a random
    subset of the deterministic measurements."""
    lo = int(math.ceil(bucket_factor * s))
    hi = 2 * lo
    if rule == "full":
        return [p for p in primes_below(hi) if p >= lo]
    if rule != "smooth":
        raise ConfigError(f"unknown pool_rule {rule!r}")
    return [p for p in primes_below(hi) if p >= lo and largest_prime_factor(p - 1) <= RADER_SMOOTH]


def passband_plan(N: int, alpha: float) -> tuple[int, int, list[int]]:
    """Algorithm 1 lines 2-4: half-width
    w = ceil(N/(alpha sqrt(ln N))), J = ceil(c2) = ceil(alpha sqrt(ln N)/2) bands,
    centres q_j = -ceil(N/2) + 1 + (2j-1) w, j = 1..J."""
    lnN = math.log(N)
    w = int(math.ceil(N / (alpha * math.sqrt(lnN))))
    J = int(math.ceil(alpha * math.sqrt(lnN) / 2.0))
    halfN_up = (N + 1) // 2
    q = [-halfN_up + 1 + (2 * j - 1) * w for j in range(1, J + 1)]
    return w, J, q


RESIDUE_PRIME_MAX = 31


def residue_moduli(P: int, N: int) -> list[int]:
    """Reading R8: the residue primes r_i of bucket prime P are the
    set of distinct odd primes below min(P, 32) with P * prod r_i >= N (so the CRT
    window q + B of N integers holds exactly one representative)
    that minimises the extra measurement rows sum_i (r_i - 1) per bucket; ties ->
    fewer primes, then the lexicographically smallest ascending list.  At least one."""
    need = -(-N // P)
    cands = [r for r in odd_primes() if r <= RESIDUE_PRIME_MAX and r < P]
    best = None
    for k in range(1, len(cands) + 1):
        for combo in itertools.combinations(cands, k):
            if math.prod(combo) >= need:
                key = (sum(r - 1 for r in combo), k, combo)
                if best is None or key < best:
                    best = key
    if best is None:
        raise ConfigError("no set of residue primes below the bucket prime reaches N")
    return list(best[2])


def clw_shifts(P: int, N: int) -> list[int]:
    """Reading R14: the grid shifts m_sigma (in steps 2 pi / N of f) of the CLW-style
    inner SFT for bucket prime P: 0 (the unshifted grid), then 1, 2, 4, ..., 2^(L-1)
    with L = ceil(log2(N / P)) + 1, the fewest dyadic scales after which the frequency
    estimate is within P/4 of the truth whenever every phase error is below pi/2
    (so the congruence omega = b (mod P) fixes it)."""
    L = 1
    while (1 << (L - 1)) * P < N:
        L += 1
    return [0] + [1 << l for l in range(L)]


def derive_plan(N: int, s: int, params: OracleParams | None = None) -> Plan:
    """Derive every parameter Algorithm 1 needs."""
    p = params or OracleParams()
    if N < 36:
        raise ConfigError("N must be >= 36 (Theorem 4 needs N >= 36 r, PAPER.md:498)")
    if not (2 <= s <= N):
        raise ConfigError("s must lie in [2, N] (PAPER.md:40)")
    if not (0.0 < p.tau < 1.0 / math.sqrt(2.0 * math.pi)):
        raise ConfigError("tau must lie in (0, 1/sqrt(2 pi)) (Lemma 3, PAPER.md:149)")
    lnN = math.log(N)

    # beta and kappa (Theorem 4 / Section 5 presets; reading R4 for DMSFT).
    if p.preset == PRESET_THM4:
        if not (1.0 <= p.r <= N / 36.0):
            raise ConfigError("r must lie in [1, N/36] (PAPER.md:498)")
        beta = 6.0 * math.sqrt(p.r)
        kappa = int(math.ceil(6.0 * p.r * lnN / (math.sqrt(2.0) * math.pi))) + 1
    elif p.preset in (PRESET_DMSFT6, PRESET_DMSFT4):
        kappa = 6 if p.preset == PRESET_DMSFT6 else 4
        beta = None
    else:
        raise ConfigError(f"unknown preset {p.preset!r}")
    if p.kappa > 0:
        kappa = int(p.kappa)
    if beta is None:
        # R4: balance Lemma 10's truncation exponent 2 pi^2 kappa^2/(beta^2 ln N)
        # against Lemma 9's aliasing exponent beta^2 ln N / 8.
        beta = math.sqrt(4.0 * math.pi * kappa / lnN)
    if 2 * kappa + 2 > N:
        raise ConfigError("window 2 kappa + 2 must fit in N (SPEC.md:256)")

    c1 = beta * math.sqrt(lnN) / N  # Algorithm 1 line 2
    if not c1 < 0.5:
        raise ConfigError("c1 >= 0.5: periodization images not negligible (reading R5)")

    # alpha (Lemma 3 admissibility; reading R2 for the Section 4 typo).
    lg = math.log(1.0 / (p.tau * math.sqrt(2.0 * math.pi)))
    if p.alpha_rule == "corrected":
        alpha = beta / math.sqrt(lg / 2.0)
    elif p.alpha_rule == "literal":
        alpha = beta * math.sqrt(2.0) / lg
    else:
        raise ConfigError(f"unknown alpha_rule {p.alpha_rule!r}")
    alpha = min(max(alpha, 1.0), N / math.sqrt(lnN))

    w, J, q = passband_plan(N, alpha)
    B_lo = -((N + 1) // 2) + 1
    B_hi = N // 2

    # Inner SFT (reading R6-R8): bucket primes and residue primes.
    pool = bucket_pool(s, p.bucket_factor, p.pool_rule)
    if int(p.n_bucket_primes) == 0:
        # Reading R13, the deterministic variant (the
        # measurements "always succeed"; the randomized variant reads a random subset
        # of them): every prime of the pool, no draw.
        T = len(pool)
        primes = list(pool)
    else:
        T = int(p.n_bucket_primes)
        if T < 1:
            raise ConfigError("need at least one bucket prime")
        if len(pool) < T:
            raise ConfigError(f"bucket-prime pool has {len(pool)} < T={T} primes")
        primes = draw_distinct(pool, T, p.seed)
    if T < 1:
        raise ConfigError("need at least one bucket prime")
    if p.inner == "gfft":
        residues = [residue_moduli(P, N) for P in primes]
        shifts = []
    elif p.inner == "clw":
        # Reading R14: one grid of length P_t (residue list [1]) sampled unshifted and
        # shifted by m = 1, 2, 4, ..., 2^(L-1) steps of f, L = ceil(log2(N/P_t)) + 1
        residues = [[1] for _ in primes]
        shifts = [clw_shifts(P, N) for P in primes]
    else:
        raise ConfigError(f"unknown inner {p.inner!r}")
    # vote_min 0: "more than half" of the T primes
    vote_min = T // 2 + 1 if int(p.vote_min) == 0 else int(p.vote_min)
    if not (1 <= vote_min <= T):
        raise ConfigError("vote_min must lie in [1, T]")
    budget = int(p.band_budget) if p.band_budget > 0 else s

    return Plan(N=N, s=s, preset=p.preset, kappa=kappa, beta=beta, c1=c1, tau=p.tau,
                alpha=alpha, w=w, J=J, q=q, B_lo=B_lo, B_hi=B_hi, pool=pool, primes=primes,
                residues=residues, vote_min=vote_min, band_budget=budget, seed=int(p.seed),
                inner=p.inner, shifts=shifts)
