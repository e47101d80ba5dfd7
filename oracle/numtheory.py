"""Integer helpers for the oracle (test infrastructure only; see oracle/__init__.py).

The paper's inner SFT measures the signal on prime-length aliasing grids
(eq. DFT_GKlam_Comp: lengths s_j, "a randomly chosen subset"
of the deterministic measurements).  The prime draw, the CRT
reconstruction and the counter-based generator below are the plain definitions.
"""

from __future__ import annotations

MASK64 = (1 << 64) - 1


class SplitMix64:
    """SplitMix64 counter-based generator (Steele, Lea, Flood 2014).

    The randomized variant draws its bucket primes from a seed (PAPER.md:175:
    "reads only a randomly chosen subset").  Both the oracle and the CUDA
    plan implement this same generator independently, so the same seed draws
    the same primes on both sides (R7).
    """

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)


def primes_below(hi: int) -> list[int]:
    """All primes p < hi by the sieve of Eratosthenes."""
    if hi <= 2:
        return []
    sieve = bytearray([1]) * hi
    sieve[0] = sieve[1] = 0
    i = 2
    while i * i < hi:
        if sieve[i]:
            sieve[i * i::i] = bytearray(len(range(i * i, hi, i)))
        i += 1
    return [p for p in range(hi) if sieve[p]]


def largest_prime_factor(n: int) -> int:
    """Largest prime factor of n >= 2 by trial division."""
    best = 1
    d = 2
    while d * d <= n:
        while n % d == 0:
            best = d
            n //= d
        d += 1
    if n > 1:
        best = max(best, n)
    return best


def crt(residues: list[int], moduli: list[int]) -> int:
    """The unique R in [0, prod(moduli)) with R = residues[i] (mod moduli[i]).

    Moduli must be pairwise coprime.  Written as the textbook constructive
    proof of the Chinese remainder theorem (used by identification, O4).
    """
    M = 1
    for m in moduli:
        M *= m
    R = 0
    for a, m in zip(residues, moduli):
        Mi = M // m
        R += (a % m) * Mi * pow(Mi, -1, m)
    return R % M


def draw_distinct(pool: list[int], count: int, seed: int) -> list[int]:
    """Draw `count` distinct entries of `pool` with a partial Fisher-Yates
    shuffle driven by SplitMix64(seed): step i swaps entry i with entry
    i + (next() mod (n - i)).  Returned sorted ascending (R7)."""
    work = list(pool)
    n = len(work)
    rng = SplitMix64(seed)
    for i in range(count):
        j = i + rng.next() % (n - i)
        work[i], work[j] = work[j], work[i]
    return sorted(work[:count])
