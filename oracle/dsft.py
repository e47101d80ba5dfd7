"""Algorithm 1 of PAPER.md (test infrastructure only; see oracle/__init__.py).

Steps, in the paper's order (DESIGN.md §3 lists the readings R1-R12):

  O2 filtered_samples  Algorithm 1 lines 5-7 with the
                       truncated semi-discrete sum of Lemma 10 / Theorem 4
                        and the centre-q modulation (R1).
  O3 alias_dft         the aliasing measurement E_j of PAPER.md:845-854.
  O4 identify          "more than half" identification (PAPER.md:161-164,
                       863-872) as residue argmax + CRT (reading R7, R8).
  O5 vote              majority over bucket primes (R9) and the passband
                       restriction of Algorithm 1 line 10.
  O6 estimate          separate real/imaginary medians ("sqrt 2",
                       872-874; R10), the s-sparse output of line 9 (R11),
                       unbiasing of line 11.
  O7 merge             line 13 with the tie rule of PAPER.md:113.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .filt import ghat
from .numtheory import crt
from .params import OracleParams, Plan, derive_plan


# --------------------------------------------------------------------------- O2
def nearest_grid_index(k, N: int, L: int):
    """j' = argmin_j |x_k - y_j| (Lemma 10) for the nodes
    x_k = -pi + 2 pi k / L and the grid y_j = -pi + 2 pi j / N:
    |x_k - y_j| = 2 pi |kN - jL| / (NL), minimised by j = round(kN / L), computed
    exactly in integers as floor((2kN + L) / (2L)).  L odd: no ties (reading R3)."""
    k = np.asarray(k, dtype=np.int64)
    return (2 * k * N + L) // (2 * L)


def filtered_samples(f: np.ndarray, plan: Plan, q: int, L: int, m: int = 0) -> np.ndarray:
    """h_q(x_k) for the L nodes x_k = -pi + 2 pi k / L + 2 pi m / N, k = 0..L-1
    (m = 0: the aliasing grid itself; m > 0: the grid shifted by m steps of f, the
    shifted measurements of the CLW-style inner SFT, reading R14).

    h_q(x) = (1/N) sum_{u=-kappa..kappa} f_{(j'+u) mod N} exp(i q d_u) g(d_u),
    d_u = x - y_{j'+u},  j' = argmin_j |x - y_j|  (Lemma 10, PAPER.md:454-457;
    indices mod N as in PAPER.md:477), g restricted to its n = 0 image (R5),
    modulation exp(+i q d) so that the passband is centred at q (R1).
    j' = round(kN/L) computed exactly in integers; L is odd so no ties (R3).  A shift
    by m whole steps of f moves the nearest grid point by exactly m: j' + m.
    The offset d_u is formed from the exact integer num = kN + mL - jL.
    """
    N = plan.N
    c1 = plan.c1
    NL = N * L
    k = np.arange(L, dtype=np.int64)
    jp = nearest_grid_index(k, N, L) + m
    acc = np.zeros(L, dtype=np.complex128)
    for u in range(-plan.kappa, plan.kappa + 1):
        j = jp + u
        num = k * N + m * L - j * L
        d = 2.0 * math.pi * num / NL
        G = np.exp(-(d * d) / (2.0 * c1 * c1)) / c1
        rho = (q * num) % NL
        phase = np.exp(2j * math.pi * rho / NL)
        acc += f[j % N] * G * phase
    return acc / N


# --------------------------------------------------------------------------- O3
def alias_dft(h: np.ndarray) -> np.ndarray:
    """E[b] = (1/L) sum_k h(x_k) exp(-2 pi i k b / L), b = 0..L-1."""
    return np.fft.fft(h) / h.shape[0]


def band_measurements(f: np.ndarray, plan: Plan, j: int) -> list[list[np.ndarray]]:
    """Y[t][i] = alias_dft(filtered_samples(f, q_j, L_{t,i})) for every grid.
    CLW (reading R14): Y[t][sigma] for the grid of length P_t shifted by m_sigma."""
    q = plan.q[j]
    if plan.inner == "clw":
        return [[alias_dft(filtered_samples(f, plan, q, plan.primes[t], m)) for m in plan.shifts[t]]
                for t in range(plan.T)]
    return [[alias_dft(filtered_samples(f, plan, q, L)) for L in plan.grid_lengths(t)]
            for t in range(plan.T)]


# --------------------------------------------------------------------------- O4
@dataclass
class Identification:
    cand: np.ndarray        # int64[P_t]: omega' per bucket, or SENTINEL
    gap: np.ndarray         # float64[P_t]: min over i of relative argmax gap


SENTINEL = np.iinfo(np.int64).min


def crt_coefficients(moduli: list[int]) -> list[int]:
    """e_m with CRT(res) = sum res_m e_m mod prod(moduli) (textbook CRT)."""
    M = 1
    for m in moduli:
        M *= m
    return [(M // m) * pow(M // m, -1, m) % M for m in moduli]


def residue_bin(a, c, P: int, r: int):
    """Index n < P r with n = a (mod P), n = c (mod r)."""
    e = crt_coefficients([P, r])
    return (np.asarray(a, dtype=np.int64) * e[0] + np.asarray(c, dtype=np.int64) * e[1]) % (P * r)


def identify(plan: Plan, j: int, t: int, Yt: list[np.ndarray]) -> Identification:
    """Reading R7 of the "more than half" identification.

    For each bucket a in [0, P_t) and residue prime r_i: b_i = argmax over
    c < r_i of |E_{t,i}[n(a, c)]|^2 (computed re*re + im*im, ties -> smallest c);
    R = CRT(a mod P_t, b_1 mod r_1, ...) in [0, M_t); omega' = the unique
    integer = R (mod M_t) in the window q + B (R8; none if absent); kept only
    if omega' lies in the passband [q - w, q + w) cap B (line 10).
    """
    P = plan.primes[t]
    rs = plan.residues[t]
    q = plan.q[j]
    N = plan.N
    a = np.arange(P, dtype=np.int64)
    res = [a]
    gap = np.full(P, np.inf)
    for i, r in enumerate(rs):
        c = np.arange(r, dtype=np.int64)
        n = residue_bin(a[:, None], c[None, :], P, r)
        Y = Yt[i][n]
        mag = Y.real * Y.real + Y.imag * Y.imag
        b = np.argmax(mag, axis=1)
        res.append(b.astype(np.int64))
        srt = np.sort(mag, axis=1)
        top1, top2 = srt[:, -1], srt[:, -2]
        with np.errstate(divide="ignore", invalid="ignore"):
            g = np.where(top1 > 0, (top1 - top2) / top1, np.inf)
        gap = np.minimum(gap, g)
    moduli = [P] + list(rs)
    M = 1
    for m in moduli:
        M *= m
    e = crt_coefficients(moduli)
    R = np.zeros(P, dtype=np.int64)
    for rr, em in zip(res, e):
        R = (R + rr * em) % M
    om = window_representative(R, M, q, N)
    ok = om != SENTINEL
    ok &= (om >= q - plan.w) & (om < q + plan.w) & (om >= plan.B_lo) & (om <= plan.B_hi)
    cand = np.where(ok, om, SENTINEL)
    return Identification(cand=cand, gap=gap)


def clw_decode(E: list[complex], shifts: list[int], b: int, P: int, q: int, N: int) -> tuple[int, float]:
    """Reading R14 (the CLW-style phase-encoding identification, SPEC.md
    Design Decisions of the inner SFT): one bucket b of a length-P grid.  For an
    isolated omega' in bucket b the shifted measurements satisfy
    E_sigma[b] = E_0[b] exp(2 pi i omega' m_sigma / N) (aliasing identity,
    PAPER.md:847, on the shifted grid), so with n = omega' - lo, lo = min(q + B):
      theta_sigma = arg(E_sigma conj(E_0)) / (2 pi) = m_sigma n / N + m_sigma lo / N  (mod 1).
    Scales m = 1, 2, 4, ... refine v ~ n / N coarse to fine: the first gives
    v = phi = theta - frac(m lo / N) (mod 1); each next one v <- (phi + k) / m with the
    integer k nearest to m v - phi.  The phases fix n only modulo N, so the estimate
    n_est = N (v mod 1) is circular: the bucket fixes the low digits by taking, over the
    three lifts n_est - N, n_est, n_est + N, the integer c = b - lo (mod P) nearest to
    each that lies in [0, N), and keeping the closest.  omega' = lo + c.  Returns
    (omega' or SENTINEL for an empty bucket, decision margin: the smallest distance of a
    rounded quantity from its rounding boundary, in units of its step)."""
    E0 = E[0]
    if E0.real == 0.0 and E0.imag == 0.0:
        return SENTINEL, math.inf
    lo = q - (N + 1) // 2 + 1
    v = None
    margin = math.inf
    for Es, m in zip(E[1:], shifts[1:]):
        r = Es * E0.conjugate()
        theta = math.atan2(r.imag, r.real) / (2.0 * math.pi)
        phi = (theta - ((m * lo) % N) / N) % 1.0
        if v is None:
            v = phi
        else:
            x = m * v - phi
            k = math.floor(x + 0.5)
            margin = min(margin, abs(abs(x - k) - 0.5))
            v = (phi + k) / m
    n_est = N * (v % 1.0)
    rb = (b - lo) % P
    best, d1, d2 = None, math.inf, math.inf
    for lift in (-N, 0, N):
        y = (n_est + lift - rb) / P
        c = rb + P * math.floor(y + 0.5)
        margin = min(margin, abs(abs(y - math.floor(y + 0.5)) - 0.5))
        if 0 <= c < N:
            dist = abs(c - (n_est + lift))
            if dist < d1:
                best, d1, d2 = c, dist, d1
            elif dist < d2:
                d2 = dist
    if best is None:
        return SENTINEL, margin
    if d2 < math.inf:
        margin = min(margin, (d2 - d1) / P)
    return lo + best, margin


def identify_clw(plan: Plan, j: int, t: int, Et: list[np.ndarray]) -> Identification:
    """Reading R14 identification for bucket prime t of band j: clw_decode in every
    bucket b < P_t (here elementwise over the buckets with numpy, the same operations
    in the same order; pinned to the scalar clw_decode by
    tests/test_oracle_clw.py::test_identify_clw_matches_decode_per_bucket), kept only
    if omega' lies in the passband [q - w, q + w) cap B (line 10)."""
    P = plan.primes[t]
    q = plan.q[j]
    N = plan.N
    shifts = plan.shifts[t]
    b = np.arange(P, dtype=np.int64)
    E0 = Et[0]
    live = ~((E0.real == 0.0) & (E0.imag == 0.0))
    lo = q - (N + 1) // 2 + 1
    gap = np.full(P, np.inf)
    v = None
    for Es, m in zip(Et[1:], shifts[1:]):
        re = Es.real * E0.real + Es.imag * E0.imag          # Es conj(E0), no contraction
        im = Es.real * (-E0.imag) + Es.imag * E0.real
        theta = np.arctan2(im, re) / (2.0 * math.pi)
        phi = (theta - ((m * lo) % N) / N) % 1.0
        if v is None:
            v = phi
        else:
            x = m * v - phi
            k = np.floor(x + 0.5)
            gap = np.minimum(gap, np.abs(np.abs(x - k) - 0.5))
            v = (phi + k) / m
    n_est = N * (v % 1.0)
    rb = (b - lo) % P
    best = np.full(P, -1, dtype=np.int64)
    d1 = np.full(P, np.inf)
    d2 = np.full(P, np.inf)
    for lift in (-N, 0, N):
        y = (n_est + lift - rb) / P
        fl = np.floor(y + 0.5)
        gap = np.minimum(gap, np.abs(np.abs(y - fl) - 0.5))
        c = rb + P * fl.astype(np.int64)
        ok = (c >= 0) & (c < N)
        dist = np.abs(c - (n_est + lift))
        better = ok & (dist < d1)
        second = ok & ~better & (dist < d2)
        d2 = np.where(better, d1, np.where(second, dist, d2))
        best = np.where(better, c, best)
        d1 = np.where(better, dist, d1)
    with np.errstate(invalid="ignore"):  # (inf - inf where no second candidate: not used)
        gap = np.where(np.isfinite(d2), np.minimum(gap, (d2 - d1) / P), gap)
    om = lo + best
    ok = live & (best >= 0)
    ok &= (om >= q - plan.w) & (om < q + plan.w) & (om >= plan.B_lo) & (om <= plan.B_hi)
    gap = np.where(live, gap, np.inf)
    return Identification(cand=np.where(ok, om, SENTINEL), gap=gap)


def window_representative(R, M: int, q: int, N: int):
    """The unique integer omega' = R (mod M) in the window
    q + B = (q - ceil(N/2), q + floor(N/2)] (B of PAPER.md:84 shifted to the band
    centre; reading R7 / G4), or SENTINEL if the window holds none.  M >= N
    (reading R8), so the window of N consecutive integers holds at most one."""
    R = np.asarray(R, dtype=np.int64)
    lo = q - (N + 1) // 2 + 1          # smallest element of q + B
    hi = q + N // 2                    # largest element of q + B
    om = lo + (R - lo) % M             # smallest integer >= lo congruent to R
    return np.where(om <= hi, om, SENTINEL)


# --------------------------------------------------------------------------- O5
def voters(plan: Plan, ids: list[Identification], omega: int) -> list[int]:
    """Bucket primes t whose identification produced omega."""
    return [t for t in range(plan.T) if ids[t].cand[omega % plan.primes[t]] == omega]


def vote(plan: Plan, ids: list[Identification]) -> list[int]:
    """Reading R9: accept omega if at least v_min distinct bucket primes
    produced it ("more than half").  Returned ascending."""
    seen = set()
    for t in range(plan.T):
        for om in ids[t].cand[ids[t].cand != SENTINEL].tolist():
            seen.add(om)
    return sorted(om for om in seen if len(voters(plan, ids, om)) >= plan.vote_min)


# --------------------------------------------------------------------------- O6
def estimate(plan: Plan, j: int, Y: list[list[np.ndarray]], ids: list[Identification],
             accepted: list[int]) -> tuple[list[int], list[complex], list[complex], list[float]]:
    """Reading R10: z_omega = median Re(v) + i median Im(v) over
    v_{t,i} = (-1)^omega E_{t,i}[omega mod L_{t,i}] for the voting t and all i
    (PAPER.md:167, 872-874); np.median averages the two middle values for even
    counts.  Line 9's s-sparse output (R11): keep the band_budget largest |z|^2
    (ties -> smaller omega).  Line 11 (R1): c = z / ghat_{omega-q}.
    Returns (omegas, c, z, boundary_gap)."""
    q = plan.q[j]
    zs = []
    for om in accepted:
        vals = []
        sgn = -1.0 if om % 2 else 1.0
        for t in voters(plan, ids, om):
            for i, L in enumerate(plan.grid_lengths(t)):
                vals.append(sgn * Y[t][i][om % L])
        v = np.array(vals, dtype=np.complex128)
        zs.append(complex(np.median(v.real), np.median(v.imag)))
    mags = [z.real * z.real + z.imag * z.imag for z in zs]
    order = sorted(range(len(accepted)), key=lambda k: (-mags[k], accepted[k]))
    keep = order[:plan.band_budget]
    gaps = []
    if len(order) > plan.band_budget and plan.band_budget > 0:
        m1, m2 = mags[order[plan.band_budget - 1]], mags[order[plan.band_budget]]
        gaps.append((m1 - m2) / m1 if m1 > 0 else math.inf)
    oms = [accepted[k] for k in keep]
    z_keep = [zs[k] for k in keep]
    cs = [z / float(ghat(om - q, plan.c1)) for om, z in zip(oms, z_keep)]
    return oms, cs, z_keep, gaps


# --------------------------------------------------------------------------- O7
def merge(plan: Plan, oms: list[int], cs: list[complex]) -> tuple[np.ndarray, np.ndarray, float]:
    """Algorithm 1 line 13: the s largest |c| over the union of
    bands, ties -> smaller omega; exact zeros dropped (R12)."""
    assert len(set(oms)) == len(oms), "passbands partition B: no duplicates"
    items = [(om, c) for om, c in zip(oms, cs) if not (c.real == 0.0 and c.imag == 0.0)]
    mags = [c.real * c.real + c.imag * c.imag for _, c in items]
    order = sorted(range(len(items)), key=lambda k: (-mags[k], items[k][0]))
    gap = math.inf
    if len(order) > plan.s:
        m1, m2 = mags[order[plan.s - 1]], mags[order[plan.s]]
        gap = (m1 - m2) / m1 if m1 > 0 else math.inf
    order = order[:plan.s]
    freqs = np.array([items[k][0] for k in order], dtype=np.int64)
    coeffs = np.array([items[k][1] for k in order], dtype=np.complex128)
    return freqs, coeffs, gap


# ---------------------------------------------------------------------- driver
@dataclass
class BandResult:
    q: int
    ids: list[Identification]
    accepted: list[int]
    omegas: list[int]
    coeffs: list[complex]
    z: list[complex]
    margin: float


@dataclass
class DsftResult:
    freqs: np.ndarray
    coeffs: np.ndarray
    plan: Plan
    bands: list[BandResult] = field(default_factory=list)
    margin: float = math.inf


def process_band(f: np.ndarray, plan: Plan, j: int) -> BandResult:
    """Algorithm 1 lines 4-12 for band j (0-based)."""
    Y = band_measurements(f, plan, j)
    if plan.inner == "clw":  # reading R14; the estimate reads the unshifted grid (Y[t][0])
        ids = [identify_clw(plan, j, t, Y[t]) for t in range(plan.T)]
        Y = [[Y[t][0]] for t in range(plan.T)]
    else:
        ids = [identify(plan, j, t, Y[t]) for t in range(plan.T)]
    accepted = vote(plan, ids)
    oms, cs, zs, gaps = estimate(plan, j, Y, ids, accepted)
    # margin audit: argmax gaps in every bucket that can touch an accepted or
    # near-accepted omega (votes >= v_min - 1), plus the band-budget boundary.
    near = set(accepted)
    for t in range(plan.T):
        for om in ids[t].cand[ids[t].cand != SENTINEL].tolist():
            if len(voters(plan, ids, om)) >= plan.vote_min - 1:
                near.add(om)
    margin = min(gaps) if gaps else math.inf
    for om in near:
        for t in range(plan.T):
            margin = min(margin, float(ids[t].gap[om % plan.primes[t]]))
    return BandResult(q=plan.q[j], ids=ids, accepted=accepted, omegas=oms, coeffs=cs, z=zs,
                      margin=margin)


def dsft(f: np.ndarray, s: int, params: OracleParams | None = None, plan: Plan | None = None,
         keep_bands: bool = False) -> DsftResult:
    """Algorithm 1: returns the s-sparse approximation of
    fhat = F f (PAPER.md:82 convention) as (freqs, coeffs), sorted by
    (|c| desc, omega asc)."""
    if isinstance(f, np.ndarray):  # (tests may pass an object that evaluates f lazily by index)
        f = np.ascontiguousarray(f, dtype=np.complex128)
    if plan is None:
        plan = derive_plan(f.shape[0], s, params)
    all_om, all_c, bands = [], [], []
    margin = math.inf
    for j in range(plan.J):
        br = process_band(f, plan, j)
        all_om += br.omegas
        all_c += br.coeffs
        margin = min(margin, br.margin)
        if keep_bands:
            bands.append(br)
    freqs, coeffs, gap = merge(plan, all_om, all_c)
    return DsftResult(freqs=freqs, coeffs=coeffs, plan=plan, bands=bands, margin=min(margin, gap))


def crt_reconstruct(residues: list[int], moduli: list[int]) -> int:
    """Scalar CRT (re-export for tests)."""
    return crt(residues, moduli)
