"""CPU oracle for the randomized discrete sparse Fourier transform of
Merhi, Zhang, Iwen, Christlieb, "A New Class of Fully Discrete Sparse Fourier
Transforms" (arXiv 1706.02740; `/root/reference/PAPER.md`).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path may import this
package: only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs call it.  It shares no code, tables
or constants with the CUDA path (`paper_1706_02740_b200/`); the only module
both sides use is the seeded input generator `dsft_synth/`, which holds none
of the method's arithmetic.

The oracle is plain numpy in float64 / complex128 and follows Algorithm 1
 step by step, with the inner randomized SFT 𝒜 (line 9)
given by the reading fixed in DESIGN.md §3 ("readings").  Every function cites
the passage it implements.  Pins (tests/test_oracle_*.py, `-m "not gpu"`)
check it against closed forms, brute force and the paper's bounds.

Parity status per function (DESIGN.md §4 lists the pin for each):
  conventions.*            pinned (brute-force F matrix)
  filt.ghat / filt.g       pinned (Lemma 2 vs quadrature of eq. (4))
  params.derive_plan       pinned (worked values, Lemma 3 exhaustive, coverage)
  numtheory.*              pinned (brute-force CRT / sieve / SplitMix64 vectors)
  dsft.nearest_grid_index  pinned (brute-force argmin over exact rationals, Lemma 10)
  dsft.filtered_samples    pinned (closed form within Theorem 4 bound; impulse-response
                           support = the brute-force windows)
  dsft.alias_dft           pinned (brute-force DFT, aliasing identity)
  dsft.window_representative pinned (brute-force scan of q + B, both edges)
  dsft.identify            pinned (brute-force CRT + window + passband)
  dsft.vote                pinned (hand-built vote sets at v_min - 1 / v_min votes)
  dsft.estimate            pinned (hand-built measurements with a closed-form median;
                           non-identifying grids in the majority; line-9 budget cut)
  dsft.merge               pinned (brute-force sort, zero drop)
  dsft.dsft (end to end)   pinned (brute-force DFT on tiny N; Theorem 5 bound;
                           passband-edge and B-extreme tones)
  dsft.clw_decode / identify_clw (CLW-style inner SFT, reading R14)
                           pinned (exhaustive decoding of exact shifted measurements on
                           tiny N, shifted-grid closed form, brute-force DFT end to end)
  scripts/mutation_check.py applies 24 plausible mistakes to the oracle; every one
  fails at least one `-m "not gpu"` test.
  inner-SFT design constants (c_b, T, v_min, pool rule, residue rule):
                           parity unpinned -- the paper prints no values for
                           them; only invariants pin them.
"""

from .params import OracleParams, Plan, derive_plan  # noqa: F401
from .dsft import dsft  # noqa: F401
