#!/usr/bin/env python3
"""Mutation check of the oracle's pins ("What's weak" 1).

Copies the repository to a scratch directory, applies one plausible mistake at a
time to oracle/*.py, runs the CPU suite (`-m "not gpu"`) there and reports which
mutants survive.  A surviving mutant means a part of the oracle no pin checks.

    python scripts/mutation_check.py [-k NAME]
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, file, old, new) -- an `old` that occurs n > 1 times (the same line in vote() and in
# the CLW-style vote) gives n mutants, one per occurrence ("name #k")
MUTANTS = [
    ("vote >= 1", "oracle/dsft.py", "len(voters(plan, ids, om)) >= plan.vote_min)",
     "len(voters(plan, ids, om)) >= 1)"),
    ("vote >= v_min + 1", "oracle/dsft.py", "len(voters(plan, ids, om)) >= plan.vote_min)",
     "len(voters(plan, ids, om)) >= plan.vote_min + 1)"),
    ("majority floor(T/2)", "oracle/params.py", "vote_min = T // 2 + 1 if", "vote_min = max(1, T // 2) if"),
    ("no band-budget cut", "oracle/dsft.py", "keep = order[:plan.band_budget]", "keep = order"),
    ("j' = floor(kN/L)", "oracle/dsft.py", "return (2 * k * N + L) // (2 * L)", "return (k * N) // L"),
    ("j' = ceil(kN/L)", "oracle/dsft.py", "return (2 * k * N + L) // (2 * L)", "return (k * N + L - 1) // L"),
    ("q+B right edge open", "oracle/dsft.py", "return np.where(om <= hi, om, SENTINEL)",
     "return np.where(om < hi, om, SENTINEL)"),
    ("q+B left edge shifted", "oracle/dsft.py", "lo = q - (N + 1) // 2 + 1          #",
     "lo = q - (N + 1) // 2          #"),
    ("estimate over all T", "oracle/dsft.py", "for t in voters(plan, ids, om):\n            for i, L",
     "for t in range(plan.T):\n            for i, L"),
    ("passband upper closed", "oracle/dsft.py", "(om < q + plan.w)", "(om <= q + plan.w)"),
    ("passband lower open", "oracle/dsft.py", "(om >= q - plan.w)", "(om > q - plan.w)"),
    ("B upper open", "oracle/dsft.py", "(om <= plan.B_hi)", "(om < plan.B_hi)"),
    ("no (-1)^omega", "oracle/dsft.py", "sgn = -1.0 if om % 2 else 1.0", "sgn = 1.0"),
    ("median -> mean", "oracle/dsft.py", "zs.append(complex(np.median(v.real), np.median(v.imag)))",
     "zs.append(complex(np.mean(v.real), np.mean(v.imag)))"),
    ("unbias ghat_{omega+q}", "oracle/dsft.py", "float(ghat(om - q, plan.c1))", "float(ghat(om + q, plan.c1))"),
    ("modulation sign", "oracle/dsft.py", "phase = np.exp(2j * math.pi * rho / NL)",
     "phase = np.exp(-2j * math.pi * rho / NL)"),
    ("merge keeps zeros", "oracle/dsft.py", "if not (c.real == 0.0 and c.imag == 0.0)]", "]"),
    ("window kappa - 1", "oracle/dsft.py", "for u in range(-plan.kappa, plan.kappa + 1):",
     "for u in range(-plan.kappa + 1, plan.kappa):"),
    # CLW-style inner SFT (reading R14)
    ("clw: phase not offset by lo", "oracle/dsft.py", "phi = (theta - ((m * lo) % N) / N) % 1.0",
     "phi = theta % 1.0"),
    ("clw: floor in refinement", "oracle/dsft.py", "            k = math.floor(x + 0.5)",
     "            k = math.floor(x)"),
    ("clw: no circular lift", "oracle/dsft.py", "for lift in (-N, 0, N):", "for lift in (0,):"),
    ("clw: shift sign", "oracle/dsft.py", "num = k * N + m * L - j * L", "num = k * N - m * L - j * L"),
    ("clw: estimate on shifted grid", "oracle/dsft.py", "Y = [[Y[t][0]] for t in range(plan.T)]",
     "Y = [[Y[t][1]] for t in range(plan.T)]"),
    ("clw: one scale fewer", "oracle/params.py", "while (1 << (L - 1)) * P < N:", "while (1 << L) * P < N:"),
]


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("-k", default=None, help="only mutants whose name contains this")
    a = ap.parse_args()
    survivors = []
    with tempfile.TemporaryDirectory() as tmp:
        dst = os.path.join(tmp, "repo")
        shutil.copytree(ROOT, dst, ignore=shutil.ignore_patterns(".git", "gpurun_out", "profiles", "*.so", "build*"))
        expanded = []
        for name, rel, old, new in MUTANTS:
            orig = open(os.path.join(ROOT, rel)).read()
            n = orig.count(old)
            assert n >= 1, (name, n)
            pos = -1
            for k in range(n):
                pos = orig.index(old, pos + 1)
                mutated = orig[:pos] + new + orig[pos + len(old):]
                expanded.append((name if n == 1 else f"{name} #{k + 1}", rel, orig, mutated))
        for name, rel, orig, mutated in expanded:
            if a.k and a.k not in name:
                continue
            path = os.path.join(dst, rel)
            open(path, "w").write(mutated)
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "not gpu", "tests",
                                "--ignore=tests/test_abi.py", "--ignore=tests/test_dist_gloo.py"],
                               cwd=dst, capture_output=True, text=True)
            killed = r.returncode != 0
            tail = [ln for ln in r.stdout.splitlines() if ln.startswith("FAILED")][:1]
            print(f"{'killed ' if killed else 'SURVIVED'}  {name:24s} {tail[0] if tail else ''}", flush=True)
            if not killed:
                survivors.append(name)
            open(path, "w").write(orig)
    print(f"{len(survivors)} surviving mutant(s): {survivors}")
    return 1 if survivors else 0


if __name__ == "__main__":
    sys.exit(main())
