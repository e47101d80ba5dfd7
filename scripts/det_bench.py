#!/usr/bin/env python3
"""Deterministic-variant throughput at BASELINE config 2 (N = 2^26, s = 1000, every
pool prime, majority vote) under the current environment (e.g. DSFT_K1GROUPS)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1706_02740_b200 as d  # noqa: E402
from dsft_synth import planted  # noqa: E402

N, s = 2 ** 26, int(sys.argv[1]) if len(sys.argv) > 1 else 1000
pl = planted(N, s, cfg=2, trial=0)
f = torch.from_numpy(pl.f).cuda()
plan = d.Plan(N, s, d.make_params(n_bucket_primes=0, vote_min=0, pool_rule="smooth"))
fr = torch.empty(s, dtype=torch.int64, device="cuda")
co = torch.empty(s, dtype=torch.complex128, device="cuda")
st = torch.cuda.current_stream()
for _ in range(3):
    plan.dsft_execute(f, fr, co, st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(10):
    plan.dsft_execute(f, fr, co, st)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
ok = sorted(x for x in fr.cpu().tolist() if x != d.SENTINEL) == pl.freqs.tolist()
print(f"det T={plan.info.T} K1GROUPS={os.environ.get('DSFT_K1GROUPS', '-')}: {ms:.3f} ms, {1e3 / ms:.1f} transforms/s, support exact {ok}")
