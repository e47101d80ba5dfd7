#!/usr/bin/env python3
"""Developer tool (GPU): run one configuration a few times (for ncu launch lists).
    python scripts/run_one.py N s [reps] [key=value ...]   (make_params keywords)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1706_02740_b200 as d  # noqa: E402
from dsft_synth import planted  # noqa: E402

N, s = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
kw = {}
for a in sys.argv[4:]:
    k, v = a.split("=")
    try:
        kw[k] = int(v)
    except ValueError:
        try:
            kw[k] = float(v)
        except ValueError:
            kw[k] = v
pl = planted(N, s, cfg=2, trial=0)
f = torch.from_numpy(pl.f).cuda()
plan = d.Plan(N, s, d.make_params(**kw))
fr = torch.empty(s, dtype=torch.int64, device="cuda")
co = torch.empty(s, dtype=torch.complex128, device="cuda")
for _ in range(reps):
    plan.dsft_execute(f, fr, co)
torch.cuda.synchronize()
ok = sorted(x for x in fr.cpu().tolist() if x != d.SENTINEL) == pl.freqs.tolist()
print("support_exact", ok, "launches", plan.launches_per_execute(), "primes", plan.primes())
