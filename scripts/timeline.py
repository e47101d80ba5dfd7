#!/usr/bin/env python3
"""Developer tool (GPU): per-launch timeline of one transform at BASELINE config 2
(CUDA events on each launch's own stream, relative to the first)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1706_02740_b200 as d
from dsft_synth import planted

N, s = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 26, int(sys.argv[2]) if len(sys.argv) > 2 else 1000
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
pl = planted(N, s, cfg=2, trial=0)
f = torch.from_numpy(pl.f).cuda()
plan = d.Plan(N, s, d.make_params(seed=0, flags=flags))
fr = torch.empty(s, dtype=torch.int64, device="cuda")
co = torch.empty(s, dtype=torch.complex128, device="cuda")
st = torch.cuda.current_stream()
for _ in range(3):
    plan.dsft_execute(f, fr, co, st)
torch.cuda.synchronize()
plan.dsft_plan_set_timing(True)
plan.dsft_execute(f, fr, co, st)
torch.cuda.synchronize()
tl = plan.dsft_plan_collect_timeline()
plan.dsft_plan_set_timing(False)
for name, a, b in sorted(tl, key=lambda r: r[1]):
    bar = " " * int(a * 200) + "#" * max(1, int((b - a) * 200))
    print(f"{name:18s} {a * 1e3:8.1f} {b * 1e3:8.1f} {(b - a) * 1e3:7.1f} us |{bar}")
print("span us", round(max(r[2] for r in tl) * 1e3, 1))
