#!/usr/bin/env python3
"""Developer tool (GPU): per-launch kernel times of one configuration in SERIAL mode
(one stream, no graph, per-launch CUDA events), for several parameter/env variants, so
kernel changes can be A/B-ed without the pipeline's overlap.  The k-th launch of a
class in one execute is reported separately (for K1/K2/K3: the k-th bucket prime in
processing order).

    python scripts/kern_times.py N s "name:key=value,DSFT_ENV=value" ... [--reps 10]
"""

from __future__ import annotations

import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1706_02740_b200 as d  # noqa: E402
from dsft_synth import planted  # noqa: E402
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from ab import parse_kw  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("N", type=int)
    ap.add_argument("s", type=int)
    ap.add_argument("variants", nargs="+")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    pl = planted(a.N, a.s, cfg=2, trial=0)
    f = torch.from_numpy(pl.f).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    fr = torch.empty(a.s, dtype=torch.int64, device="cuda")
    co = torch.empty(a.s, dtype=torch.complex128, device="cuda")
    st = torch.cuda.current_stream()
    ref = None
    for spec in a.variants:
        name, kw = parse_kw(spec)
        env = {k: str(v) for k, v in kw.items() if k.startswith("DSFT_")}
        kw = {k: v for k, v in kw.items() if not k.startswith("DSFT_")}
        kw["flags"] = kw.get("flags", 0) | 16 | 32  # SERIAL | NO_GRAPH
        os.environ.update(env)
        p = d.Plan(a.N, a.s, d.make_params(**kw))
        for k in env:
            del os.environ[k]
        for _ in range(3):
            p.dsft_execute(f, fr, co, st)
        torch.cuda.synchronize()
        ok = sorted(x for x in fr.cpu().tolist() if x != d.SENTINEL) == pl.freqs.tolist()
        out = (fr.cpu().clone(), co.cpu().clone())
        if ref is None:
            ref = out
        same = bool(torch.equal(out[0], ref[0]) and torch.equal(out[1], ref[1]))
        per: dict = {}
        for _ in range(a.reps):
            flush.zero_()
            p.dsft_plan_set_timing(True)
            p.dsft_execute(f, fr, co, st)
            torch.cuda.synchronize()
            tl = p.dsft_plan_collect_timeline()
            p.dsft_plan_set_timing(False)
            seen: dict = {}
            for cls, t0, t1 in sorted(tl, key=lambda r: r[1]):
                k = seen.get(cls, 0)
                seen[cls] = k + 1
                per.setdefault((cls, k), []).append((t1 - t0) * 1e3)
        tot = {}
        for (cls, k), v in per.items():
            tot[cls] = tot.get(cls, 0.0) + statistics.median(v)
        line = "  ".join(f"{c[:2]}={tot[c]:.1f}" for c in sorted(tot))
        print(f"{name:12s} support {ok} bitwise-as-first {same}  primes {p.primes()}  [{line}] us  sum {sum(tot.values()):.1f}", flush=True)
        for (cls, k) in sorted(per):
            if cls.startswith("k2"):
                print(f"    {cls} #{k}: {statistics.median(per[(cls, k)]):.2f} us")


if __name__ == "__main__":
    main()
