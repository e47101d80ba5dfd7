#!/usr/bin/env python3
"""Developer tool (GPU): A/B timing of dsft_execute for several parameter sets on the
same vector (L2 flushed between reps outside the events, CUDA-graph replay as in the
bench), interleaved over rounds so clock drift hits every variant alike.

    python scripts/ab.py N s "name:key=value,key=value" "name2:..." [--reps 30 --rounds 3]
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


def parse_kw(spec: str):
    name, _, rest = spec.partition(":")
    kw = {}
    for item in filter(None, rest.split(",")):
        k, v = item.split("=")
        try:
            kw[k] = int(v)
        except ValueError:
            try:
                kw[k] = float(v)
            except ValueError:
                kw[k] = v
    return name, kw


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("N", type=int)
    ap.add_argument("s", type=int)
    ap.add_argument("variants", nargs="+")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--rounds", type=int, default=3)
    a = ap.parse_args()
    pl = planted(a.N, a.s, cfg=2, trial=0)
    f = torch.from_numpy(pl.f).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    fr = torch.empty(a.s, dtype=torch.int64, device="cuda")
    co = torch.empty(a.s, dtype=torch.complex128, device="cuda")
    plans = []
    for spec in a.variants:
        name, kw = parse_kw(spec)
        env = {k: str(v) for k, v in kw.items() if k.startswith("DSFT_")}  # plan-time experiment knobs
        kw = {k: v for k, v in kw.items() if not k.startswith("DSFT_")}
        os.environ.update(env)
        p = d.Plan(a.N, a.s, d.make_params(**kw))
        for k in env:
            del os.environ[k]
        for _ in range(3):
            p.dsft_execute(f, fr, co)
        torch.cuda.synchronize()
        ok = sorted(x for x in fr.cpu().tolist() if x != d.SENTINEL) == pl.freqs.tolist()
        plans.append((name, p, ok, []))
    st = torch.cuda.current_stream()
    for _ in range(a.rounds):
        for name, p, ok, times in plans:
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.reps)]
            for e0, e1 in ev:
                flush.zero_()
                e0.record(st)
                p.dsft_execute(f, fr, co, st)
                e1.record(st)
            torch.cuda.synchronize()
            times += [e0.elapsed_time(e1) for e0, e1 in ev]
    for name, p, ok, times in plans:
        ms = statistics.median(times)
        print(f"{name:16s} median {ms:.4f} ms  {1e3 / ms:8.1f} transforms/s  mean {statistics.mean(times):.4f}  "
              f"support {ok}  launches {p.launches_per_execute()}", flush=True)


if __name__ == "__main__":
    main()
