#!/usr/bin/env python3
"""Single-transform latency of dsft_execute per configuration, CUDA-graph replay on
and off (DSFT_FLAG_NO_GRAPH), beside one dense torch.fft of the same length
(context only; the FFTW analogue of PAPER.md:663-673).  L2 flushed between reps
outside the events, f resident in HBM.

    python scripts/latency.py [--reps 50] [--out gpurun_out/latency.json]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1706_02740_b200 as d  # noqa: E402
from dsft_synth import planted  # noqa: E402

CONFIGS = [("c0", 4096, 8, {}), ("c1", 2**22, 50, {}), ("c2_s50", 2**26, 50, {}), ("c3", 6000011, 100, {}),
           ("c2_s1000", 2**26, 1000, {}), ("c2_s1000_thm4", 2**26, 1000, {"preset": "thm4"}),
           ("c1_thm4", 2**22, 50, {"preset": "thm4"})]


def time_ms(fn, reps, flush):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    for e0, e1 in evs:
        flush.zero_()
        e0.record(st)
        fn()
        e1.record(st)
    torch.cuda.synchronize()
    return statistics.median(e0.elapsed_time(e1) for e0, e1 in evs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--only", default=None)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "latency.json"))
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    rows = []
    for name, N, s, kw in CONFIGS:
        if a.only and name not in a.only.split(","):
            continue
        pl = planted(N, s, cfg=50, trial=0)
        f = torch.from_numpy(pl.f).to(dev)
        fr = torch.empty(s, dtype=torch.int64, device=dev)
        co = torch.empty(s, dtype=torch.complex128, device=dev)
        row = {"config": name, "N": N, "s": s, **kw}
        for tag, flags in (("graph", 0), ("no_graph", d.FLAG_NO_GRAPH)):
            plan = d.Plan(N, s, d.make_params(flags=flags, **kw))
            ms = time_ms(lambda: plan.dsft_execute(f, fr, co), a.reps, flush)
            ok = sorted(x for x in fr.cpu().tolist() if x != d.SENTINEL) == pl.freqs.tolist()
            row[tag] = {"ms": ms, "support_exact": ok, "launches": plan.launches_per_execute()}
            plan.close()
        out = torch.empty_like(f)
        row["dense_fft_ms"] = time_ms(lambda: torch.fft.fft(f, out=out), a.reps, flush)
        rows.append(row)
        print(json.dumps(row), flush=True)
        del f, out
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(rows, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
