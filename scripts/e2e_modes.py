#!/usr/bin/env python3
"""dsft_execute_host in its two modes (zero copy / copy) on one B200, per (N, s):
the measurement behind the zero-copy threshold in plan.cpp host_alias.

    python scripts/e2e_modes.py [--cases 67108864:1000,67108864:4000] [--reps 5]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1706_02740_b200 as d  # noqa: E402
from dsft_synth import planted  # noqa: E402


def e2e_ms(plan, fh, frh, coh, reps):
    st = torch.cuda.current_stream()
    plan.dsft_execute_host(fh, frh, coh, st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        plan.dsft_execute_host(fh, frh, coh, st)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="67108864:1000,67108864:2000,67108864:4000,4194304:50,6000011:100,16777216:256")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    out = []
    for c in a.cases.split(","):
        N, s = (int(x) for x in c.split(":"))
        plan = d.Plan(N, s)
        fh = torch.from_numpy(planted(N, s, cfg=2, trial=0).f).pin_memory()
        frh = torch.empty(s, dtype=torch.int64).pin_memory()
        coh = torch.empty(s, dtype=torch.complex128).pin_memory()
        row = {"N": N, "s": s, "window_bytes": plan.info.nodes * (2 * plan.info.kappa + 1) * 16,
               "f_bytes": N * 16, "default_zero_copy": plan.dsft_plan_host_zero_copy(fh)[0]}
        for mode, env in (("zero_copy", "1"), ("copy", "0")):
            os.environ["DSFT_HOST_ZERO_COPY"] = env
            ms = e2e_ms(plan, fh, frh, coh, a.reps)
            row[mode] = {"ms": ms, "transforms_per_s": 1e3 / ms}
        del os.environ["DSFT_HOST_ZERO_COPY"]
        row["window_frac"] = row["window_bytes"] / row["f_bytes"]
        print(json.dumps(row), flush=True)
        out.append(row)
        del fh
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "e2e_modes.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
