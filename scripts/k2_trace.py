#!/usr/bin/env python3
"""Developer tool: per-stage K2 timings from an instrumented build (-DDSFT_K2_TRACE).

    python scripts/k2_trace.py build        # here (CPU): builds paper_1706_02740_b200/libdsft_trace.so
    python scripts/k2_trace.py run          # on the GPU box: one c2 transform, prints stage cycles
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
TRACE_LIB = os.path.join(ROOT, "paper_1706_02740_b200", "libdsft_trace.so")

if sys.argv[1] == "build":
    from paper_1706_02740_b200 import build as b
    b.build(force=True, defines=("DSFT_K2_TRACE",), out=TRACE_LIB)
    sys.exit(0)

os.environ["DSFT_LIB"] = TRACE_LIB
import numpy as np
import torch
import paper_1706_02740_b200 as d
from dsft_synth import planted

N, s = 2 ** 26, 1000
pl = planted(N, s, cfg=2, trial=0)
f = torch.from_numpy(pl.f).cuda()
plan = d.Plan(N, s, d.make_params(seed=0))
fr = torch.empty(s, dtype=torch.int64, device="cuda")
co = torch.empty(s, dtype=torch.complex128, device="cuda")
for _ in range(3):
    plan.dsft_execute(f, fr, co, torch.cuda.current_stream())
torch.cuda.synchronize()
L = C.CDLL(TRACE_LIB)
buf = np.zeros((8, 1024, 16), dtype=np.int64)
assert L.dsft_debug_k2_trace(buf.ctypes.data_as(C.c_void_p), C.c_size_t(buf.size)) == 0
info = plan.info
for t in range(info.T):
    P = info.primes[t]
    nb = info.J * info.n_shifts[t]
    tr = buf[t, :min(nb, 1024)]
    nst = int(np.max(np.sum(tr[:, :15] != 0, axis=1)))
    d_ = np.diff(tr[:, :nst], axis=1)
    start = tr[:, 15]
    print(f"t={t} P={P} rows={nb} stage-boundaries={nst}: mean cycles per phase",
          np.round(d_.mean(axis=0)).astype(int).tolist(), "total", int(d_.sum(axis=1).mean()),
          "| start spread us", round((start.max() - start.min()) / 1e3, 1))


t5 = np.zeros((64, 8), dtype=np.uint64)
if hasattr(L, "dsft_debug_k5_trace") and L.dsft_debug_k5_trace(t5.ctypes.data_as(C.c_void_p)) == 0:
    t5 = t5.astype(np.int64)[:info.J]
    t0 = t5[:, 0].min()
    for j in range(info.J):
        r = t5[j]
        print(f"K5b band {j}: start {(r[0]-t0)/1e3:7.2f} select {(r[1]-r[0])/1e3:7.2f} us "
              f"(stage {(r[2]-r[0])/1e3:6.2f}, rank1 {(r[3]-r[2])/1e3:6.2f}, rank2 {(r[4]-r[3])/1e3:6.2f}) "
              f"ticket {(r[5]-r[1])/1e3:6.2f}")
