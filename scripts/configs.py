#!/usr/bin/env python3
"""All five BASELINE.json configs on the GPU (one B200): throughput, accuracy against
the planted spectrum, and parity with the oracle on samples.  Writes one JSON file
(default gpurun_out/configs.json) and prints a summary; profiles/r1_configs.md
records a run.

    python scripts/configs.py [--only c0,c1,c2,c3,c4] [--out PATH] [--quick]

Inputs follow DESIGN.md §5 (dsft_synth).  Config 4's 256 x 2^24 batch (64 GiB) is
synthesised on the device: frequencies, phases and noise are drawn with the same
seeded numpy generator as dsft_synth.planted (vector = batch index), the inverse
DFT runs on the GPU (torch.fft, plumbing), so the oracle samples are fed the exact
device bytes copied back.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_02740_b200 as d  # noqa: E402
from dsft_synth import planted, rng_for  # noqa: E402
from oracle import OracleParams, dsft  # noqa: E402
from oracle.dsft import SENTINEL  # noqa: E402

DEV = torch.device("cuda:0")


def run(plan, f_dev):
    fr, co = plan(f_dev)
    torch.cuda.synchronize()
    return fr.cpu().numpy(), co.cpu().numpy()


def parity(gpu, ref):
    fr, co = gpu
    ok = fr != SENTINEL
    fr, co = fr[ok], co[ok]
    same = sorted(fr.tolist()) == sorted(ref.freqs.tolist())
    rel = None
    if same and len(fr):
        a = dict(zip(fr.tolist(), co))
        keys = ref.freqs.tolist()
        va = np.array([a[k] for k in keys])
        rel = float(np.linalg.norm(va - ref.coeffs) / np.linalg.norm(ref.coeffs))
    return {"freq_set_equal": same, "coeff_rel_l2": rel, "pass": bool(same and (rel is None or rel <= 1e-10))}


def accuracy(gpu, freqs_true, fhat_true, s):
    """support-exact flag and (1/s) sum over the union support of |fhat - v| (missing counts |fhat|)."""
    fr, co = gpu
    ok = fr != SENTINEL
    rec = dict(zip(fr[ok].tolist(), co[ok]))
    tru = dict(zip(freqs_true.tolist(), fhat_true))
    keys = set(rec) | set(tru)
    l1 = sum(abs(tru.get(k, 0.0) - rec.get(k, 0.0)) for k in keys) / s
    return {"support_exact": set(rec) == set(tru), "avg_l1": float(l1), "found": len(set(rec) & set(tru))}


def timed(fn, reps):
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def c0(quick):
    N, s = 4096, 8
    trials = 10 if quick else 100
    plan = d.Plan(N, s, d.make_params(seed=0))
    par, exact = 0, 0
    for t in range(trials):
        pl = planted(N, s, cfg=0, trial=t)
        g = run(plan, torch.from_numpy(pl.f).to(DEV))
        par += parity(g, dsft(pl.f, s, OracleParams(seed=0)))["pass"]
        exact += accuracy(g, pl.freqs, pl.fhat, s)["support_exact"]
    f1 = torch.from_numpy(planted(N, s, cfg=0, trial=0).f).to(DEV)
    fr = torch.empty(s, dtype=torch.int64, device=DEV)
    co = torch.empty(s, dtype=torch.complex128, device=DEV)
    lat = timed(lambda: plan.dsft_execute(f1, fr, co), 200)
    B = 4096
    fb = torch.stack([torch.from_numpy(planted(N, s, cfg=0, trial=t % trials, vector=t // trials).f)
                      for t in range(B)]).to(DEV)
    frb = torch.empty(B * s, dtype=torch.int64, device=DEV)
    cob = torch.empty(B * s, dtype=torch.complex128, device=DEV)
    bt = timed(lambda: plan.dsft_execute_batched(fb.view(-1), B, N, frb, cob), 5)
    return {"N": N, "s": s, "trials": trials, "oracle_parity_pass": par, "support_exact": exact,
            "latency_ms": lat, "batched_vectors": B, "batched_transforms_per_s": B / (bt / 1e3)}


def c1(quick):
    N, s = 2 ** 22, 50
    trials = 3 if quick else 10
    plan = d.Plan(N, s, d.make_params(seed=0))
    par, exact = 0, 0
    for t in range(trials):
        pl = planted(N, s, cfg=1, trial=t)
        g = run(plan, torch.from_numpy(pl.f).to(DEV))
        par += parity(g, dsft(pl.f, s, OracleParams(seed=0)))["pass"]
        exact += accuracy(g, pl.freqs, pl.fhat, s)["support_exact"]
    f1 = torch.from_numpy(planted(N, s, cfg=1, trial=0).f).to(DEV)
    fr = torch.empty(s, dtype=torch.int64, device=DEV)
    co = torch.empty(s, dtype=torch.complex128, device=DEV)
    ms = timed(lambda: plan.dsft_execute(f1, fr, co), 50)
    return {"N": N, "s": s, "trials": trials, "oracle_parity_pass": par, "support_exact": exact,
            "ms_per_transform": ms, "transforms_per_s": 1e3 / ms}


def c2(quick):
    N = 2 ** 26
    out = []
    for s in (50, 100, 200, 500, 1000, 2000, 4000):
        pl = planted(N, s, cfg=2, trial=0)
        f = torch.from_numpy(pl.f).to(DEV)
        plan = d.Plan(N, s, d.make_params(seed=0))
        g = run(plan, f)
        fr = torch.empty(s, dtype=torch.int64, device=DEV)
        co = torch.empty(s, dtype=torch.complex128, device=DEV)
        ms = timed(lambda: plan.dsft_execute(f, fr, co), 5 if quick else 20)
        row = {"s": s, "primes": plan.primes(), "ms_per_transform": ms, "transforms_per_s": 1e3 / ms,
               **accuracy(g, pl.freqs, pl.fhat, s)}
        if not quick or s in (50, 1000):
            t0 = time.perf_counter()
            row["oracle"] = parity(g, dsft(pl.f, s, OracleParams(seed=0)))
            row["oracle_s"] = time.perf_counter() - t0
        out.append(row)
        print("  c2", {k: v for k, v in row.items() if k != "primes"}, flush=True)
        del f
    return {"N": N, "sweep": out}


def c3(quick):
    N, s = 6000011, 100
    trials = 2 if quick else 5
    plan = d.Plan(N, s, d.make_params(seed=0))
    out = []
    for snr in (0.0, 10.0, 20.0, 40.0, 60.0, 80.0):
        l1, exact, par = [], 0, 0
        for t in range(trials):
            pl = planted(N, s, cfg=3, trial=t, snr_db=snr)
            g = run(plan, torch.from_numpy(pl.f).to(DEV))
            a = accuracy(g, pl.freqs, pl.fhat, s)
            l1.append(a["avg_l1"])
            exact += a["support_exact"]
            if t == 0:
                par = parity(g, dsft(pl.f, s, OracleParams(seed=0)))["pass"]
        out.append({"snr_db": snr, "avg_l1_mean": float(np.mean(l1)), "avg_l1_max": float(np.max(l1)),
                    "support_exact": exact, "trials": trials, "oracle_parity_trial0": par})
        print("  c3", out[-1], flush=True)
    f1 = torch.from_numpy(planted(N, s, cfg=3, trial=0, snr_db=20.0).f).to(DEV)
    fr = torch.empty(s, dtype=torch.int64, device=DEV)
    co = torch.empty(s, dtype=torch.complex128, device=DEV)
    ms = timed(lambda: plan.dsft_execute(f1, fr, co), 50)
    return {"N": N, "s": s, "snr_sweep": out, "ms_per_transform": ms}


def det(quick):
    """SURVEY 8(f) next row 1, the deterministic variant (reading R13): every pool prime
    (n_bucket_primes = 0), majority vote; throughput and exact support at c1 / c2 sizes,
    oracle parity where the oracle finishes in seconds (c1)."""
    out = []
    prm = dict(n_bucket_primes=0, vote_min=0, pool_rule="smooth")
    for N, s, cfg in ((2 ** 22, 50, 1), (2 ** 26, 200, 2), (2 ** 26, 1000, 2)):
        pl = planted(N, s, cfg=cfg, trial=0)
        f = torch.from_numpy(pl.f).to(DEV)
        plan = d.Plan(N, s, d.make_params(**prm))
        g = run(plan, f)
        fr = torch.empty(s, dtype=torch.int64, device=DEV)
        co = torch.empty(s, dtype=torch.complex128, device=DEV)
        ms = timed(lambda: plan.dsft_execute(f, fr, co), 5 if quick else 20)
        row = {"N": N, "s": s, "T": plan.info.T, "vote_min": plan.info.vote_min, "ms_per_transform": ms,
               "transforms_per_s": 1e3 / ms, **accuracy(g, pl.freqs, pl.fhat, s)}
        if N == 2 ** 22:
            row["oracle"] = parity(g, dsft(pl.f, s, OracleParams(**prm)))
        out.append(row)
        print("  det", row, flush=True)
        del f
    return {"rows": out}


def thm4(quick):
    """the THM4 preset (kappa = O(log N) windows, larger J) at
    the headline sizes: throughput, exact support, error against the planted spectrum;
    oracle parity at N = 2^16 (the oracle needs minutes at N = 2^26 here)."""
    out = []
    for N, s in ((2 ** 16, 50), (2 ** 22, 50), (2 ** 26, 1000)):
        pl = planted(N, s, cfg=2, trial=0)
        f = torch.from_numpy(pl.f).to(DEV)
        plan = d.Plan(N, s, d.make_params(preset="thm4"))
        g = run(plan, f)
        fr = torch.empty(s, dtype=torch.int64, device=DEV)
        co = torch.empty(s, dtype=torch.complex128, device=DEV)
        ms = timed(lambda: plan.dsft_execute(f, fr, co), 5 if quick else 20)
        row = {"N": N, "s": s, "kappa": plan.info.kappa, "J": plan.info.J, "nodes": plan.info.nodes,
               "ms_per_transform": ms, "transforms_per_s": 1e3 / ms, **accuracy(g, pl.freqs, pl.fhat, s)}
        if N == 2 ** 16:
            row["oracle"] = parity(g, dsft(pl.f, s, OracleParams(preset="thm4")))
        out.append(row)
        print("  thm4", row, flush=True)
        del f
    return {"rows": out}


def nsweep(quick):
    """SURVEY 8(f) next row 3 (PAPER.md:663-673 protocol): runtime vs N at s = 50,
    N = 2^16 .. 2^30 (2^30 complex128 = 16 GiB, synthesised on the device)."""
    out = []
    s = 50
    for e in range(16, 31, 2):
        N = 2 ** e
        plan = d.Plan(N, s, d.make_params(seed=0))
        f = torch.empty(N, dtype=torch.complex128, device=DEV)
        try:
            freqs, fhat = synth_device(N, s, 5, 0, 0, None, f)
        except RuntimeError as e:  # device synthesis out of memory: record and stop
            out.append({"N": N, "s": s, "error": str(e)[:200]})
            break
        g = run(plan, f)
        fr = torch.empty(s, dtype=torch.int64, device=DEV)
        co = torch.empty(s, dtype=torch.complex128, device=DEV)
        ms = timed(lambda: plan.dsft_execute(f, fr, co), 5 if quick else 20)
        row = {"N": N, "s": s, "ms_per_transform": ms, "transforms_per_s": 1e3 / ms,
               "window_MB": plan.info.nodes * (2 * plan.info.kappa + 1) * 16 / 1e6,
               **accuracy(g, freqs, fhat, s)}
        out.append(row)
        print("  nsweep", row, flush=True)
        del f
        torch.cuda.empty_cache()
    return {"rows": out}


def noise22(quick):
    """noise robustness at N = 2^22, s = 50 (PAPER.md:685-702
    protocol), avg-l1 against the planted spectrum per SNR."""
    N, s = 2 ** 22, 50
    trials = 3 if quick else 10
    plan = d.Plan(N, s, d.make_params(seed=0))
    out = []
    for snr in (0.0, 10.0, 20.0, 40.0, 60.0, 80.0):
        l1, exact = [], 0
        for t in range(trials):
            pl = planted(N, s, cfg=6, trial=t, snr_db=snr)
            a = accuracy(run(plan, torch.from_numpy(pl.f).to(DEV)), pl.freqs, pl.fhat, s)
            l1.append(a["avg_l1"])
            exact += a["support_exact"]
        out.append({"snr_db": snr, "avg_l1_mean": float(np.mean(l1)), "avg_l1_max": float(np.max(l1)),
                    "support_exact": exact, "trials": trials})
        print("  noise22", out[-1], flush=True)
    return {"N": N, "s": s, "snr_sweep": out}


def dense(quick):
    """Context only (the FFTW analogue): a dense complex128 cuFFT of
    the whole vector (torch.fft.fft, a library call) at N = 2^22 and 2^26."""
    out = []
    for e in (22, 26):
        N = 2 ** e
        x = torch.randn(N, dtype=torch.complex128, device=DEV)
        ms = timed(lambda: torch.fft.fft(x), 5 if quick else 20)
        out.append({"N": N, "ms": ms, "transforms_per_s": 1e3 / ms})
        print("  dense", out[-1], flush=True)
        del x
    return {"rows": out}


def synth_device(N, s, cfg, trial, vector, snr_db, out_row):
    """dsft_synth.planted's draws (same generator, same order), inverse DFT on the device."""
    rng = rng_for(cfg, trial, vector)
    lo = -((N + 1) // 2) + 1
    idx = rng.choice(N, s, replace=False).astype(np.int64)
    theta = 2.0 * math.pi * rng.random(s)
    c = np.exp(1j * theta)
    freqs = idx + lo
    chat = torch.zeros(N, dtype=torch.complex128, device=DEV)
    chat[torch.from_numpy(freqs % N).to(DEV)] = torch.from_numpy(c).to(DEV)
    f = N * torch.fft.ifft(chat)
    del chat
    if snr_db is None:  # noiseless
        out_row.copy_(f)
    else:
        n = torch.complex(torch.from_numpy(rng.standard_normal(N)).to(DEV),
                          torch.from_numpy(rng.standard_normal(N)).to(DEV))
        n *= torch.linalg.vector_norm(f) / (torch.linalg.vector_norm(n) * 10.0 ** (snr_db / 20.0))
        out_row.copy_(f + n)
    order = np.argsort(freqs)
    sign = np.where(freqs % 2 == 0, 1.0, -1.0)
    return freqs[order], (sign * c)[order]


def c4(quick):
    N, s, B, snr = 2 ** 24, 256, (32 if quick else 256), 20.0
    plan = d.Plan(N, s, d.make_params(seed=0))
    f = torch.empty(B, N, dtype=torch.complex128, device=DEV)
    truth = []
    t0 = time.perf_counter()
    for v in range(B):
        truth.append(synth_device(N, s, 4, v, v, snr, f[v]))
    synth_s = time.perf_counter() - t0
    fr = torch.empty(B * s, dtype=torch.int64, device=DEV)
    co = torch.empty(B * s, dtype=torch.complex128, device=DEV)
    ms = timed(lambda: plan.dsft_execute_batched(f.view(-1), B, N, fr, co), 2 if quick else 3)
    frn, con = fr.cpu().numpy().reshape(B, s), co.cpu().numpy().reshape(B, s)
    accs = [accuracy((frn[v], con[v]), truth[v][0], truth[v][1], s) for v in range(B)]
    par = {}
    for v in (0, 1, B - 1):
        fh = f[v].cpu().numpy()
        par[v] = parity((frn[v], con[v]), dsft(fh, s, OracleParams(seed=0)))["pass"]
    return {"N": N, "s": s, "batch": B, "snr_db": snr, "batch_ms": ms, "transforms_per_s": B / (ms / 1e3),
            "support_exact": int(sum(a["support_exact"] for a in accs)),
            "found_frac_min": float(min(a["found"] for a in accs) / s),
            "avg_l1_mean": float(np.mean([a["avg_l1"] for a in accs])),
            "oracle_parity": par, "synth_s": synth_s}


def variants(quick):
    """The inner-SFT and pool options on BASELINE config 2 (N = 2^26, s = 1000) and the
    noise sweep of the CLW-style inner SFT at N = 2^22, s = 50 (kappa = 12, PAPER.md:653;
    the paper reports CLW-DSFT losing exact support below 40 dB)."""
    out = []
    N, s = 2 ** 26, 1000
    pl = planted(N, s, cfg=2, trial=0)
    f = torch.from_numpy(pl.f).to(DEV)
    for name, kw in (("gfft/smooth", {}), ("gfft/full", {"pool_rule": "full"}), ("clw/smooth", {"inner": "clw"}),
                     ("clw/smooth/kappa12", {"inner": "clw", "kappa": 12}), ("thm4", {"preset": "thm4"})):
        plan = d.Plan(N, s, d.make_params(seed=0, **kw))
        g = run(plan, f)
        fr = torch.empty(s, dtype=torch.int64, device=DEV)
        co = torch.empty(s, dtype=torch.complex128, device=DEV)
        ms = timed(lambda: plan.dsft_execute(f, fr, co), 5 if quick else 20)
        row = {"variant": name, "N": N, "s": s, "ms_per_transform": ms, "transforms_per_s": 1e3 / ms,
               **accuracy(g, pl.freqs, pl.fhat, s)}
        out.append(row)
        print("  variants", row, flush=True)
        plan.close()
    del f
    N, s = 2 ** 22, 50
    trials = 3 if quick else 10
    plan = d.Plan(N, s, d.make_params(seed=0, inner="clw", kappa=12))
    sweep = []
    for snr in (0.0, 10.0, 20.0, 40.0, 60.0, 80.0):
        l1, exact = [], 0
        for t in range(trials):
            pl = planted(N, s, cfg=6, trial=t, snr_db=snr)
            a = accuracy(run(plan, torch.from_numpy(pl.f).to(DEV)), pl.freqs, pl.fhat, s)
            l1.append(a["avg_l1"])
            exact += a["support_exact"]
        sweep.append({"snr_db": snr, "avg_l1_mean": float(np.mean(l1)), "support_exact": exact, "trials": trials})
        print("  clw noise22", sweep[-1], flush=True)
    return {"rows": out, "clw_noise22": sweep}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c0,c1,c2,c3,c4,det,thm4,nsweep,noise22,dense,variants")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "configs.json"))
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    res = {"gpu": torch.cuda.get_device_name(0), "quick": a.quick}
    for name in a.only.split(","):
        t0 = time.perf_counter()
        res[name] = globals()[name](a.quick)
        res[name]["wall_s"] = time.perf_counter() - t0
        print(name, json.dumps(res[name])[:1500], flush=True)
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        json.dump(res, open(a.out, "w"), indent=1)
    return 0


if __name__ == "__main__":
    sys.exit(main())
