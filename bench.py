#!/usr/bin/env python3
"""Benchmark of the DSFT hot path on B200 (BASELINE.json metric:
"sparse DFTs/sec at N=2^26, s=1000; filter-gather GB/s vs HBM peak").

One step = one complete transform (K1..K6, every §8(a) row) of one synthetic
N = 2^26 complex128 vector with s = 1000 planted unit tones (BASELINE config 2,
DMSFT-6 preset), input already resident in HBM.  Timing: CUDA events on the
launching stream around each step, L2 flushed (256 MiB write) between steps
outside the events, W warm-up steps, max over ranks.  The timed loop runs with
the library's per-launch timing OFF; a second, separately reported pass with
per-launch CUDA events gives the kernel breakdown and the rooflines.

Multi-GPU (`--gpus N`, N > 1; self-spawns N ranks with torch.distributed.run when
WORLD_SIZE is unset): every rank transforms its own vector and the results of all
ranks are exchanged with the library's NCCL allgather inside the timed region
(dsft_execute_batched_sharded: weak scaling).  The band-sharded
single-vector path (dsft_execute_sharded: one vector, its J bands split over the
ranks, one allgather of band blocks, strong scaling) is timed beside it and
reported under "band_sharded".  `--mode` selects either path at any N (N = 1
exercises the same code with a one-rank communicator).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--mode ...]
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sparse DFTs/sec at N=2^26, s=1000; filter-gather GB/s vs HBM peak"
UNIT = "transforms/s"
FP64_PEAK_TFLOPS = 36.62  # measured DFMA peak, profiles/r1_fp64_peak.md


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="auto", choices=["auto", "single", "batched-sharded", "band-sharded"],
                    help="auto: single at N=1, batched-sharded (plus a band-sharded line) at N>1")
    ap.add_argument("--N", type=int, default=2**26)
    ap.add_argument("--s", type=int, default=1000)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--pool", default=None, choices=[None, "full", "smooth"], help="bucket-prime pool (default: library's)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def spawn_ranks(a) -> int:
    """--gpus N > 1 without a torch.distributed launcher: re-run this script as N
    ranks (one process per GPU) with torch.distributed.run on 127.0.0.1."""
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def source_hash() -> str:
    """Hash of the library sources: a stored ncu traffic figure applies only to them."""
    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_1706_02740_b200", "csrc")
    for name in sorted(os.listdir(csrc)):
        if name.endswith((".cu", ".cuh", ".cpp", ".h")):
            h.update(name.encode())
            h.update(open(os.path.join(csrc, name), "rb").read())
    return h.hexdigest()[:16]


def stored_traffic(kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from the
    ncu --set full capture committed under profiles/ (scripts/ncu_traffic.py), if it
    was taken on the current sources; else (None, reason)."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(path))
    except Exception:
        return None, "no profiles/traffic.json"
    if d.get("source_hash") != source_hash():
        return None, f"profiles/traffic.json was captured on other sources ({d.get('source_hash')})"
    k = d.get("kernels", {}).get(kernel)
    if not k:
        return None, f"{kernel} not in profiles/traffic.json"
    return k["dram_bytes_per_launch"], d.get("capture", "profiles/traffic.json")


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons while the timed region runs."""

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        self.max_mhz = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.nv = None
        self._stop = threading.Event()
        self._t = None

    NAMES = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
             0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting",
             0x100: "display_clock_setting", 0x1: "gpu_idle"}

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.NAMES.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()
        if not self.samples:
            return None
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def window_entries(info, N: int) -> list[int]:
    """Distinct f entries read by K1 for each bucket prime t (union of the
    2 kappa + 1 windows of all S_t * P_t nodes) -- the algorithmic read bytes / 16."""
    import numpy as np
    out = []
    kap = info.kappa
    for t in range(info.T):
        P = info.primes[t]
        rs = list(info.residues[t][:info.n_residues[t]])
        shifts = [(1, 0)] + [(r, n2) for r in rs for n2 in range(1, r)]
        n1 = np.arange(P, dtype=np.int64)
        cols = []
        for r, n2 in shifts:
            L = P * r
            k = (r * n1 + P * n2) % L
            jp = (2 * k * N + L) // (2 * L)
            cols.append(jp)
        jp = np.concatenate(cols)
        idx = (jp[:, None] + np.arange(-kap, kap + 1)[None, :]) % N
        out.append(int(np.unique(idx).size))
    return out


def workload_config(N, s, units, mode, world, pool, J, T, primes, nodes):
    """The `config` object of the JSON line.  Both arms print the same one (the
    reference arm derives J, T, primes and nodes from the oracle's own plan; the ABI
    test pins the two derivations to each other), so the driver's same-config check
    compares like with like; the entries that describe the GPU arm's timing say so."""
    return {"workload": f"BASELINE config 2: N=2^{int(math.log2(N))} complex128, s={s}, noiseless, "
                        "dmsft6 (kappa=6, tau=1/3, c_b=4, T=5, v_min=3)",
            "global_batch": units, "mode": mode,
            "parallelism": {"single": "one vector per step, one process (GPU arm: 1 GPU)",
                            "batched-sharded": f"{world} vectors, 1 per GPU, results allgathered (NCCL) every step",
                            "band-sharded": f"1 vector, J bands over {world} GPUs, band blocks allgathered (NCCL)"}[mode],
            "pool": pool,
            "l2": "GPU arm: flushed (256 MiB write) between steps, outside the timed events; f is 1 GiB",
            "J": int(J), "T": int(T), "primes": [int(x) for x in primes], "nodes": int(nodes)}



# ------------------------------------------------------------------ reference
def run_reference(a):
    """--impl reference: the oracle (numpy, CPU) as it stands, on this host."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np
    from dsft_synth import planted
    from oracle import OracleParams, derive_plan
    from oracle.dsft import process_band

    N, s = a.N, a.s
    pl = planted(N, s, cfg=2, trial=0)
    pool = a.pool or "smooth"
    plan = derive_plan(N, s, OracleParams(seed=a.seed, pool_rule=pool))
    if plan.inner == "clw":
        ref_nodes = sum(P * len(sh) for P, sh in zip(plan.primes, plan.shifts))
    else:
        ref_nodes = sum(P * (1 + sum(r - 1 for r in rs)) for P, rs in zip(plan.primes, plan.residues))
    times = []
    for k in range(a.warmup + a.steps):
        j = k % plan.J
        t0 = time.perf_counter()
        process_band(pl.f, plan, j)
        dt = time.perf_counter() - t0
        if k >= a.warmup:
            times.append(dt)
    band_s = statistics.mean(times)
    value = 1.0 / (plan.J * band_s)  # one transform = J bands (+ a negligible merge)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": band_s * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(N, s, 1, "single", 1, pool, plan.J, plan.T, plan.primes, ref_nodes),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "host_cores": os.cpu_count(), "kind": "oracle",
                         "sample": f"each step = one of the J={plan.J} bands of Algorithm 1 (oracle.process_band); "
                                   "value = 1/(J * mean band time)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------- ours
def busy_union(iv):
    """Length of the union of [t0, t1) intervals."""
    tot, cur0, cur1 = 0.0, None, None
    for t0, t1 in sorted(iv):
        if cur1 is None or t0 > cur1:
            if cur1 is not None:
                tot += cur1 - cur0
            cur0, cur1 = t0, t1
        else:
            cur1 = max(cur1, t1)
    if cur1 is not None:
        tot += cur1 - cur0
    return tot


def run_ours(a):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1706_02740_b200 as d
    from dsft_synth import planted

    world, rank, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    N, s = a.N, a.s
    mode = a.mode if a.mode != "auto" else ("single" if world == 1 else "batched-sharded")

    pl = planted(N, s, cfg=2, trial=rank)
    f = torch.from_numpy(pl.f).to(dev)
    prm = dict(seed=a.seed, pool_rule=a.pool)
    plan = d.Plan(N, s, d.make_params(**prm))
    info = plan.info
    pool = a.pool or d.default_pool_rule()
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    comm = None
    if mode != "single":
        uid = bytearray(d.Comm.unique_id() if rank == 0 else bytes(128))
        if world > 1:
            t = torch.tensor(list(uid), dtype=torch.uint8, device=dev)
            dist.broadcast(t, 0)
            uid = bytes(t.cpu().tolist())
        comm = d.Comm(rank, world, bytes(uid))

    # outputs: one vector per rank; batched-sharded gathers every rank's result
    nout = world * s if mode == "batched-sharded" else s
    freqs = torch.empty(nout, dtype=torch.int64, device=dev)
    coeffs = torch.empty(nout, dtype=torch.complex128, device=dev)

    def step(p=plan, fv=f, md=mode):
        if md == "single":
            p.dsft_execute(fv, freqs, coeffs, stream)
        elif md == "batched-sharded":
            p.dsft_execute_batched_sharded(comm, fv, 1, N, freqs, coeffs, stream)
        else:
            p.dsft_execute_sharded(comm, fv, freqs[:s], coeffs[:s], stream)

    def timed_loop(steps, md=mode, p=plan):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(steps):
            flush.zero_()  # L2 flush outside the timed events
            evs[k][0].record(stream)
            step(p, f, md)
            evs[k][1].record(stream)
        if comm is not None:
            comm.wait(stream, timeout_ms=300_000)  # bounded: a lost peer aborts instead of hanging
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms_ = statistics.mean(e0.elapsed_time(e1) for e0, e1 in evs)
        if world > 1:
            tt = torch.tensor([ms_], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms_ = float(tt.item())
        return ms_

    for _ in range(a.warmup):
        step()
    if comm is not None:
        comm.wait(stream, timeout_ms=300_000)
    torch.cuda.synchronize()
    fr = freqs[rank * s:(rank + 1) * s] if mode == "batched-sharded" else freqs[:s]
    fr = fr.cpu().numpy()
    support_exact = sorted(fr[fr != d.SENTINEL].tolist()) == pl.freqs.tolist()

    # ---- the timed region (per-launch library timing off)
    clk = ClockSampler(local)
    clk.start()
    t_wall = time.perf_counter()
    ms = timed_loop(a.steps)
    t_wall = time.perf_counter() - t_wall
    clocks = clk.stop()
    units = world if mode != "band-sharded" else 1  # transforms completed per step by the whole job
    value = units / (ms / 1e3)

    # ---- band-sharded single vector beside the weak-scaling line (N > 1)
    band = None
    if world > 1 and a.mode == "auto":
        bms = timed_loop(max(5, a.steps // 4), md="band-sharded")
        band = {"value": 1.0 / (bms / 1e3), "unit": UNIT, "ms_per_step": bms, "scaling": "strong",
                "path": "dsft_execute_sharded: one vector, bands j = rank mod N, one NCCL allgather of band blocks"}

    # ---- the other bucket-prime pool (reading R6) on the same vector, same protocol
    other_pool = None
    if world == 1 and mode == "single" and a.pool is None:
        op_ = "full" if pool == "smooth" else "smooth"
        plan2 = d.Plan(N, s, d.make_params(seed=a.seed, pool_rule=op_))
        for _ in range(a.warmup):
            step(plan2, f, "single")
        torch.cuda.synchronize()
        fr2 = freqs[:s].cpu().numpy()
        oms = timed_loop(max(10, a.steps // 2), md="single", p=plan2)
        other_pool = {"pool": op_, "value": 1.0 / (oms / 1e3), "unit": UNIT, "ms_per_step": oms,
                      "primes": list(plan2.info.primes[:plan2.info.T]),
                      "support_exact": sorted(fr2[fr2 != d.SENTINEL].tolist()) == pl.freqs.tolist(),
                      "note": "full = every prime in [4s, 8s) (general primes: zero-padded Rader, FFT length "
                              ">= 2(P-1)-1); smooth = primes with 13-smooth P-1 (DESIGN.md R6)"}
        plan2.close()

    # ---- the CLW-style inner SFT (reading R14) on the same vector, same protocol
    clw = None
    if world == 1 and mode == "single":
        plan3 = d.Plan(N, s, d.make_params(seed=a.seed, pool_rule=a.pool, inner="clw"))
        for _ in range(a.warmup):
            step(plan3, f, "single")
        torch.cuda.synchronize()
        fr3 = freqs[:s].cpu().numpy()
        cms = timed_loop(max(10, a.steps // 2), md="single", p=plan3)
        clw = {"inner": "clw", "value": 1.0 / (cms / 1e3), "unit": UNIT, "ms_per_step": cms,
               "support_exact": sorted(fr3[fr3 != d.SENTINEL].tolist()) == pl.freqs.tolist(),
               "shift_rows_per_prime": [plan3.info.n_shifts[t] for t in range(plan3.info.T)],
               "note": "DMSFT-6 window with the phase-encoding inner SFT (CLW-DSFT family, PAPER.md:653)"}
        plan3.close()

    # ---- kernel breakdown: a second pass with per-launch CUDA events on each launch's stream
    plan.dsft_plan_set_timing(True)
    kpass = max(10, min(a.steps, 50))
    kms = timed_loop(kpass)
    tl = plan.dsft_plan_collect_timeline(plan.launches_per_execute() * kpass + 64)
    plan.dsft_plan_set_timing(False)
    kt = {k: (0.0, 0) for k in plan.KERNEL_CLASSES}
    ivs = {k: [] for k in plan.KERNEL_CLASSES}
    for name, t0, t1 in tl:
        kt[name] = (kt[name][0] + (t1 - t0), kt[name][1] + 1)
        ivs[name].append((t0, t1))
    busy = {k: busy_union(iv) for k, iv in ivs.items()}

    # ---- end to end through the public API with HOST buffers (dsft_execute_host)
    e2e = None
    if not a.no_e2e:
        fh = torch.from_numpy(pl.f).pin_memory()
        frh = torch.empty(s, dtype=torch.int64).pin_memory()
        coh = torch.empty(s, dtype=torch.complex128).pin_memory()

        def e2e_ms(p):
            p.dsft_execute_host(fh, frh, coh, stream)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(a.e2e_steps):
                p.dsft_execute_host(fh, frh, coh, stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ems = e0.elapsed_time(e1) / a.e2e_steps
            if world > 1:
                tt = torch.tensor([ems], device=dev, dtype=torch.float64)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                ems = float(tt.item())
            return ems

        # default mode: K1 gathers its windows straight from the pinned host vector
        # (zero copy, include/dsft.h) when they cover at most half of f
        zero_copy, h2d = plan.dsft_plan_host_zero_copy(fh)
        ems = e2e_ms(plan)
        e2e = {"value": world / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": s * 24, "ms_per_step": ems,
               "path": "dsft_execute_host (C ABI, pinned host buffers, every rank its own vector)",
               "mode": "zero_copy (K1 reads the sampled windows of pinned host f)" if zero_copy
               else "copy (1 H2D of f per step)"}
        if zero_copy:  # context: the same call forced to copy all of f first
            pc = d.Plan(N, s, d.make_params(flags=d.FLAG_HOST_COPY, **prm))
            cms = e2e_ms(pc)
            e2e["copy_mode"] = {"value": world / (cms / 1e3), "h2d_bytes_per_step": N * 16, "ms_per_step": cms}
            pc.close()

    # ---- roofline of the dominant kernel: K2 (the aliasing DFTs), FP64-bound.  Algorithmic
    # flops = SURVEY §8(d)'s 5 L log2 L per residue grid L = P_t r_{t,i} per band (the grid
    # DFT that K2's length-P DFTs and K3's length-r fold implement together, Good-Thomas);
    # peak = measured DFMA peak (profiles/r1_fp64_peak.md: 36.6 TFLOP/s)
    peaks = measured_peaks()
    nb_local = info.J if mode != "band-sharded" else len(d.dsft_shard_bands(info.J, rank, world))
    k2_flops = sum(nb_local * 5.0 * L * math.log2(L)
                   for t in range(info.T)
                   for L in (info.primes[t] * r for r in info.residues[t][:info.n_residues[t]]))
    k2_ms, k2_n = kt["k2_prime_dft"]
    k2_avg_ms = k2_ms / max(k2_n, 1)
    k2_achieved = (k2_flops / info.T / 1e12) / (k2_avg_ms / 1e3)
    k2_busy_ms = busy["k2_prime_dft"] / kpass  # union of the K2 launch intervals per step
    k2_achieved_busy = (k2_flops / 1e12) / (k2_busy_ms / 1e3) if k2_busy_ms > 0 else None
    k2_traffic, k2_tsrc = stored_traffic("k2")
    # ---- roofline of the filter-gather kernel K1 (the metric's named ratio)
    peak_gbs = peaks["hbm_gbs"] if peaks else 6650.0
    wins = window_entries(info, N)
    k1_ms, k1_n = kt["k1_gather_mix"]
    # algorithmic bytes of K1 = the distinct f entries its windows read;
    # the filtered samples it writes to Z (L2-resident, consumed by K2) are reported apart
    per_vec_bytes = sum(16 * wins[t] for t in range(info.T))
    z_bytes = sum(16 * nb_local * info.n_shifts[t] * info.primes[t] for t in range(info.T))
    k1_launches = max(k1_n / kpass, 1.0)
    k1_launch_bytes = per_vec_bytes / k1_launches
    k1_avg_ms = k1_ms / max(k1_n, 1)
    achieved = (k1_launch_bytes / 1e9) / (k1_avg_ms / 1e3)
    k1_traffic, k1_tsrc = stored_traffic("k1")
    # K1 is also FP64 work: SURVEY 8(d) counts (2 kappa + 1)(8 J + 3) flops per node (band
    # mix + Gaussian taps); at J = 15 its intensity sits near the FP64 ridge, so the
    # binding roof of K1 is the larger of the two times (SURVEY 8(d) "Targets")
    k1_flops = (2 * info.kappa + 1) * (8 * nb_local + 3) * info.nodes
    k1_launch_flops = k1_flops / k1_launches
    k1_tflops = (k1_launch_flops / 1e12) / (k1_avg_ms / 1e3)
    k1_roof_ms = max(k1_launch_bytes / (peak_gbs * 1e9), k1_launch_flops / (FP64_PEAK_TFLOPS * 1e12)) * 1e3
    step_flops = k1_flops + k2_flops  # the two FP64 bodies of the path (K3-K6: O(T K) per candidate)
    total_kernel_ms = sum(v[0] for v in kt.values())
    kernels = {k: {"ms_per_step": v[0] / kpass, "busy_ms_per_step": busy[k] / kpass,
                   "launches_per_step": v[1] / kpass,
                   "share": (v[0] / total_kernel_ms if total_kernel_ms else None)} for k, v in kt.items()}

    # ---- CPU baseline: the oracle on this host (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        from oracle import OracleParams, derive_plan
        from oracle.dsft import process_band
        op = derive_plan(N, s, OracleParams(seed=a.seed, pool_rule=pool))
        nb = op.J
        t0 = time.perf_counter()
        for j in range(nb):
            process_band(pl.f, op, j)
        dt = time.perf_counter() - t0
        cpu = {"value": 1.0 / (op.J * dt / nb), "unit": UNIT, "cores": 1, "host_cores": os.cpu_count(),
               "kind": "oracle",
               "sample": f"all J={op.J} bands of one transform of the same vector (oracle.process_band, numpy, "
                         f"1 thread of {os.cpu_count()} host cores; the merge is negligible), {dt:.1f} s of CPU work"}

    launches = plan.launches_per_execute() * a.steps
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong" if mode == "band-sharded" else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (dsft_synth: s unit-magnitude random-phase tones on B, seeded)",
        "config": workload_config(N, s, units, mode, world, pool, info.J, info.T, info.primes[:info.T], info.nodes),
        "gpu_launches": launches,
        "roofline": {"kernel": "k2_prime_dft", "bound": "alu", "achieved": k2_achieved, "peak": FP64_PEAK_TFLOPS,
                     "unit": "TFLOP/s", "frac": k2_achieved / FP64_PEAK_TFLOPS, "traffic": k2_traffic,
                     "traffic_source": k2_tsrc,
                     "peak_source": "measured FP64 DFMA peak (profiles/r1_fp64_peak.md); FP64, no tensor path",
                     "algorithmic_flops_per_launch": k2_flops / info.T, "avg_launch_ms": k2_avg_ms,
                     "busy": {"achieved": k2_achieved_busy, "frac": (k2_achieved_busy / FP64_PEAK_TFLOPS
                                                                     if k2_achieved_busy else None),
                              "ms_per_step": k2_busy_ms,
                              "note": "algorithmic flops per step / union of the K2 launch intervals per step "
                                      "(consecutive K2 launches overlap on two streams, so avg_launch_ms "
                                      "counts shared time twice)"},
                     "algorithmic": "SURVEY 8(d): 5 L log2 L per residue grid L = P_t r_ti, x J bands (K2 + K3 fold; "
                                    "Rader executes 2 FFTs of P-1 per row)",
                     "timing_pass": f"{kpass} steps with per-launch CUDA events ({kms:.4f} ms/step)"},
        "roofline_gather": {"kernel": "k1_gather_mix", "bound": "hbm", "achieved": achieved, "peak": peak_gbs,
                            "unit": "GB/s", "frac": achieved / peak_gbs, "traffic": k1_traffic,
                            "frac_of_nominal_8tbs": achieved / 8000.0,
                            "traffic_source": k1_tsrc,
                            "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if peaks else "fallback 6.65 TB/s",
                            "algorithmic_bytes_per_launch": k1_launch_bytes, "avg_launch_ms": k1_avg_ms,
                            "launches_per_step": k1_launches,
                            "algorithmic": "16 B x distinct f entries under the 2kappa+1 windows of the launch's nodes",
                            "note": "launch duration measured inside the pipeline (K1 shares the SMs with K2/K3)",
                            "z_samples_bytes_per_launch": z_bytes / k1_launches,
                            "fp64": {"achieved": k1_tflops, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                                     "frac": k1_tflops / FP64_PEAK_TFLOPS,
                                     "algorithmic_flops_per_launch": k1_launch_flops,
                                     "algorithmic": "SURVEY 8(d): (2 kappa + 1)(8 J + 3) per node"},
                            "binding_roof": ("fp64" if k1_launch_flops / FP64_PEAK_TFLOPS / 1e3 >
                                             k1_launch_bytes / peak_gbs else "hbm"),
                            "frac_of_binding_roof": k1_roof_ms / k1_avg_ms},
        "step_roofline": {"algorithmic_flops": step_flops, "floor_ms": step_flops / (FP64_PEAK_TFLOPS * 1e12) * 1e3,
                          "frac": step_flops / (FP64_PEAK_TFLOPS * 1e12) * 1e3 / ms,
                          "note": "K1 band mix + K2 aliasing DFTs (SURVEY 8(d) algorithmic counts) at the FP64 "
                                  "peak, against ms_per_step"},
        "kernels": kernels,
        "k2_specialized": plan.dsft_plan_k2_specialized()[0],
        "filtered_samples_per_s": units * info.J * info.nodes / (ms / 1e3),
        "support_exact": bool(support_exact),
        "band_sharded": band,
        "other_pool": other_pool,
        "inner_clw": clw,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "wall_s_timed_loop": t_wall,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(a)
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
