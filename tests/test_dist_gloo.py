"""Multi-process (world size 2, gloo, CPU) test of the band-sharded PROTOCOL of
dsft_execute_sharded: the band partition comes from the library's
host function dsft_shard_bands; each rank computes its bands with the oracle
standing in for K1-K5 (there is no GPU here), packs fixed-capacity per-band blocks
padded with the sentinel, all_gathers them, and merges.  The merged result must be
identical to the single-process transform on every rank.

The library's own sharded code (dsft_execute_sharded_local -> rank-major gather
layout -> dsft_merge_sharded, the halves of dsft_execute_sharded) is driven on the
GPU by tests/test_gpu_parity.py::test_sharded_virtual_ranks_equal_execute (R
virtual ranks on one GPU, bitwise against dsft_execute)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1706_02740_b200 as d
from dsft_synth import planted
from oracle.dsft import dsft, merge, process_band
from oracle.params import OracleParams, derive_plan

SENT = np.iinfo(np.int64).min


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, N, s, seed, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = derive_plan(N, s, OracleParams(seed=seed))
    pl = planted(N, s, cfg=40, trial=seed)
    bands = d.dsft_shard_bands(plan.J, rank, world)
    nbmax = -(-plan.J // world)
    budget = plan.band_budget
    w = np.full((nbmax, budget), SENT, dtype=np.int64)
    c = np.zeros((nbmax, budget), dtype=np.complex128)
    n = np.zeros(nbmax, dtype=np.int64)
    for jl, j in enumerate(bands):
        br = process_band(pl.f, plan, j)
        k = len(br.omegas)
        w[jl, :k] = br.omegas
        c[jl, :k] = br.coeffs
        n[jl] = k
    tw = [torch.empty(nbmax * budget, dtype=torch.int64) for _ in range(world)]
    tc = [torch.empty(2 * nbmax * budget, dtype=torch.float64) for _ in range(world)]
    tn = [torch.empty(nbmax, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(tw, torch.from_numpy(w.reshape(-1)))
    dist.all_gather(tc, torch.from_numpy(c.reshape(-1).view(np.float64)))
    dist.all_gather(tn, torch.from_numpy(n))
    oms, cs = [], []
    for r in range(world):
        wr = tw[r].numpy().reshape(nbmax, budget)
        cr = tc[r].numpy().view(np.complex128).reshape(nbmax, budget)
        nr = tn[r].numpy()
        for b in range(nbmax):
            oms += wr[b, :nr[b]].tolist()
            cs += cr[b, :nr[b]].tolist()
    freqs, coeffs, _ = merge(plan, oms, cs)
    out[rank] = (freqs, coeffs)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("N,s,seed", [(4096, 8, 0), (6007, 16, 1)])
def test_band_sharded_world2_equals_single(N, s, seed):
    ref = dsft(planted(N, s, cfg=40, trial=seed).f, s, OracleParams(seed=seed))
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, N, s, seed, out), nprocs=2, join=True)
    for rank in range(2):
        f, c = out[rank]
        assert np.array_equal(f, ref.freqs) and np.array_equal(c, ref.coeffs)


def test_shard_partition_covers_bands_once():
    for J in (15, 43):
        for world in (2, 3, 8):
            seen = [j for r in range(world) for j in d.dsft_shard_bands(J, r, world)]
            assert sorted(seen) == list(range(J))
