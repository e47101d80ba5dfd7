"""C-ABI checks that need no GPU: the library loads, exports every symbol the
header declares, and its host-side plan derivation agrees exactly with the
oracle's independent derivation (integers bit-exact, reals bitwise)."""

import pytest

import paper_1706_02740_b200 as d
from oracle.params import ConfigError, OracleParams, derive_plan


def test_library_exports_every_header_symbol():
    L = d.lib()
    names = d.header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), n
    assert b"sm_100a" in L.dsft_version()


CASES = [(4096, 8, 0), (4096, 8, 5), (64, 4, 1), (97, 4, 2), (255, 6, 3), (2**16, 50, 4), (2**22, 50, 3),
         (2**26, 1000, 1), (2**26, 500, 9), (2**26, 1500, 4), (6000011, 100, 7), (2**24, 256, 2)]


@pytest.mark.parametrize("N,s,seed", CASES)
@pytest.mark.parametrize("preset", ["dmsft6", "dmsft4", "thm4"])
def test_plan_matches_oracle(N, s, seed, preset):
    info = d.dsft_plan_derive_info(N, s, d.make_params(preset=preset, seed=seed))
    p = derive_plan(N, s, OracleParams(preset=preset, seed=seed))
    assert list(info.primes[:info.T]) == p.primes
    assert [list(info.residues[t][:info.n_residues[t]]) for t in range(info.T)] == p.residues
    assert (info.w, info.J, info.q1, info.kappa, info.band_budget) == (p.w, p.J, p.q[0], p.kappa, p.band_budget)
    assert info.c1 == p.c1 and info.alpha == p.alpha and info.beta == p.beta
    assert info.sum_primes == sum(p.primes)
    assert info.grid_points == sum(P * r for P, rs in zip(p.primes, p.residues) for r in rs)
    assert info.nodes == sum(P * (1 + sum(r - 1 for r in rs)) for P, rs in zip(p.primes, p.residues))


def test_literal_alpha_and_kappa_override_match():
    for kw in (dict(alpha_rule="literal"), dict(kappa=5), dict(tau=0.1), dict(bucket_factor=5.0, n_bucket_primes=7, vote_min=4),
               dict(n_bucket_primes=0, vote_min=0, pool_rule="smooth"), dict(n_bucket_primes=0, vote_min=5, pool_rule="smooth"), dict(vote_min=0)):
        info = d.dsft_plan_derive_info(2**20, 100, d.make_params(**kw))
        p = derive_plan(2**20, 100, OracleParams(**kw))
        assert (info.w, info.J, info.kappa, list(info.primes[:info.T])) == (p.w, p.J, p.kappa, p.primes)
        assert (info.T, info.vote_min) == (len(p.primes), p.vote_min)
    # the deterministic variant at the headline s: T = 37 bucket primes (<= DSFT_MAX_T)
    info = d.dsft_plan_derive_info(2**26, 1000, d.make_params(n_bucket_primes=0, vote_min=0, pool_rule="smooth"))
    p = derive_plan(2**26, 1000, OracleParams(n_bucket_primes=0, vote_min=0, pool_rule="smooth"))
    assert info.T == len(p.primes) == 37 and list(info.primes[:info.T]) == p.primes and info.vote_min == 19


@pytest.mark.parametrize("N,s,kw", [(30, 4, {}), (4096, 1, {}), (4096, 4097, {}), (4096, 8, dict(tau=0.5)),
                                    (4096, 8, dict(preset="thm4", r=0.5)), (4096, 3, {}),
                                    (4096, 8, dict(vote_min=6))])
def test_config_errors_match_oracle(N, s, kw):
    with pytest.raises(ConfigError):
        derive_plan(N, s, OracleParams(**kw))
    with pytest.raises(d.DsftError) as ei:
        d.dsft_plan_derive_info(N, s, d.make_params(**kw))
    assert ei.value.status == d.DSFT_ERR_CONFIG


@pytest.mark.parametrize("rule", ["full", "smooth"])
def test_pool_rule_matches_oracle(rule):
    """Reading R6 on both sides: the same pool and the same seeded draw (DSFT_POOL_FULL:
    every prime in range -- general primes run the zero-padded Rader K2)."""
    for N, s, seed in ((2**26, 1000, 0), (2**22, 50, 3), (4096, 8, 1), (2**21, 4000, 2)):
        info = d.dsft_plan_derive_info(N, s, d.make_params(seed=seed, pool_rule=rule))
        p = derive_plan(N, s, OracleParams(seed=seed, pool_rule=rule))
        assert list(info.primes[:info.T]) == p.primes
    assert d.default_pool_rule() == OracleParams().pool_rule == "smooth"


@pytest.mark.parametrize("N,s,kw", [(4096, 8, {}), (2**26, 1000, {}), (2**22, 50, {"kappa": 12}), (97, 4, {}),
                                    (2**31 + 11, 8, {})])
def test_clw_plan_matches_oracle(N, s, kw):
    """Reading R14 on both sides: the same primes and, per prime, one grid with the
    shifts 0, 1, 2, ..., 2^(L-1) (n_shifts = 1 + L)."""
    info = d.dsft_plan_derive_info(N, s, d.make_params(inner="clw", seed=3, **kw))
    p = derive_plan(N, s, OracleParams(inner="clw", seed=3, **kw))
    assert info.inner == 1 and list(info.primes[:info.T]) == p.primes
    assert [info.n_shifts[t] for t in range(info.T)] == [len(sh) for sh in p.shifts]
    assert all(info.n_residues[t] == 1 and info.residues[t][0] == 1 for t in range(info.T))
    assert info.grid_points == sum(p.primes)
    assert info.nodes == sum(P * len(sh) for P, sh in zip(p.primes, p.shifts))


def test_shard_bands_partition():
    for J in (1, 7, 15, 43):
        for world in (1, 2, 3, 4, 8):
            got = sorted(j for r in range(world) for j in d.dsft_shard_bands(J, r, world))
            assert got == list(range(J))
            assert all(j % world == r for r in range(world) for j in d.dsft_shard_bands(J, r, world))


def test_k2_specialisation_compiles_with_nvrtc(tmp_path, monkeypatch):
    """Plan-time K2 specialisation (jit.cpp): the embedded device sources compile
    with NVRTC for sm_100a (no GPU needed), for 1- to 4-pass radix tuples."""
    monkeypatch.setenv("DSFT_JIT_CACHE", str(tmp_path))  # force real compiles
    import paper_1706_02740_b200 as d
    for nt, minb, rad in ((256, 2, [10, 9, 9, 5]), (512, 1, [12, 10, 9, 7]), (256, 2, [13]), (256, 2, [16, 3])):
        st, log = d.dsft_debug_jit_compile(nt, minb, rad)
        assert st == 0, log
    # cluster mode (thread-block cluster of C CTAs per row, DSMEM stages): C = 2 and 4
    for rad in ([2, 12, 9, 5, 7], [4, 13, 7, 7, 7]):
        st, log = d.dsft_debug_jit_compile(256, 2, rad, cluster=True)
        assert st == 0, log
    # Good-Thomas dimensions: twiddle-free stages (M = 8 * 3 * 13^2, 9 * 11 * 50)
    for rad, twf in (([8, 3, 13, 13], 0b011), ([9, 11, 10, 5], 0b011)):
        st, log = d.dsft_debug_jit_compile(256, 2, rad, twf=twf)
        assert st == 0, log
    # zero-padded Rader rows of a general bucket prime (bit 31 of twf): M = 8192 >= 2 (P - 1) - 1
    st, log = d.dsft_debug_jit_compile(512, 1, [16, 16, 8, 4], twf=0x80000000)
    assert st == 0, log
    assert len(list(tmp_path.glob("k2_*.cubin"))) == 9
