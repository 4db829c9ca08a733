"""CPU parity of the C-ABI library (libtiletune.so) against the oracle: configuration space,
J_hw tables, G-BFS / N-A2C traversal under deterministic cost tables, ABI surface.  No GPU."""
import math
import os
import re

import numpy as np
import pytest

from oracle import costs, gbfs as ogbfs, hw, na2c as ona2c, space
from oracle.rng import SplitMix64
from oracle.space import Spec
from paper_1909_10616_b200 import tiletune as tt

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def lib_space(sp: Spec):
    # oracle Spec is (m, k, n); the ABI takes (M, N, K)
    return tt.make_space(sp.m, sp.n, sp.k, sp.dm, sp.dk, sp.dn, sp.family)


def test_abi_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "tiletune.h")).read()
    declared = set(re.findall(r"\b(tt_[a-z0-9_]+)\s*\(", hdr)) - {"tt_cost_fn", "tt_batch_eval_fn"}
    assert len(declared) >= 20
    for name in sorted(declared):
        assert hasattr(tt.lib, name), name
    assert set(tt.EXPORTS) == declared
    assert tt.lib.tt_version() == 6


@pytest.mark.parametrize("dims,d,fam", [((512, 512, 512), (4, 2, 4), 0), ((1024, 1024, 1024), (4, 2, 4), 0),
                                        ((2048, 2048, 2048), (4, 2, 4), 0), ((64, 64, 64), (4, 2, 4), 1),
                                        ((12, 18, 30), (2, 3, 2), 0), ((256, 128, 512), (4, 2, 4), 1),
                                        ((4096, 4096, 4096), (4, 2, 4), 3), ((2048, 2048, 2048), (4, 2, 4), 2),
                                        ((1024, 8192, 8192), (4, 2, 4), 3), ((16, 16, 16), (1, 1, 1), 0)])
def test_counts_match_oracle(dims, d, fam):
    sp = Spec(*dims, *d, family=fam)
    raw, feas = tt.count_configs(lib_space(sp), feasible=True)
    assert raw == space.count_configs(sp)
    if raw <= 600000:
        assert feas == sum(1 for s in space.enumerate_configs(sp) if space.legitimate(sp, s))


def test_overflow_reported():
    p47 = 614889782588491410          # primorial 47#: 15 distinct primes -> 4^15 per axis at d = 4
    sp = tt.make_space(p47, p47, p47, 4, 4, 4)
    with pytest.raises(tt.TileTuneError) as e:
        tt.count_configs(sp)
    assert e.value.status == tt.E_OVERFLOW


def test_enumeration_rank_legitimacy_neighbors_64():
    sp = Spec(64, 64, 64)
    ls = lib_space(sp)
    ora = list(space.enumerate_configs(sp))
    lib = tt.enumerate_configs(ls)
    assert lib == ora                                        # bit-exact order (reading O4)
    for r in range(0, len(ora), 211):
        assert tt.rank(ls, ora[r]) == r and tt.unrank(ls, r) == ora[r]
    for s in ora[::7]:
        assert tt.neighbors(ls, s) == space.neighbors(sp, s)
    assert tt.is_legitimate(ls, ((64, 1, 1, 1), (64, 1), (64, 1, 1, 1))) == (True, True)
    assert tt.is_legitimate(ls, ((32, 1, 1, 1), (64, 1), (64, 1, 1, 1)))[0] is False
    with pytest.raises(tt.TileTuneError) as e:
        tt.rank(ls, ((32, 1, 1, 1), (64, 1), (64, 1, 1, 1)))
    assert e.value.status == tt.E_ILLEGITIMATE


def test_step_matches_oracle():
    sp = Spec(1024, 1024, 1024)
    ls = lib_space(sp)
    s0 = space.initial_state(sp)
    for (a, i, j) in space.actions(sp):
        o = space.step(s0, (a, i, j))
        o = o if (o is not None and space.legitimate(sp, o)) else None
        assert tt.step(ls, s0, a, i, j) == o


@pytest.mark.parametrize("dims,fam", [((512, 512, 512), 1), ((4096, 4096, 4096), 3), ((2048, 2048, 2048), 2),
                                      ((512, 512, 512), 3)])
def test_feasible_sets_match_oracle(dims, fam):
    sp = Spec(*dims, family=fam)
    cfgs, ranks = tt.enumerate_feasible(lib_space(sp))
    ora = [(r, s) for r, s in enumerate(space.enumerate_configs(sp)) if hw.j_hw(sp, s)]
    assert ranks == [r for r, _ in ora]
    assert cfgs == [s for _, s in ora]


def test_feasible_neighbors_match_oracle():
    sp = Spec(4096, 4096, 4096, family=3)
    ls = lib_space(sp)
    for s in [s for s in space.enumerate_configs(sp) if hw.j_hw(sp, s)]:
        assert tt.neighbors(ls, s) == space.neighbors(sp, s)
    sp = Spec(512, 512, 512, family=1)
    ls = lib_space(sp)
    allst = list(space.enumerate_configs(sp))
    for s in allst[::97]:
        if space.legitimate(sp, s):
            assert tt.neighbors(ls, s) == space.neighbors(sp, s)


def _trace_key(rows):
    return [(r["eval_index"], r["state"], r["cost"], r["best"]) for r in rows]


def _oracle_key(res):
    return [(r.eval_index, r.state, r.cost, r.best) for r in res.trace]


@pytest.mark.parametrize("width", [1, 8])
def test_gbfs_trace_parity_tables(width):
    # reading O8: library trace == oracle trace byte-for-byte under T1 / T2, seeds 0-9
    sp = Spec(64, 64, 64)
    t1 = costs.table(sp, costs.t1_cost)
    t2 = costs.table(sp, lambda s: costs.t2_cost(sp, s))
    for tab in (t1, t2):
        for seed in range(10):
            o = ogbfs.gbfs(sp, ogbfs.table_source(sp, tab), budget=988, rho=5, seed=seed, width=width)
            lres = tt.gbfs_search(64, 64, 64, 988, tt.search_opts(seed=seed, width=width, rho=5), table=tab)
            assert _trace_key(lres.trace) == _oracle_key(o), (seed, width)
            assert lres.best == o.best_state and lres.best_cost == o.best_cost
            assert lres.evals == o.evals and lres.space_raw == 49392


def test_gbfs_callback_and_completeness():
    sp = Spec(16, 16, 16, 2, 2, 2)
    tg = ((1.0, 3.0), (2.0, 2.0), (3.0, 1.0))
    fn = lambda s: costs.t1_cost(s, targets=tg)
    res = tt.gbfs_search(16, 16, 16, 0, tt.search_opts(dm=2, dk=2, dn=2, rho=6, seed=4), cost=fn)
    assert res.evals == 125 and res.best_cost == ogbfs.brute_force(sp, fn)[0]
    o = ogbfs.gbfs(sp, ogbfs.fn_source(fn), rho=6, seed=4)
    assert _trace_key(res.trace) == _oracle_key(o)


def test_gbfs_non_square_parity():
    # (M, N, K) = (256, 64, 128): paper order (m, k, n) = (256, 128, 64)
    sp = Spec(256, 128, 64)
    tab = costs.table(sp, lambda s: costs.t2_cost(sp, s, seed_t=3))
    o = ogbfs.gbfs(sp, ogbfs.table_source(sp, tab), budget=500, rho=5, seed=11)
    lres = tt.gbfs_search(256, 64, 128, 500, tt.search_opts(seed=11), table=tab)
    assert _trace_key(lres.trace) == _oracle_key(o)


def test_gbfs_feasible_family_parity():
    # family tables restrict g(s): parity on the SIMT space of 512^3 with a T2 table
    sp = Spec(512, 512, 512, family=1)
    tab = costs.table(sp, lambda s: costs.t2_cost(sp, s))
    for seed in (0, 1):
        o = ogbfs.gbfs(sp, ogbfs.table_source(sp, tab), budget=484, rho=5, seed=seed)
        lres = tt.gbfs_search(512, 512, 512, 484, tt.search_opts(family=1, seed=seed), table=tab)
        assert _trace_key(lres.trace) == _oracle_key(o)
        assert lres.space_feasible == 130438


def test_gbfs_bad_s0():
    with pytest.raises(tt.TileTuneError) as e:
        tt.gbfs_search(64, 64, 64, 10, tt.search_opts(has_s0=1, s0=tt.to_config(((32, 1, 1, 1), (64, 1), (64, 1, 1, 1)))),
                       cost=lambda s: 1.0)
    assert e.value.status == tt.E_INVAL


def test_gbfs_batch_source_and_evaluator_failure():
    sp = Spec(64, 64, 64)
    seen = []

    def batch(states):
        seen.append(len(states))
        return [costs.t1_cost(s) for s in states]

    res = tt.gbfs_search(64, 64, 64, 300, tt.search_opts(seed=5, width=8), batch=batch)
    o = ogbfs.gbfs(sp, ogbfs.fn_source(costs.t1_cost), budget=300, rho=5, seed=5, width=8)
    assert _trace_key(res.trace) == _oracle_key(o)
    assert max(seen) > 5                                     # W = 8 rounds expose > rho candidates

    calls = []

    def failing(states):
        calls.append(1)
        if len(calls) > 3:
            raise RuntimeError("boom")
        return [1.0] * len(states)

    with pytest.raises(tt.TileTuneError) as e:
        tt.gbfs_search(64, 64, 64, 300, tt.search_opts(seed=5), batch=failing)
    assert e.value.status == tt.E_EVALUATOR


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_na2c_eps0_trace_parity(seed):
    # epsilon = 0: the policy is never consulted -> bit-exact traversal (reading O9)
    sp = Spec(64, 64, 64)
    tab = costs.table(sp, lambda s: costs.t2_cost(sp, s))
    p = ona2c.Params(epsilon=0.0)
    o = ona2c.na2c(sp, ogbfs.table_source(sp, tab), budget=300, params=p, seed=seed)
    lres = tt.na2c_search(64, 64, 64, 300, tt.search_opts(seed=seed, epsilon=0.0), table=tab)
    assert _trace_key(lres.trace) == _oracle_key(o)


def test_na2c_eps0_small_batch_parity():
    sp = Spec(64, 64, 64)
    p = ona2c.Params(epsilon=0.0, batch=3, steps=2)
    o = ona2c.na2c(sp, ogbfs.fn_source(costs.t1_cost), budget=150, params=p, seed=7)
    lres = tt.na2c_search(64, 64, 64, 150, tt.search_opts(seed=7, epsilon=0.0, batch=3, steps_T=2),
                          cost=costs.t1_cost)
    assert _trace_key(lres.trace) == _oracle_key(o)


@pytest.mark.parametrize("seed,table,budget,kw", [
    (0, "t2", 200, {}),
    (1, "t1", 200, {}),
    (2, "t2", 160, {"batch": 8, "steps": 2, "gamma": 0.5}),
    # Alg. 2's own placement of "Train ..." inside the "for s' in B_collect" loop
    (3, "t2", 96, {"train_per_candidate": True}),
    (4, "t1", 80, {"train_per_candidate": True, "batch": 6}),
])
def test_na2c_policy_trace_parity(seed, table, budget, kw):
    # epsilon = 0.8 (the policy is followed with probability eps): the actor is sampled
    # and both networks are trained after every batch, so the traversal depends on the MLP
    # arithmetic.  Oracle and library sum in the same order with the same libm (reading Z24):
    # the traces, i.e. every state and cost in order, must be identical.
    sp = Spec(64, 64, 64)
    f = (lambda s: costs.t2_cost(sp, s)) if table == "t2" else costs.t1_cost
    tab = costs.table(sp, f)
    p = ona2c.Params(epsilon=0.8, **kw)
    o = ona2c.na2c(sp, ogbfs.table_source(sp, tab), budget=budget, params=p, seed=seed)
    lo = {"batch": "batch", "steps": "steps_T", "gamma": "gamma", "train_per_candidate": "train_per_candidate"}
    lres = tt.na2c_search(64, 64, 64, budget, tt.search_opts(seed=seed, epsilon=0.8, **{lo[k]: v for k, v in kw.items()}),
                          table=tab)
    assert _trace_key(lres.trace) == _oracle_key(o)
    assert lres.best_cost == o.best_cost
    if kw.get("train_per_candidate"):     # the placement of line 24 really changes the trajectory
        kb = dict(kw, train_per_candidate=False)
        ob = ona2c.na2c(sp, ogbfs.table_source(sp, tab), budget=budget, params=ona2c.Params(epsilon=0.8, **kb),
                        seed=seed)
        assert _oracle_key(ob) != _oracle_key(o)


def test_na2c_policy_properties():
    # epsilon = 0.8 (policy consulted): invariants and search quality on top of the trace parity
    sp = Spec(64, 64, 64)
    res = tt.na2c_search(64, 64, 64, 988, tt.search_opts(seed=3), cost=costs.t1_cost)
    states = [r["state"] for r in res.trace]
    assert len(states) == len(set(states)) == 988
    bests = [r["best"] for r in res.trace]
    assert all(x >= y for x, y in zip(bests, bests[1:]))
    assert all(space.legitimate(sp, s) for s in states)
    # S:536-style: beats random search on the T1 preset in most paired seeds
    allst = list(space.enumerate_configs(sp))
    wins = 0
    for seed in range(10):
        a = tt.na2c_search(64, 64, 64, 988, tt.search_opts(seed=seed), cost=costs.t1_cost).best_cost
        pick = SplitMix64(1000 + seed).sample_indices(len(allst), 988)
        wins += a <= min(costs.t1_cost(allst[i]) for i in pick)
    assert wins >= 7


def test_binding_simt_and_umma():
    ls = tt.make_space(512, 512, 512, family=1)
    b = tt.binding(ls, ((4, 2, 8, 8), (64, 8), (4, 4, 4, 8)))
    assert (b.grid_x, b.grid_y, b.block_x, b.tile_m, b.tile_n, b.tile_k) == (4, 4, 256, 128, 128, 8)
    assert b.smem_bytes == 2 * (128 + 128 + 8) * 8 * 4
    ls = tt.make_space(4096, 4096, 4096, family=3)
    b = tt.binding(ls, ((16, 2, 1, 128), (64, 64), (16, 1, 1, 256)))
    assert b.cluster_x == 2 and b.tile_m == 256 and b.tile_n == 256 and b.stages >= 2
    # idesc: F32 accum (bit 4), bf16 A/B (bits 7, 10), B MN-major (bit 16), N>>3 at 17, M>>4 at 24
    assert b.idesc == (1 << 4) | (1 << 7) | (1 << 10) | (1 << 16) | ((256 >> 3) << 17) | ((256 >> 4) << 24)
    with pytest.raises(tt.TileTuneError) as e:
        tt.binding(ls, space.initial_state(Spec(4096, 4096, 4096)))
    assert e.value.status == tt.E_INFEASIBLE
    # n1 = 2: clusters of m1 n1 CTAs along N sharing A (multicast); the cluster tile spans n1 n2 n3
    b = tt.binding(ls, ((16, 2, 1, 128), (32, 128), (8, 2, 1, 256)))
    assert (b.cluster_x, b.tile_m, b.tile_n) == (4, 256, 512) and b.grid_x % 4 == 0
    b = tt.binding(ls, ((32, 1, 1, 128), (32, 128), (16, 2, 1, 128)))
    assert (b.cluster_x, b.tile_m, b.tile_n) == (2, 128, 256) and b.grid_x % 2 == 0
    with pytest.raises(tt.TileTuneError) as e:                 # n1 = 4 stays outside J_hw
        tt.binding(ls, ((16, 2, 1, 128), (32, 128), (4, 4, 1, 256)))
    assert e.value.status == tt.E_INFEASIBLE


@pytest.mark.parametrize("width,fam,dims", [(1, 0, (64, 64, 64)), (8, 0, (64, 64, 64)), (4, 1, (512, 512, 512))])
def test_random_search_parity(width, fam, dims):
    from oracle import random_search as orand
    sp = Spec(*dims, family=fam)
    tab = costs.table(sp, lambda s: costs.t2_cost(sp, s))
    o = orand.random_search(sp, ogbfs.table_source(sp, tab), budget=200, seed=9, width=width)
    m, k, n = dims
    lres = tt.random_search(m, n, k, 200, tt.search_opts(family=fam, seed=9, width=width), table=tab)
    assert _trace_key(lres.trace) == _oracle_key(o)
    # whole feasible set when budget exceeds it ("evaluates the whole space")
    small = Spec(16, 16, 16, 2, 2, 2)
    fn = lambda s: costs.t1_cost(s, targets=((1.0, 3.0), (2.0, 2.0), (3.0, 1.0)))
    r = tt.random_search(16, 16, 16, 1000, tt.search_opts(dm=2, dk=2, dn=2, seed=1), cost=fn)
    assert r.evals == 125 and r.best_cost == ogbfs.brute_force(small, fn)[0]


def test_na2c_T_decay_schedule_parity():
    # P:336 decay process: T_e = max(floor, T0 - e // every); eps = 0 keeps the traversal exact
    sp = Spec(64, 64, 64)
    tab = costs.table(sp, lambda s: costs.t2_cost(sp, s))
    p = ona2c.Params(epsilon=0.0, steps=8, steps_floor=2, decay_every=3, batch=6)
    o = ona2c.na2c(sp, ogbfs.table_source(sp, tab), budget=250, params=p, seed=2)
    lres = tt.na2c_search(64, 64, 64, 250, tt.search_opts(seed=2, epsilon=0.0, steps_T=8, steps_T_floor=2,
                                                          steps_T_decay_every=3, batch=6), table=tab)
    assert _trace_key(lres.trace) == _oracle_key(o)
    # the schedule changes the traversal relative to a constant T = 8
    const = tt.na2c_search(64, 64, 64, 250, tt.search_opts(seed=2, epsilon=0.0, steps_T=8, batch=6), table=tab)
    assert _trace_key(const.trace) != _trace_key(lres.trace)


def test_umma_tail_split_policy(monkeypatch):
    # default policy (runs with and without a GPU: 74 co-resident pairs either way): split 4096^3 bf16 256-pair-tile configs (one full wave of
    # data-parallel tiles, double-buffered accumulator, >= 8 us estimated saving); never when
    # every tile would be split or the accumulator is single-buffered; TT_TAIL_SPLIT=0 disables
    monkeypatch.delenv("TT_TAIL_SPLIT", raising=False)
    sp = tt.make_space(4096, 4096, 4096, family=3)
    # round 2: the last full wave joins the remainder (stream-K over 256 % 74 + 74 tiles, all 74 clusters)
    info = tt.binding(sp, ((16, 2, 1, 128), (32, 128), (16, 1, 1, 256)))
    assert (info.split_tiles, info.split_workers) == (256 % 74 + 74, 74)
    assert tt.binding(sp, ((16, 2, 1, 128), (64, 64), (8, 1, 2, 256))).split_tiles == 0       # 512 acc columns
    assert tt.binding(tt.make_space(1024, 8192, 8192, family=3),
                      ((2, 2, 2, 128), (128, 64), (32, 1, 1, 256))).split_tiles == 0          # 64 tiles < 74
    assert tt.binding(tt.make_space(2048, 2048, 2048, family=3),
                      ((16, 1, 1, 128), (16, 128), (16, 1, 1, 128))).split_tiles == 0        # saving < 8 us
    monkeypatch.setenv("TT_TAIL_SPLIT", "0")
    assert tt.binding(sp, ((16, 2, 1, 128), (32, 128), (16, 1, 1, 256))).split_tiles == 0


def test_aggregate_matches_oracle():
    # a7 / reading Z10: the statistic tt_measure applies to its per-repeat event timings
    # (tt_aggregate, the same host function) equals oracle/measure.py bit for bit on injected
    # samples ("fake clock"), odd and even R, ties, R = 1, one outlier.
    from oracle import measure
    rng = np.random.default_rng(5)
    cases = [[1.0, 2.0, 3.0, 4.0, 100.0, 5.0, 6.0, 7.0, 8.0, 9.0], [2.5], [3.0, 1.0, 2.0], [4.0, 4.0, 1.0, 4.0]]
    cases += [list(rng.lognormal(-9, 0.3, size=R)) for R in (2, 5, 10, 11, 64)]
    for xs in cases:
        got = tt.aggregate(xs)
        want = measure.aggregate(xs)
        assert (got.cost_s, got.mean_s, got.min_s, got.stdev_s, got.repeats) == \
            (want["cost"], want["mean"], want["min"], want["stdev"], want["repeats"]), xs
    with pytest.raises(tt.TileTuneError):
        tt.aggregate([])


def test_binding_rejects_bad_operands():
    # the ABI sees raw pointers only: the binding must stop wrong dtypes, strided views, shape
    # mismatches and host tensors before the library reads or writes past a buffer (CPU-only check:
    # every case raises before any library call)
    import torch
    cfg = ((2, 2, 4, 4), (4, 8), (2, 2, 4, 4))
    A = torch.zeros(64, 32)
    B = torch.zeros(32, 64)
    C = torch.zeros(64, 64)
    with pytest.raises(ValueError):                      # host tensors to the device entry point
        tt.gemm(A, B, C, tt.FAM_F32_SIMT, cfg)
    with pytest.raises(TypeError):                       # bf16 operands for the fp32 family
        tt.gemm(A.bfloat16(), B.bfloat16(), C, tt.FAM_F32_SIMT, cfg)
    with pytest.raises(TypeError):                       # fp32 operands for the bf16 family
        tt.gemm(A, B, C, tt.FAM_BF16_UMMA, cfg)
    with pytest.raises(TypeError):                       # C must be fp32
        tt.gemm(A, B, C.bfloat16(), tt.FAM_F32_SIMT, cfg)
    with pytest.raises(ValueError):                      # a transposed view is not row-major
        tt.gemm(A, torch.zeros(64, 32).t(), C, tt.FAM_F32_SIMT, cfg)
    ctx = object.__new__(tt.Context)
    ctx.h = None
    with pytest.raises(ValueError):                      # shapes that do not chain
        tt.Context.gemm_host(ctx, A, torch.zeros(16, 64), C, tt.FAM_F32_SIMT, cfg)
    with pytest.raises(TypeError):
        tt.Context.gemm_host(ctx, A.double(), B, C, tt.FAM_F32_SIMT, cfg)


def test_scoring_opts_reading_z12():
    # reading Z12 (slow candidates) and racing: the options every DEVICE / sharded search uses
    sp = tt.make_space(2048, 2048, 2048, family=tt.FAM_F32_SIMT)
    t_roof = tt.roofline_seconds(sp, device=-1)
    import torch
    if not torch.cuda.is_available():                 # no device: 148 SMs x 1965 MHz x 256 flop/clk/SM
        assert t_roof == pytest.approx(2 * 2048 ** 3 / (148 * 1965e6 * 256), rel=1e-12)
    o = tt.search_opts(family=1)
    s0 = tt.scoring_opts(sp, o, math.inf)
    assert s0.cut_s == pytest.approx(max(1e-3, 50 * t_roof)) and s0.race_s == 0.0   # applies to s0 too
    inc = 385e-6
    m = tt.scoring_opts(sp, o, inc)
    assert m.cut_s == pytest.approx(min(max(20 * inc, 1e-3), max(1e-3, 50 * t_roof)))
    assert m.race_s == pytest.approx(1.1 * inc)
    big = tt.scoring_opts(sp, o, 5.0)                  # an incumbent near s0: the absolute cut rules
    assert big.cut_s == pytest.approx(max(1e-3, 50 * t_roof))
    off = tt.scoring_opts(sp, tt.search_opts(family=1, cut_roofline_x=0.0, race_factor=0.0), math.inf)
    assert off.cut_s == 0.0 and off.race_s == 0.0
    fixed = tt.scoring_opts(sp, tt.search_opts(family=1, measure={"cut_s": 0.5}), inc)
    assert fixed.cut_s == 0.5                          # an explicit cut is kept
    bf = tt.make_space(4096, 4096, 4096, family=tt.FAM_BF16_UMMA)
    assert tt.roofline_seconds(bf) < tt.roofline_seconds(tt.make_space(4096, 4096, 4096, family=tt.FAM_F32_SIMT)) / 16


@pytest.mark.parametrize("mode", ["1", "2", "3", "4"])
@pytest.mark.parametrize("fam,dims,cfg", [
    (3, (4096, 4096, 4096), ((16, 2, 1, 128), (32, 128), (16, 1, 1, 256))),   # bench config: 256 pair tiles
    (3, (2048, 2048, 512), ((16, 1, 1, 128), (8, 64), (16, 1, 1, 128))),      # 256 single-CTA tiles
    (3, (2048, 2048, 512), ((8, 2, 1, 128), (8, 64), (8, 1, 1, 256))),        # 64 pair tiles < 74 pairs
    (3, (2048, 2048, 512), ((16, 1, 1, 128), (8, 64), (16, 2, 1, 64))),       # n1 = 2 clusters
    (2, (4096, 4096, 4096), ((16, 2, 1, 128), (64, 64), (16, 1, 1, 256))),    # tf32 best (round 2)
    (3, (1024, 8192, 8192), ((2, 2, 2, 128), (128, 64), (32, 1, 2, 128))),   # 8-GPU shard
])
def test_umma_schedule_covers_and_waits_only_on_lower_clusters(mode, fam, dims, cfg, monkeypatch):
    # the persistent tcgen05 schedule (the kernel's own Sched code, evaluated on the
    # host) gives every (tile, k-block) to exactly one cluster; a split tile's pieces combine in
    # ascending k (order = pieces below); and every piece that waits (order > 0) waits only on
    # pieces that are the FIRST item of a LOWER-index cluster -- the deadlock-freedom argument
    # (no co-residency assumption), for every split policy.
    monkeypatch.setenv("TT_TAIL_SPLIT", mode)
    M, N, K = dims
    sp = tt.make_space(M, N, K, family=fam)
    assert tt.is_legitimate(sp, cfg) == (True, True)
    k0, per = tt.umma_schedule(sp, cfg)
    tiles = cfg[0][0] * cfg[2][0]
    owner = {}
    pieces = {}
    for w, items in enumerate(per):
        for q, (tile, kb0, kb1, order, split) in enumerate(items):
            assert 0 <= tile < tiles and 0 <= kb0 < kb1 <= k0
            assert bool(split) == (not (kb0 == 0 and kb1 == k0))
            for kb in range(kb0, kb1):
                assert (tile, kb) not in owner            # covered at most once
                owner[(tile, kb)] = (w, q)
            pieces.setdefault(tile, []).append((kb0, kb1, order, w, q))
    assert len(owner) == tiles * k0                       # ... and at least once
    for tile, ps in pieces.items():
        ps.sort()
        for rank, (kb0, kb1, order, w, q) in enumerate(ps):
            assert order == rank                          # ascending-k combine order
            for (b0, b1, o2, v, q2) in ps[:rank]:
                assert v < w and q2 == 0                  # waits only on lower clusters' first items
