"""Property-based parity (hypothesis): library vs oracle on random problem instances, including
non-power-of-two dimensions and depths 1-4 (search stays on the 2-adic sublattice)."""
import math

from hypothesis import given, settings, strategies as st

from oracle import costs, gbfs as ogbfs, space
from oracle.rng import SplitMix64
from oracle.space import Spec
from paper_1909_10616_b200 import tiletune as tt

dims = st.sampled_from([1, 2, 3, 4, 6, 8, 12, 16, 18, 24, 30, 32, 36, 48, 64, 96])
depths = st.integers(min_value=1, max_value=4)


def lib(sp):
    return tt.make_space(sp.m, sp.n, sp.k, sp.dm, sp.dk, sp.dn)


@settings(max_examples=60, deadline=None)
@given(m=dims, k=dims, n=dims, dm=depths, dk=depths, dn=depths)
def test_count_enumerate_rank_neighbors(m, k, n, dm, dk, dn):
    sp = Spec(m, k, n, dm, dk, dn)
    raw = space.count_configs(sp)
    if raw > 20000:
        return
    ls = lib(sp)
    assert tt.count_configs(ls) == raw
    ora = list(space.enumerate_configs(sp))
    assert tt.enumerate_configs(ls) == ora
    r = SplitMix64(m * 1000 + k * 10 + n)
    for i in r.sample_indices(len(ora), 10):
        s = ora[i]
        assert tt.rank(ls, s) == i and tt.unrank(ls, i) == s
        assert tt.neighbors(ls, s) == space.neighbors(sp, s)
        # predecessors of s are exactly the states whose neighbour list contains s (symmetry)
        for t in space.neighbors(sp, s):
            assert s in tt.neighbors(ls, t)


@settings(max_examples=25, deadline=None)
@given(m=st.sampled_from([8, 16, 32, 64]), k=st.sampled_from([8, 16, 32, 64]), n=st.sampled_from([8, 16, 32, 64]),
       seed=st.integers(min_value=0, max_value=2 ** 40), rho=st.integers(min_value=1, max_value=8),
       width=st.integers(min_value=1, max_value=4))
def test_gbfs_parity_random_instances(m, k, n, seed, rho, width):
    sp = Spec(m, k, n)
    raw = space.count_configs(sp)
    budget = max(2, raw // 20)
    fn = lambda s: costs.t2_cost(sp, s, seed_t=seed % 97)
    o = ogbfs.gbfs(sp, ogbfs.fn_source(fn), budget=budget, rho=rho, seed=seed, width=width)
    res = tt.gbfs_search(m, n, k, budget, tt.search_opts(seed=seed, rho=rho, width=width), cost=fn)
    assert [(r["state"], r["cost"]) for r in res.trace] == [(r.state, r.cost) for r in o.trace]
    assert res.best_cost == min(r.cost for r in o.trace)
    assert math.isclose(res.frac_raw, o.evals / raw)
