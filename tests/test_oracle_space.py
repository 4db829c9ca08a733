"""Pins for oracle.space (Eq. 1-9) against paper-printed values, closed forms and brute force."""
import itertools
import json
import math
import os

import pytest

from oracle import space
from oracle.space import Spec

AX = {"m": 0, "k": 1, "n": 2}


def S(st):
    return tuple(tuple(v) for v in st)


def test_paper_space_sizes(golden):
    # 484000 / 899756 / 1589952 at d = (4,2,4)
    for row in golden["space_sizes_d424"]:
        assert space.count_configs(Spec(row["m"], row["k"], row["n"])) == row["count"], row["cite"]


def test_small_counts(golden):
    for row in golden["small_counts"]:
        sp = Spec(row["m"], row["k"], row["n"], *row["d"])
        assert space.count_configs(sp) == row["count"], row["cite"]
        assert sum(1 for _ in space.enumerate_configs(sp)) == row["count"]


def test_axis_12(golden):
    g = golden["axis_count_12_d2"]
    assert space.count_axis(12, 2) == g["count"]
    assert [list(t) for t in space.factorizations(12, 2)] == g["list"]


def _brute_axis(value, d):
    """Independent brute force: every d-tuple over range(1, value+1) with the right product."""
    return sum(1 for t in itertools.product(range(1, value + 1), repeat=d) if math.prod(t) == value)


@pytest.mark.parametrize("value,d", [(1, 3), (12, 2), (12, 3), (18, 3), (30, 2), (36, 3), (64, 2),
                                     (16, 4), (27, 3), (60, 3), (7, 4), (8, 4), (96, 2), (100, 3), (45, 2),
                                     (32, 3), (24, 4), (20, 3), (2, 4), (90, 3), (50, 2)])
def test_count_closed_form_vs_bruteforce(value, d):
    # S:91 closed form against exhaustive product check (>= 20 specs)
    assert space.count_axis(value, d) == _brute_axis(value, d) == len(space.factorizations(value, d))


def test_enumeration_order_rank_64():
    sp = Spec(64, 64, 64)
    lst = list(space.enumerate_configs(sp))
    n = space.count_configs(sp)
    assert len(lst) == n == 49392
    flat = [sum(s, ()) for s in lst]
    assert flat == sorted(flat) and len(set(flat)) == n
    assert lst[0] == ((1, 1, 1, 64), (1, 64), (1, 1, 1, 64))
    s0 = space.initial_state(sp)
    assert lst[-1] == s0 and space.rank(sp, s0) == n - 1
    for r in range(0, n, 997):
        assert space.rank(sp, space.unrank(sp, r)) == r
        assert space.unrank(sp, r) == lst[r]


def test_non_square_rank_order():
    # (m, k, n) = (8, 4, 2): rank is mixed radix over (m, k, n) in the paper's order
    sp = Spec(8, 4, 2, 2, 2, 2)
    lst = list(space.enumerate_configs(sp))
    assert len(lst) == 4 * 3 * 2
    for r, s in enumerate(lst):
        assert space.rank(sp, s) == r
        assert math.prod(s[0]) == 8 and math.prod(s[1]) == 4 and math.prod(s[2]) == 2


def test_legitimacy_examples(golden):
    sp = Spec(1024, 1024, 1024)
    assert space.legitimate(sp, space.initial_state(sp))
    ex = golden["illegitimate_example"]
    assert space.legitimate(sp, S(ex["state"])) is ex["legitimate"]
    f = golden["fig4_config_d424"]
    assert space.legitimate(sp, S(f["state"]))                      # S:56 / P:166
    f2 = golden["fig4_config"]
    assert space.legitimate(Spec(1024, 1024, 1024, 2, 2, 2), S(f2["state"]))
    assert not space.legitimate(sp, ((1024, 1, 1), (1024, 1), (1024, 1, 1, 1)))   # wrong length
    assert not space.legitimate(sp, ((2048, 1, 1, 0), (1024, 1), (1024, 1, 1, 1)))  # non-positive


def test_step_examples(golden):
    sp = Spec(1024, 1024, 1024)
    for ex in golden["step_examples"]:
        x, i, j = ex["action"]
        got = space.step(S(ex["state"]), (AX[x], i, j))
        if ex["result"] is None:
            assert got is None or not space.legitimate(sp, got), ex["cite"]
        else:
            assert got == S(ex["result"]), ex["cite"]


def test_action_count(golden):
    assert len(space.actions(Spec(8, 8, 8))) == golden["action_count_d424"]["count"]
    assert len(space.actions(Spec(16, 16, 16, 1, 1, 1))) == 0


def test_s0_neighbors(golden):
    sp = Spec(1024, 1024, 1024)
    g = space.neighbors(sp, space.initial_state(sp))
    assert len(g) == golden["s0_neighbors_1024"]["count"]
    # order: (m,1,0), (m,2,0), (m,3,0), (k,1,0), (n,1,0), (n,2,0), (n,3,0)
    assert g[0] == ((512, 2, 1, 1), (1024, 1), (1024, 1, 1, 1))
    assert g[1] == ((512, 1, 2, 1), (1024, 1), (1024, 1, 1, 1))
    assert g[2] == ((512, 1, 1, 2), (1024, 1), (1024, 1, 1, 1))
    assert g[3] == ((1024, 1, 1, 1), (512, 2), (1024, 1, 1, 1))
    assert g[6] == ((1024, 1, 1, 1), (1024, 1), (512, 1, 1, 2))
    # [[1,1,1,1024],...] contributes 3 states in dim m
    s = ((1, 1, 1, 1024), (1024, 1), (1024, 1, 1, 1))
    assert sum(1 for t in space.neighbors(sp, s) if t[0] != s[0]) == 3
    assert space.neighbors(Spec(16, 16, 16, 1, 1, 1), ((16,), (16,), (16,))) == []


def test_inverse_and_predecessors(golden):
    sp = Spec(1024, 1024, 1024)
    for a in space.actions(sp):
        assert space.inverse_action(space.inverse_action(a)) == a
    s = ((512, 2, 1, 1), (1024, 1), (1024, 1, 1, 1))
    t = space.step(s, (0, 0, 1))
    assert space.step(t, space.inverse_action((0, 0, 1))) == s
    ex = golden["predecessors_example"]
    preds = space.predecessors(sp, S(ex["state"]))
    assert len(preds) == ex["count"]
    for p, a in preds:
        assert space.step(p, a) == S(ex["state"])


@pytest.mark.parametrize("dims,d", [((16, 16, 16), (2, 2, 2)), ((4, 2, 4), (2, 1, 2)), ((64, 64, 64), (4, 2, 4)),
                                    ((32, 8, 16), (4, 2, 4))])
def test_symmetry_closure_conservation(dims, d):
    sp = Spec(*dims, *d)
    allst = list(space.enumerate_configs(sp))
    nb = {s: space.neighbors(sp, s) for s in allst}
    nbset = {s: set(v) for s, v in nb.items()}
    for s, g in nb.items():
        for t in g:
            assert s in nbset[t]                                        # S:120 symmetry
            assert all(math.prod(t[a]) == math.prod(s[a]) for a in range(3))
    s0 = space.initial_state(sp)
    seen, todo = {s0}, [s0]
    while todo:
        for t in nb[todo.pop()]:
            if t not in seen:
                seen.add(t)
                todo.append(t)
    assert seen == set(allst)                                           # S:122 closure


def test_degree_stats_64():
    sp = Spec(64, 64, 64)
    degs = [len(space.neighbors(sp, s)) for s in space.enumerate_configs(sp)]
    assert min(degs) == 7 and max(degs) == 26


def test_encode_decode():
    s = ((32, 32, 1, 1), (256, 4), (32, 32, 1, 1))
    txt = space.encode(s)
    assert txt == '{"m":[32,32,1,1],"k":[256,4],"n":[32,32,1,1]}'
    assert space.decode(txt, Spec(1024, 1024, 1024)) == s
    with pytest.raises(ValueError):
        space.decode('{"m":[32,1.5,1,1],"k":[256,4],"n":[32,32,1,1]}')
    with pytest.raises(ValueError):
        space.decode('{"m":[32,32,1],"k":[256,4],"n":[32,32,1,1]}', Spec(1024, 1024, 1024))


def test_features_s0():
    sp = Spec(1024, 1024, 1024)
    assert space.features(sp, space.initial_state(sp)) == [1, 0, 0, 0, 1, 0, 1, 0, 0, 0]
