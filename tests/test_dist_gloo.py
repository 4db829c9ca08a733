"""Multi-process (gloo, world size 2, CPU) coverage of the sharded search:
every rank runs the identical G-BFS / N-A2C, candidates are measured round-robin over ranks and the
costs are all-gathered; the traversal must equal the single-process oracle traversal."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from oracle import costs, gbfs as ogbfs, na2c as ona2c, space
from oracle.space import Spec
from paper_1909_10616_b200 import dist as tdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, algo, out, mode="static"):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1909_10616_b200 import dist as tdist
    from paper_1909_10616_b200 import tiletune as tt

    sp = Spec(64, 64, 64)
    measured = []

    def measure_one(s):
        measured.append(s)
        return costs.t2_cost(sp, s)

    if mode == "auto_dyn":                  # auto with every round long enough to claim dynamically
        tdist._AUTO_CLAIMS = 0
    amode = "auto" if mode.startswith("auto") else mode

    def make():
        return tdist.ShardedEvaluator(measure_one, store=tdist.default_store() if amode in ("dynamic", "auto") else None,
                                      assign=amode if amode != "dynamic" else None,
                                      space=tt.make_space(64, 64, 64) if amode in ("lpt", "auto") else None)

    ev = make()
    assert ev.assign == amode
    if algo == "gbfs":
        res = tt.gbfs_search(64, 64, 64, 300, tt.search_opts(seed=4, width=8), batch=ev)
    else:
        res = tt.na2c_search(64, 64, 64, 200, tt.search_opts(seed=4, epsilon=0.0), batch=ev)
    # a second search in the same process group (fresh evaluator: its own store keys)
    n_first = len(measured)
    ev2 = make()
    res2 = tt.gbfs_search(64, 64, 64, 120, tt.search_opts(seed=9, width=4), batch=ev2)
    row_ranges = tdist.row_shard(8192, world, rank)
    out[rank] = ([(r["state"], r["cost"]) for r in res.trace], n_first, ev.rounds, row_ranges,
                 [(r["state"], r["cost"]) for r in res2.trace], len(measured) - n_first,
                 (ev.spec_measured, ev.spec_used, ev2.spec_measured, ev2.spec_used), sorted(set(ev.round_modes)))
    dist.destroy_process_group()


@pytest.mark.parametrize("algo,mode", [("gbfs", "static"), ("na2c", "static"), ("gbfs", "dynamic"),
                                       ("na2c", "dynamic"), ("gbfs", "lpt"), ("na2c", "lpt"),
                                       ("gbfs", "auto"), ("gbfs", "auto_dyn")])
def test_sharded_search_matches_oracle(algo, mode):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), algo, out, mode), nprocs=world, join=True)
    sp = Spec(64, 64, 64)
    tab = costs.table(sp, lambda s: costs.t2_cost(sp, s))
    if algo == "gbfs":
        o = ogbfs.gbfs(sp, ogbfs.table_source(sp, tab), budget=300, rho=5, seed=4, width=8)
    else:
        o = ona2c.na2c(sp, ogbfs.table_source(sp, tab), budget=200, params=ona2c.Params(epsilon=0.0), seed=4)
    ref = [(r.state, r.cost) for r in o.trace]
    t0, n0, rounds0, rr0, u0, m0, sp0, md0 = out[0]
    t1, n1, rounds1, rr1, u1, m1, sp1, md1 = out[1]
    assert md0 == md1                                      # every rank took the same per-round modes
    if mode == "auto_dyn":
        assert md0 == ["dynamic"]
    assert t0 == t1 == ref                                 # identical traversal on every rank = oracle
    assert sp0 == sp1                                      # every rank agrees on the speculation
    if mode in ("lpt", "auto", "auto_dyn"):                # g(s0) measured while s0 runs (1 idle rank)
        assert sp0[0] == len(space.neighbors(sp, space.initial_state(sp))) and 5 <= sp0[1] <= sp0[0]
    else:
        assert sp0 == (0, 0, 0, 0)
    assert n0 + n1 == len(ref) + sp0[0] - sp0[1]           # each candidate measured exactly once
    if mode == "static":
        assert abs(n0 - n1) <= rounds0                     # round-robin balance
    assert rr0 == (0, 4096) and rr1 == (4096, 8192)        # exact row partition
    # second search in the same group: still the oracle traversal, each candidate measured once
    o2 = ogbfs.gbfs(sp, ogbfs.table_source(sp, tab), budget=120, rho=5, seed=9, width=4)
    assert u0 == u1 == [(r.state, r.cost) for r in o2.trace]
    assert m0 + m1 == 120 + sp0[2] - sp0[3]


def test_lpt_owners():
    # longest first to the least-loaded rank; deterministic ties
    assert tdist.ShardedEvaluator.lpt_owners([1.0, 1.0, 1.0, 1.0], 2) == [0, 1, 0, 1]
    assert tdist.ShardedEvaluator.lpt_owners([5.0, 1.0, 1.0, 1.0, 1.0, 1.0], 2) == [0, 1, 1, 1, 1, 1]
    assert tdist.ShardedEvaluator.lpt_owners([3.0, 3.0, 2.0, 2.0, 2.0], 2) == [0, 1, 0, 1, 0]

def test_projection():
    rt = [[1.0], [1.0, 2.0, 3.0, 4.0], [0.5] * 8]
    assert tdist.projected_sharded_wall(rt, 1) == 1.0 + 10.0 + 4.0
    # G = 2: round 2 shares (1+3, 2+4) -> 6; round 3 -> 2.0
    assert tdist.projected_sharded_wall(rt, 2) == 1.0 + 6.0 + 2.0
    assert tdist.projected_sharded_wall(rt, 8, per_round_s=0.1) == 1.1 + 4.1 + 0.6
    # dynamic: list scheduling in index order, each candidate to the first free rank
    assert tdist.projected_sharded_wall([[4.0, 1.0, 1.0, 1.0, 1.0]], 2, dynamic=True) == 4.0
    assert tdist.projected_sharded_wall([[4.0, 1.0, 1.0, 1.0, 1.0]], 2) == 6.0
    # LPT from predicted weights: the long candidate alone on one rank
    assert tdist.projected_sharded_wall([[4.0, 1.0, 1.0, 1.0, 1.0]], 2, weights=[[4.0, 1.0, 1.0, 1.0, 1.0]]) == 4.0
    # speculative round 0: s0 (2.0) alone; its neighbours a, b (measured later at 1.5 / 1.0) run on
    # the idle ranks meanwhile, so round 1 (a, b) costs nothing and round 2 (c) runs as usual
    nb = {"s0": ["a", "b"], "a": [], "b": []}
    st = [["s0"], ["a", "b"], ["c"]]
    rt = [[2.0], [1.5, 1.0], [3.0]]
    assert tdist.projected_sharded_wall(rt, 1, states=st, neighbors=nb.get) == 2.0 + 2.5 + 3.0
    assert tdist.projected_sharded_wall(rt, 2, states=st, neighbors=nb.get) == 2.5 + 0.0 + 3.0
    assert tdist.projected_sharded_wall(rt, 3, states=st, neighbors=nb.get) == 2.0 + 0.0 + 3.0


def test_predicted_cost_equals_min_over_legit_neighbors():
    # the LPT prediction walks raw moves (no ctypes); with only legitimate states measured it must
    # equal the min over g(s) from the library's neighbour function
    import random

    from paper_1909_10616_b200 import tiletune as tt
    for fam, M in ((tt.FAM_BF16_UMMA, 4096), (tt.FAM_F32_SIMT, 512)):
        sp = tt.make_space(M, M, M, family=fam)
        feas = tt.enumerate_feasible(sp)[0]
        rng = random.Random(fam)
        ev = tdist.ShardedEvaluator(lambda s: 1.0, space=sp)
        ev.known = {s: rng.random() for s in rng.sample(feas, min(len(feas), 150))}
        for s in rng.sample(feas, 60):
            nb = [ev.known[t] for t in tt.neighbors(sp, s) if t in ev.known]
            want = min(nb) if nb else min(ev.known.values())
            assert ev._predicted_cost(s) == want
            assert set(tt.neighbors(sp, s)) <= set(ev._moves(s))


def test_auto_mode_and_projection():
    # auto: dynamic claims only when the median predicted measurement time is >= 10 claims (2 ms)
    short = [tdist._PER_CANDIDATE_S + 1e-3] * 5
    long_ = [tdist._PER_CANDIDATE_S + 5e-3] * 5
    assert tdist.auto_mode(short) == "lpt" and tdist.auto_mode(long_) == "dynamic"
    rt = [[4.0, 1.0, 1.0, 1.0, 1.0]]
    # a round of short predictions projects exactly like LPT, a round of long ones like dynamic
    w_short = [[tdist._PER_CANDIDATE_S + x * 1e-4 for x in (4, 1, 1, 1, 1)]]
    w_long = [[tdist._PER_CANDIDATE_S + x * 1e-2 for x in (4, 1, 1, 1, 1)]]
    for w, kw in ((w_short, {}), (w_long, {"dynamic": True})):
        assert tdist.projected_sharded_wall(rt, 2, auto=True, per_claim_s=0.1, weights=w) == \
            tdist.projected_sharded_wall(rt, 2, per_claim_s=0.1, weights=w, **kw)
