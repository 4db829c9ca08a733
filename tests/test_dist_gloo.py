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

    if mode.startswith("auto_dyn"):         # auto with every round long enough to claim dynamically
        tdist._AUTO_CLAIMS = 0
    amode = "auto" if mode.startswith("auto") else ("lpt" if mode == "two_phase" else mode)
    phase_log = []

    def measure_phase(states, mine, phase, probes):
        # fake tt_measure_phase: the probe is the cost; the probe alone decides states above 1.8
        # (T2 costs lie in [1, 2): about a fifth of them)
        vals, fin, secs = [0.0] * len(states), [False] * len(states), [0.0] * len(states)
        for j, (s, m) in enumerate(zip(states, mine)):
            if not m:
                continue
            c = costs.t2_cost(sp, s)
            phase_log.append((phase, s))
            if phase == 1:
                vals[j], fin[j], secs[j] = c, c > 1.8, 1e-4
                if fin[j]:
                    measured.append(s)
            else:
                assert probes[j] == c
                measured.append(s)
                vals[j], fin[j], secs[j] = c, True, 1e-3
        return vals, fin, secs

    def make():
        return tdist.ShardedEvaluator(measure_one, store=tdist.default_store() if amode in ("dynamic", "auto") else None,
                                      assign=amode if amode != "dynamic" else None,
                                      space=tt.make_space(64, 64, 64) if amode in ("lpt", "auto") else None,
                                      measure_phase=measure_phase if mode.endswith("two_phase") else None)

    ev = make()
    assert ev.assign == amode
    if algo == "gbfs":
        res = tt.gbfs_search(64, 64, 64, 300, tt.search_opts(seed=4, width=8), batch=ev)
    else:
        res = tt.na2c_search(64, 64, 64, 200, tt.search_opts(seed=4, epsilon=0.0), batch=ev)
    # a second search in the same process group (fresh evaluator: its own store keys)
    n_first = len(measured)
    phases_first = list(phase_log)
    ev2 = make()
    res2 = tt.gbfs_search(64, 64, 64, 120, tt.search_opts(seed=9, width=4), batch=ev2)
    row_ranges = tdist.row_shard(8192, world, rank)
    out[rank] = ([(r["state"], r["cost"]) for r in res.trace], n_first, ev.rounds, row_ranges,
                 [(r["state"], r["cost"]) for r in res2.trace], len(measured) - n_first,
                 (ev.spec_measured, ev.spec_used, ev2.spec_measured, ev2.spec_used), sorted(set(ev.round_modes)),
                 phases_first, list(measured[:n_first]))
    dist.destroy_process_group()


@pytest.mark.parametrize("algo,mode", [("gbfs", "static"), ("na2c", "static"), ("gbfs", "dynamic"),
                                       ("na2c", "dynamic"), ("gbfs", "lpt"), ("na2c", "lpt"),
                                       ("gbfs", "auto"), ("gbfs", "auto_dyn"), ("gbfs", "two_phase"),
                                       ("na2c", "two_phase"), ("gbfs", "auto_dyn_two_phase")])
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
    t0, n0, rounds0, rr0, u0, m0, sp0, md0, pl0, done0 = out[0]
    t1, n1, rounds1, rr1, u1, m1, sp1, md1, pl1, done1 = out[1]
    assert md0 == md1                                      # every rank took the same per-round modes
    if mode == "auto_dyn":
        assert md0 == ["dynamic"]
    if mode == "auto_dyn_two_phase":
        # dynamic claims everywhere (speculative probes of g(s0) claimed in round 0), except the
        # round that finishes those probes, which runs its phase 2 as a two-phase round
        assert md0 == ["dynamic", "two-phase"]
    if mode.endswith("two_phase"):
        # rounds with more candidates than ranks (or with probes taken speculatively in round 0)
        # ran in two phases; over both ranks every state was probed at most once, every requested
        # state was completed exactly once (whole, by its probe when the probe decided it -- cost
        # > 1.8 in the fake --, or by phase 2), and phase 2 ran only for probed states
        assert "two-phase" in md0
        p1 = [s for ph, s in pl0 + pl1 if ph == 1]
        p2 = [s for ph, s in pl0 + pl1 if ph == 2]
        assert len(p1) == len(set(p1)) and len(p2) == len(set(p2)) and set(p2) <= set(p1)
        sp64 = Spec(64, 64, 64)
        assert all(costs.t2_cost(sp64, s) <= 1.8 for s in p2)
        done = done0 + done1
        requested = [s for s, _ in ref]
        assert len(done) == len(set(done)) and set(requested) <= set(done)
        # the only completed states nobody requested are speculative probes the cut decided
        g0 = set(space.neighbors(sp64, space.initial_state(sp64)))
        assert set(done) - set(requested) <= {s for s in g0 if costs.t2_cost(sp64, s) > 1.8}
    assert t0 == t1 == ref                                 # identical traversal on every rank = oracle
    assert sp0 == sp1                                      # every rank agrees on the speculation
    if mode != "static" and mode != "dynamic":             # g(s0) measured while s0 runs (1 idle rank)
        assert sp0[0] == len(space.neighbors(sp, space.initial_state(sp))) and 5 <= sp0[1] <= sp0[0]
    else:
        assert sp0 == (0, 0, 0, 0)
    if not mode.endswith("two_phase"):
        assert n0 + n1 == len(ref) + sp0[0] - sp0[1]       # each candidate measured exactly once
    if mode == "static":
        assert abs(n0 - n1) <= rounds0                     # round-robin balance
    assert rr0 == (0, 4096) and rr1 == (4096, 8192)        # exact row partition
    # second search in the same group: still the oracle traversal, each candidate measured once
    o2 = ogbfs.gbfs(sp, ogbfs.table_source(sp, tab), budget=120, rho=5, seed=9, width=4)
    assert u0 == u1 == [(r.state, r.cost) for r in o2.trace]
    if not mode.endswith("two_phase"):
        assert m0 + m1 == 120 + sp0[2] - sp0[3]


def test_lpt_owners():
    # longest first to the least-loaded rank; deterministic ties
    assert tdist.ShardedEvaluator.lpt_owners([1.0, 1.0, 1.0, 1.0], 2) == [0, 1, 0, 1]
    assert tdist.ShardedEvaluator.lpt_owners([5.0, 1.0, 1.0, 1.0, 1.0, 1.0], 2) == [0, 1, 1, 1, 1, 1]
    assert tdist.ShardedEvaluator.lpt_owners([3.0, 3.0, 2.0, 2.0, 2.0], 2) == [0, 1, 0, 1, 0]

def _states(n, M=64):
    from paper_1909_10616_b200 import tiletune as tt
    return tt.enumerate_configs(tt.make_space(M, M, M), 0, n)


def test_projection_static_and_exchange():
    st = _states(13)
    rounds = [st[:1], st[1:5], st[5:13]]
    rt = [[1.0], [1.0, 2.0, 3.0, 4.0], [0.5] * 8]
    rc = [[1.0] * len(r) for r in rounds]
    kw = dict(space=None, assign="static", speculate=False, per_round_s=0.0)
    assert tdist.simulate_sharded(rounds, rc, rt, 1, **kw)["wall_s"] == 1.0 + 10.0 + 4.0
    # G = 2 round robin: round 2 shares (1+3, 2+4) -> 6; round 3 -> 2.0
    assert tdist.simulate_sharded(rounds, rc, rt, 2, **kw)["wall_s"] == 1.0 + 6.0 + 2.0
    kw["per_round_s"] = 0.1
    assert abs(tdist.simulate_sharded(rounds, rc, rt, 8, **kw)["wall_s"] - (1.1 + 4.1 + 0.6)) < 1e-12


def test_projection_lpt_dynamic_and_speculation():
    from paper_1909_10616_b200 import tiletune as tt
    sp = tt.make_space(64, 64, 64)
    s0 = tt.unrank(sp, tt.count_configs(sp) - 1)            # the untiled s0 (rank count - 1)
    g = tt.neighbors(sp, s0)
    assert len(g) >= 4
    # round 0 = s0 (2.0); round 1 = four of g(s0), measured at 1.5 / 1.0 / 1.0 / 1.0; round 2 = one more
    rest = [s for s in _states(40) if s not in g and s != s0][:1]
    rounds = [[s0], g[:4], rest]
    rt = [[2.0], [1.5, 1.0, 1.0, 1.0], [3.0]]
    rc = [[1e-3], [2e-3, 1e-3, 1e-3, 1e-3], [1e-3]]
    one = tdist.simulate_sharded(rounds, rc, rt, 1, space=sp, per_round_s=0.0)
    assert one["wall_s"] == 2.0 + 4.5 + 3.0 and one["spec_measured"] == 0
    # G = 2: the idle rank measures g(s0) while s0 runs (each speculative state costing 1.5 here);
    # round 1 is served from that cache
    two = tdist.simulate_sharded(rounds, rc, rt, 2, space=sp, per_round_s=0.0, spec_time=lambda s: 1.5)
    n_spec = len(g)
    assert two["spec_measured"] == n_spec and two["spec_used"] == 4
    assert two["wall_s"] == max(2.0, 1.5 * n_spec) + 0.0 + 3.0
    # default round-0 cost of a speculative state: a whole measurement with no incumbent to race
    # against, 11 launches of (cost + calibrated per-launch overhead)
    # The calibration rule (secs / launches - cost; launches 11, or 3 when raced at 1.1 x the
    # incumbent) over the recorded rounds gives 2/11 - 1e-3, 1.5/3 - 2e-3, 3 x (1/11 - 1e-3),
    # 3/11 - 1e-3: median (index 3 of 6) 2/11 - 1e-3.  Unrecorded states cost the median recorded
    # cost, 1e-3.
    dflt = tdist.simulate_sharded(rounds, rc, rt, 2, space=sp, per_round_s=0.0)
    o = 2 / 11 - 1e-3
    r0 = 11 * ((2e-3 + o) + (n_spec - 1) * (1e-3 + o))
    assert abs(dflt["wall_s"] - (max(2.0, r0) + 0.0 + 3.0)) < 1e-9
    # without speculation: LPT puts the dear candidate (predicted from its costlier neighbour) alone
    nos = tdist.simulate_sharded(rounds, rc, rt, 2, space=sp, per_round_s=0.0, speculate=False)
    assert nos["spec_measured"] == 0 and nos["wall_s"] <= 2.0 + 2.5 + 3.0
    # dynamic claims: list scheduling, each claim costs per_claim_s
    dyn = tdist.simulate_sharded([g[:4]], [[1e-3] * 4], [[4.0, 1.0, 1.0, 1.0]], 2, space=sp, assign="dynamic",
                                 per_round_s=0.0, per_claim_s=0.0)
    assert dyn["wall_s"] in (4.0, 3.0 + 1.0) and dyn["modes"] == ["dynamic"]


def test_projection_two_phase():
    # one round of 5 candidates on 2 ranks, with the one-GPU run's phase split recorded: phase 1
    # (probes) then phase 2 (the rest), each balanced by LPT, two exchanges
    st = _states(6)
    rounds = [st[:1], st[1:6]]
    costs_ = [[1e-3], [1e-3, 1e-3, 1e-3, 5e-3, 1e-3]]
    rt = [[0.011], [0.011, 0.011, 0.011, 0.015, 0.011]]
    ph = [([], [], []), ((0.001, 0.001, 0.001, 0.005, 0.001), (1e-3, 1e-3, 1e-3, 5e-3, 1e-3), (0, 0, 0, 1, 0))]
    r = tdist.simulate_sharded(rounds, costs_, rt, 2, space=None, two_phase=True, round_phase1=ph,
                               per_round_s=0.0, speculate=False)
    assert r["modes"] == ["lpt", "two-phase"]
    # phase 1: probes 5 ms + 1 ms vs 4 x 1 ms -> LPT gives max(0.005 + ..., ...); phase 2: the four
    # unfinished candidates' 10 ms each split 2 + 2 -> 20 ms; the probe-finished one has none
    p1 = [0.001, 0.001, 0.001, 0.005, 0.001]
    w_lpt = tdist.ShardedEvaluator.lpt_owners([1.0] * 5, 2)     # equal predictions (no space)
    b1 = [sum(t for t, o in zip(p1, w_lpt) if o == r_) for r_ in (0, 1)]
    assert abs(r["wall_s"] - (0.011 + max(b1) + 0.020)) < 1e-12


def test_launch_model_and_phase2_plan():
    ev = tdist.ShardedEvaluator(lambda s: 1.0)
    L = tdist.ShardedEvaluator.launches
    assert L(1.0, float("inf"), 0.0) == 11 and L(1.0, 1.0, 0.0) == 11
    assert L(1.2, 1.0, 0.0) == 3 and L(1.2, 1.0, 1.1) == 1
    ev.world = 2
    ev.set_known({((1,), (1,), (1,)): 1.0})                     # incumbent 1.0
    owner2, w2 = ev.phase2_plan([1.0, 2.0, 1.05, 9.0], [False, False, False, True], 5.0)
    # full (10 more launches), raced (2 more), full; the probe-finished one has no phase 2
    assert owner2[3] is None and w2 == [10 * 1.0, 2 * 2.0, 10 * 1.05]
    assert owner2[:3] == [1, 1, 0]                             # LPT: 10.5 | 10.0 + 4.0
    # the overhead calibrates from (cost, seconds): 11 launches of 1.0 + 0.5 each
    ev._calibrate([1.0], [11 * 1.5], float("inf"), 0.0)
    assert ev._over == 0.5


def test_predicted_cost_is_geomean_over_legit_neighbors():
    # the LPT prediction walks raw moves (no ctypes); with only legitimate states measured it must
    # equal the geometric mean over the measured part of g(s) from the library's neighbour function
    import math
    import random

    from paper_1909_10616_b200 import tiletune as tt
    for fam, M in ((tt.FAM_BF16_UMMA, 4096), (tt.FAM_F32_SIMT, 512)):
        sp = tt.make_space(M, M, M, family=fam)
        feas = tt.enumerate_feasible(sp)[0]
        rng = random.Random(fam)
        ev = tdist.ShardedEvaluator(lambda s: 1.0, space=sp)
        ev.set_known({s: rng.random() for s in rng.sample(feas, min(len(feas), 150))})
        for s in rng.sample(feas, 60):
            nb = [ev.known[t] for t in tt.neighbors(sp, s) if t in ev.known]
            want = math.exp(sum(math.log(v) for v in nb) / len(nb)) if nb else min(ev.known.values())
            assert abs(ev._predicted_cost(s) - want) <= 1e-12 * want
            assert set(tt.neighbors(sp, s)) <= set(ev._moves(s))


def test_auto_mode():
    # auto: dynamic claims only when the median predicted measurement time is >= 10 claims (2 ms)
    assert tdist.auto_mode([1e-3] * 5) == "lpt" and tdist.auto_mode([5e-3] * 5) == "dynamic"
    assert tdist.auto_mode([5e-3, 5e-3, 1e-3, 1e-3, 1e-3]) == "lpt"


def test_warm_up_leaves_no_state():
    from paper_1909_10616_b200 import tiletune as tt
    sp = tt.make_space(4096, 4096, 4096, family=tt.FAM_BF16_UMMA)
    ev = tdist.ShardedEvaluator(lambda s: 1.0, space=sp)
    ev.warm_up(tt.enumerate_configs(sp, 0, 16))
    assert ev.known == {} and ev._known_code == {} and ev._over == 0.0 and ev._over_obs == []
    assert ev.rounds == 0 and ev.plan_s == 0.0


def test_projection_two_phase_speculative_probes():
    # round 0 (s0 alone) on 2 ranks: the idle rank takes only the cold probes of g(s0) (recorded
    # phase-1 seconds, else their median); round 1 (four of g(s0)) then runs only phase 2
    from paper_1909_10616_b200 import tiletune as tt
    sp = tt.make_space(64, 64, 64)
    s0 = tt.unrank(sp, tt.count_configs(sp) - 1)
    g = tt.neighbors(sp, s0)
    rounds = [[s0], g[:4]]
    rc = [[1e-3], [1e-3, 1e-3, 1e-3, 1e-3]]
    rt = [[0.011], [0.011, 0.011, 0.011, 0.011]]
    ph = [([], [], []), ((0.001, 0.002, 0.001, 0.001), (1e-3, 1e-3, 1e-3, 1e-3), (0, 0, 0, 0))]
    r = tdist.simulate_sharded(rounds, rc, rt, 2, space=sp, two_phase=True, round_phase1=ph, per_round_s=0.0)
    assert r["modes"][1] == "two-phase" and r["spec_used"] == 4 and r["spec_measured"] == len(g)
    # round 0: s0 (0.011) vs the probes of g(s0) on the idle rank: 4 recorded (0.005) + the rest at
    # the recorded median 0.001; round 1: phase 1 free, phase 2 = 4 x 0.010 (or 0.009) over 2 ranks
    r0 = max(0.011, 0.005 + 0.001 * (len(g) - 4))
    phase2 = sorted([0.010, 0.009, 0.010, 0.010], reverse=True)
    load = [0.0, 0.0]
    for x in phase2:
        load[load.index(min(load))] += x
    assert abs(r["wall_s"] - (r0 + max(load))) < 1e-9
