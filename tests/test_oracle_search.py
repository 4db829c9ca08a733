"""Pins for oracle.rng, oracle.costs, oracle.gbfs (Alg. 1), oracle.mlp, oracle.na2c (Alg. 2) and
oracle.measure against published vectors, hand-worked traces, brute force and closed forms."""
import json
import math
import os
import statistics

import numpy as np
import pytest

from oracle import costs, gbfs, measure, mlp, na2c, space
from oracle.rng import SplitMix64
from oracle.space import Spec

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ------------------------------------------------------------------ rng (reading O7)
def test_splitmix64_published_vector():
    with open(os.path.join(ROOT, "tests", "golden", "splitmix64.json")) as f:
        g = json.load(f)
    r = SplitMix64(g["seed"])
    assert [r.next() for _ in range(5)] == [int(x) for x in g["outputs"]]


def test_sample_without_replacement_uniform():
    r = SplitMix64(3)
    counts = np.zeros(7)
    for _ in range(7000):
        idx = r.sample_indices(7, 3)
        assert len(set(idx)) == 3 and all(0 <= i < 7 for i in idx)
        counts[idx] += 1
    # each index chosen with probability 3/7: 3000 expected, chi^2 with 6 dof well below 30
    chi2 = float(((counts - 3000) ** 2 / 3000).sum())
    assert chi2 < 30
    assert sorted(SplitMix64(1).sample_indices(4, 9)) == [0, 1, 2, 3]   # all if |g| < rho (Z5)


def _published():
    with open(os.path.join(ROOT, "tests", "golden", "splitmix64.json")) as f:
        g = json.load(f)
    return g["seed"], [int(x) for x in g["outputs"]]


def test_bounded_exact_from_published_vector():
    # O7: bounded(n) = floor(next() * n / 2^64) (Lemire multiply-shift).  Expected values are
    # derived here, by integer arithmetic, from the PUBLISHED outputs -- not from oracle.rng.
    seed, outs = _published()
    want = [(o * 26) >> 64 for o in outs]
    assert want == [9, 4, 13, 6, 23]
    assert want != [o % 26 for o in outs]              # a modulo reduction would fail here
    r = SplitMix64(seed)
    assert [r.bounded(26) for _ in range(5)] == want
    # uniform() = (next() >> 11) 2^-53: the top 53 bits as an exact dyadic fraction
    r = SplitMix64(seed)
    assert [r.uniform() for _ in range(5)] == [(o >> 11) / float(1 << 53) for o in outs]


def test_sample_indices_exact_from_published_vector():
    # O7: partial Fisher-Yates, t = 0..r-1: j = t + bounded(L - t), swap idx[t], idx[j];
    # L = 7, r = 3 worked by hand from the published outputs o0, o1, o2:
    #   t=0: j = 0 + (o0 * 7 >> 64) = 2 -> [2,1,0,3,4,5,6]
    #   t=1: j = 1 + (o1 * 6 >> 64) = 2 -> [2,0,1,3,4,5,6]
    #   t=2: j = 2 + (o2 * 5 >> 64) = 4 -> [2,0,4,3,1,5,6]
    seed, outs = _published()
    assert [(outs[0] * 7) >> 64, (outs[1] * 6) >> 64, (outs[2] * 5) >> 64] == [2, 1, 2]
    assert SplitMix64(seed).sample_indices(7, 3) == [2, 0, 4]
    # rho >= L takes every index, in the shuffled order of a full Fisher-Yates
    full = SplitMix64(seed).sample_indices(4, 9)
    idx = [0, 1, 2, 3]
    for t, o in zip(range(4), outs):
        j = t + ((o * (4 - t)) >> 64)
        idx[t], idx[j] = idx[j], idx[t]
    assert full == idx


def test_bounded_range_and_uniform():
    r = SplitMix64(11)
    xs = [r.bounded(26) for _ in range(26000)]
    assert min(xs) == 0 and max(xs) == 25
    assert abs(statistics.mean(xs) - 12.5) < 0.3
    us = [r.uniform() for _ in range(10000)]
    assert 0.0 <= min(us) and max(us) < 1.0


# ------------------------------------------------------------------ cost tables
def test_t1_examples():
    # targets 0, weights 1, [[16],[16],[16]] -> 1 + 3*(4-0)^2 = 49
    assert costs.t1_cost(((16,), (16,), (16,)), targets=((0.0,), (0.0,), (0.0,))) == 49.0
    # targets = own log2 -> exactly 1
    s = ((4, 4, 2, 2), (8, 8), (4, 4, 2, 2))
    assert costs.t1_cost(s) == 1.0


def test_t1_preset_unique_argmin():
    sp = Spec(64, 64, 64)
    best, arg = gbfs.brute_force(sp, costs.t1_cost)
    assert best == 1.0 and arg == ((4, 4, 2, 2), (8, 8), (4, 4, 2, 2))
    vals = [costs.t1_cost(s) for s in space.enumerate_configs(sp)]
    assert vals.count(1.0) == 1


def test_t2_range_and_ties():
    sp = Spec(16, 16, 16, 2, 2, 2)
    vals = [costs.t2_cost(sp, s) for s in space.enumerate_configs(sp)]
    assert all(1.0 <= v < 2.0 for v in vals)
    assert len(set(vals)) == len(vals)


# ------------------------------------------------------------------ G-BFS (Alg. 1)
def test_gbfs_hand_worked_trace():
    # spec m=4,k=1,n=1, d=(2,1,1): states (4,1),(2,2),(1,4).  cost = 3,2,1.  Alg. 1 with rho=5:
    # test s0=(4,1) [3]; pop s0; g = [(2,2)]; test -> push [2], best;  pop (2,2); g = [(4,1),(1,4)];
    # (4,1) visited, test (1,4) [1] -> best; pop (1,4): g = [(2,2)] visited; queue still holds (4,1);
    # pop (4,1): nothing new; queue empty -> stop.
    sp = Spec(4, 1, 1, 2, 1, 1)
    c = {(4, 1): 3.0, (2, 2): 2.0, (1, 4): 1.0}
    res = gbfs.gbfs(sp, gbfs.fn_source(lambda s: c[s[0]]), rho=5, seed=0)
    assert [r.state[0] for r in res.trace] == [(4, 1), (2, 2), (1, 4)]
    assert [r.best for r in res.trace] == [3.0, 2.0, 1.0]
    assert res.best_state[0] == (1, 4) and res.evals == 3


def test_gbfs_no_actions():
    # d = (1,1,1): g(s0) empty -> one evaluation, s0 returned
    sp = Spec(16, 16, 16, 1, 1, 1)
    res = gbfs.gbfs(sp, gbfs.fn_source(lambda s: 5.0))
    assert res.evals == 1 and res.best_state == ((16,), (16,), (16,))


def test_gbfs_completeness_16(golden):
    # P:267 / S:259 / S:534: rho = |A| = 6, no budget -> all 125 visited, best = argmin
    sp = Spec(16, 16, 16, 2, 2, 2)
    tg = ((1.0, 3.0), (2.0, 2.0), (3.0, 1.0))
    fn = lambda s: costs.t1_cost(s, targets=tg)
    res = gbfs.gbfs(sp, gbfs.fn_source(fn), rho=6, seed=4)
    assert res.evals == golden["completeness"]["visited"] == 125
    assert len({r.state for r in res.trace}) == 125
    assert res.best_cost == gbfs.brute_force(sp, fn)[0]


def test_gbfs_completeness_64_t2():
    sp = Spec(64, 64, 64)
    tab = costs.table(sp, lambda s: costs.t2_cost(sp, s))
    res = gbfs.gbfs(sp, gbfs.table_source(sp, tab), rho=26, seed=1)
    assert res.evals == 49392
    assert res.best_cost == min(tab)


def test_gbfs_invariants_and_determinism():
    sp = Spec(64, 64, 64)
    src = gbfs.fn_source(costs.t1_cost)
    a = gbfs.gbfs(sp, src, budget=300, rho=5, seed=7)
    b = gbfs.gbfs(sp, src, budget=300, rho=5, seed=7)
    assert [r.key() for r in a.trace] == [r.key() for r in b.trace]
    states = [r.state for r in a.trace]
    assert len(states) == len(set(states)) == 300
    bests = [r.best for r in a.trace]
    assert all(x >= y for x, y in zip(bests, bests[1:]))
    assert a.best_cost == min(r.cost for r in a.trace)
    c = gbfs.gbfs(sp, src, budget=300, rho=5, seed=8)
    assert [r.key() for r in c.trace] != [r.key() for r in a.trace]


def test_gbfs_queue_discipline(monkeypatch):
    # every popped state has (cost, seq) <= every key remaining in Q at pop time
    import heapq as hq
    sp = Spec(64, 64, 64)
    tab = costs.table(sp, lambda s: costs.t2_cost(sp, s))
    pops = []
    real_pop = hq.heappop

    def checked_pop(h):
        item = real_pop(h)
        assert all(item[:2] <= other[:2] for other in h)
        pops.append(item)
        return item

    monkeypatch.setattr(gbfs.heapq, "heappop", checked_pop)
    res = gbfs.gbfs(sp, gbfs.table_source(sp, tab), budget=200, rho=5, seed=3, width=2)
    assert len(pops) > 20 and res.evals == 200


def test_gbfs_efficiency_64_t1():
    # rho=5, budget 988 (2%), 10 seeds: within 5% of the optimum in >= 8/10
    sp = Spec(64, 64, 64)
    src = gbfs.fn_source(costs.t1_cost)
    ok = sum(1 for seed in range(10) if gbfs.gbfs(sp, src, budget=988, rho=5, seed=seed).best_cost <= 1.05)
    assert ok >= 8


def test_gbfs_width_budget_exact():
    sp = Spec(64, 64, 64)
    res = gbfs.gbfs(sp, gbfs.fn_source(costs.t1_cost), budget=97, rho=5, seed=2, width=8)
    assert res.evals == 97 and len(res.trace) == 97


def test_fraction_example(golden):
    ex = golden["fraction_example"]
    frac = ex["distinct"] / space.count_configs(Spec(ex["m"], ex["k"], ex["n"]))
    assert abs(frac - ex["frac_approx"]) < 1e-4


# ------------------------------------------------------------------ MLP
def test_mlp_zero_weights_and_softmax_symmetry():
    net = mlp.Mlp([10, 64, 64, 3])
    net.b[-1][:] = [0.5, -1.0, 2.0]
    out, _ = net.forward(np.ones((1, 10)))
    assert np.array_equal(out[0], [0.5, -1.0, 2.0])
    p = mlp.masked_softmax(np.zeros(26), np.ones(26, dtype=bool))
    assert np.allclose(p, 1.0 / 26) and abs(p.sum() - 1) < 1e-15
    mask = np.zeros(26, dtype=bool)
    mask[[0, 3, 5, 7, 11, 19, 25]] = True
    p = mlp.masked_softmax(np.full(26, 3.0), mask)
    assert np.allclose(p[mask], 1.0 / 7) and (p[~mask] == 0).all()
    z = np.random.default_rng(0).normal(size=26)
    assert np.allclose(mlp.masked_softmax(z, mask), mlp.masked_softmax(z + 5.0, mask))
    H = -float((p[mask] * np.log(p[mask])).sum())
    p26 = mlp.masked_softmax(np.zeros(26), np.ones(26, dtype=bool))
    assert abs(-float((p26 * np.log(p26)).sum()) - math.log(26)) < 1e-12
    assert abs(H - math.log(7)) < 1e-12


def test_mlp_finite_difference_gradient():
    # S:323 / S:537: central differences, h = 1e-5, max relative error <= 1e-4
    rng = SplitMix64(5)
    for sizes in ([10, 64, 64, 26], [10, 64, 64, 1]):
        net = mlp.Mlp(sizes, rng)
        X = np.random.default_rng(1).normal(size=(3, 10))
        W = np.random.default_rng(2).normal(size=(3, sizes[-1]))
        out, acts = net.forward(X)
        gW, gb = net.backward(acts, W)
        loss = lambda: float((net.forward(X)[0] * W).sum())
        worst = 0.0
        for l in range(len(net.W)):
            for (o, i) in [(0, 0), (min(1, sizes[l + 1] - 1), 2), (sizes[l + 1] - 1, sizes[l] - 1)]:
                old = net.W[l][o, i]
                net.W[l][o, i] = old + 1e-5
                lp = loss()
                net.W[l][o, i] = old - 1e-5
                lm = loss()
                net.W[l][o, i] = old
                fd = (lp - lm) / 2e-5
                worst = max(worst, abs(fd - gW[l][o, i]) / max(1e-8, abs(fd), abs(gW[l][o, i])))
            old = net.b[l][0]
            net.b[l][0] = old + 1e-5
            lp = loss()
            net.b[l][0] = old - 1e-5
            lm = loss()
            net.b[l][0] = old
            fd = (lp - lm) / 2e-5
            worst = max(worst, abs(fd - gb[l][0]) / max(1e-8, abs(fd), abs(gb[l][0])))
        assert worst <= 1e-4


def test_mlp_clip():
    net = mlp.Mlp([2, 3, 1], SplitMix64(1))
    gW = [np.full_like(w, 10.0) for w in net.W]
    gb = [np.full_like(b, 10.0) for b in net.b]
    W0 = [w.copy() for w in net.W]
    b0 = [b.copy() for b in net.b]
    net.sgd_step(gW, gb, lr=1.0, clip=1.0)
    step = math.sqrt(sum(((w - w0) ** 2).sum() for w, w0 in zip(net.W, W0)) +
                     sum(((b - b0_) ** 2).sum() for b, b0_ in zip(net.b, b0)))
    assert step <= 1.0 + 1e-12


def _np_forward(Ws, bs, X):
    """Plain forward pass written independently of oracle.mlp (numpy @, np.tanh)."""
    h = X
    for l, (W, b) in enumerate(zip(Ws, bs)):
        z = h @ W.T + b
        h = np.tanh(z) if l < len(Ws) - 1 else z
    return h


def _np_masked_log_softmax(z, mask):
    zm = np.where(mask, z, -np.inf)
    mx = zm.max()
    lse = mx + np.log(np.exp(zm[mask] - mx).sum())
    return np.where(mask, zm - lse, -np.inf)


def _train_memory(sp, ag):
    """A few predecessor transitions ("Store (s, a, r(s, a), s') to M") of two states."""
    mem = []
    for s2, r in ((((4, 4, 2, 2), (8, 8), (4, 4, 2, 2)), 1.7), (((2, 8, 2, 2), (16, 4), (8, 2, 2, 2)), 0.6)):
        for t, (pred, a) in enumerate(space.predecessors(sp, s2)[:3]):
            mem.append((pred, ag.acts.index(a), r * (1.0 + 0.25 * t), s2))
    return mem


@pytest.mark.parametrize("gamma,beta", [(0.9, 0.01), (0.0, 0.5), (0.9, 0.3)])
def test_agent_train_is_sgd_on_stated_losses(gamma, beta):
    """Pin of Agent.train (Alg. 2 line "Train actor's and critic's neural networks with M", P:327;
    A2C, P:284 / S:400-406): one epoch with lr = 1 and clipping off must move every parameter by
    minus the gradient of the stated losses over the drawn minibatch, computed here by central
    finite differences with an independent numpy forward pass:
        critic  L_c = mean_b (r_b + gamma V0(s'_b) - V(s_b))^2          (V0 = critic before the step)
        actor   L_a = mean_b [-A_b log pi(a_b | s_b) - beta H(pi(. | s_b))],  A_b = r_b + gamma V0(s'_b) - V0(s_b)
    with pi the softmax over the legitimate actions of s_b.  A flipped entropy sign, a dropped
    factor 2 in dL_c/dV, or a wrong advantage fails this test."""
    sp = Spec(64, 64, 64)
    p = na2c.Params(gamma=gamma, beta=beta, lr=1.0, clip=0.0, epochs=1, minibatch=6, hidden=8)
    rng_nn = SplitMix64(21)
    ag = na2c.Agent(sp, p, rng_nn)
    mem = _train_memory(sp, ag)
    probe = SplitMix64(0)
    probe.state = rng_nn.state                       # the same minibatch draws as train's
    mb = [mem[probe.bounded(len(mem))] for _ in range(p.minibatch)]
    Xs = np.array([space.features(sp, t[0]) for t in mb])
    X2 = np.array([space.features(sp, t[3]) for t in mb])
    r = np.array([t[2] for t in mb])
    acts = [t[1] for t in mb]
    masks = [ag.legal_mask(t[0]) for t in mb]
    Wc0, bc0 = [w.copy() for w in ag.critic.W], [b.copy() for b in ag.critic.b]
    Wa0, ba0 = [w.copy() for w in ag.actor.W], [b.copy() for b in ag.actor.b]
    V0s = _np_forward(Wc0, bc0, Xs)[:, 0]
    V0n = _np_forward(Wc0, bc0, X2)[:, 0]
    target = r + gamma * V0n
    adv = target - V0s

    def loss_c(Ws, bs):
        return float(np.mean((target - _np_forward(Ws, bs, Xs)[:, 0]) ** 2))

    def loss_a(Ws, bs):
        Z = _np_forward(Ws, bs, Xs)
        tot = 0.0
        for b in range(len(mb)):
            lp = _np_masked_log_softmax(Z[b], masks[b])
            pi = np.exp(lp[masks[b]])
            H = -float((pi * lp[masks[b]]).sum())
            tot += -adv[b] * lp[acts[b]] - beta * H
        return tot / len(mb)

    ag.train(mem, rng_nn)

    def check(W0, b0, W1, b1, loss):
        worst, gmax = 0.0, 0.0
        for params0, params1 in ((W0, W1), (b0, b1)):
            for l in range(len(params0)):
                g_train = params0[l] - params1[l]              # = lr * grad with lr = 1
                for idx in np.ndindex(params0[l].shape):
                    Wp = [w.copy() for w in W0]
                    bp = [b.copy() for b in b0]
                    tgt = (Wp if params0 is W0 else bp)[l]
                    h = 1e-6
                    tgt[idx] += h
                    lp_ = loss(Wp, bp)
                    tgt[idx] -= 2 * h
                    lm_ = loss(Wp, bp)
                    fd = (lp_ - lm_) / (2 * h)
                    worst = max(worst, abs(fd - g_train[idx]))
                    gmax = max(gmax, abs(fd))
        return worst, gmax

    wc, gc = check(Wc0, bc0, ag.critic.W, ag.critic.b, loss_c)
    wa, ga = check(Wa0, ba0, ag.actor.W, ag.actor.b, loss_a)
    assert gc > 1e-3 and ga > 1e-3                                  # non-trivial gradients
    assert wc <= 1e-7 + 1e-6 * gc, (wc, gc)
    assert wa <= 1e-7 + 1e-6 * ga, (wa, ga)


def test_advantage_gamma0_zero_critic():
    # gamma = 0 and V == 0 -> A = r, so the actor step is the REINFORCE step on r.
    # Through Agent.train: a zero critic stays zero-output only through its bias, so compare the
    # actor update against the same train with gamma = 0.9 (V(s') = 0 makes gamma irrelevant).
    sp = Spec(64, 64, 64)
    outs = []
    for g in (0.0, 0.9):
        p = na2c.Params(gamma=g, lr=0.5, clip=0.0, epochs=1, minibatch=4, hidden=8)
        rng = SplitMix64(3)
        ag = na2c.Agent(sp, p, rng)
        for w in ag.critic.W + ag.critic.b:
            w[...] = 0.0
        ag.train(_train_memory(sp, ag), rng)
        outs.append([w.copy() for w in ag.actor.W])
    assert all(np.array_equal(a, b) for a, b in zip(*outs))


# ------------------------------------------------------------------ N-A2C (Alg. 2)
def test_na2c_eps0_properties():
    sp = Spec(64, 64, 64)
    p = na2c.Params(epsilon=0.0, batch=7, steps=1)
    res = na2c.na2c(sp, gbfs.fn_source(costs.t1_cost), budget=8, params=p, seed=3)
    # one episode from s0 with T=1 collects only neighbours of s0
    g0 = set(space.neighbors(sp, space.initial_state(sp)))
    assert all(r.state in g0 for r in res.trace[1:])


def test_na2c_invariants():
    sp = Spec(64, 64, 64)
    for eps in (0.0, 0.8):
        p = na2c.Params(epsilon=eps)
        res = na2c.na2c(sp, gbfs.fn_source(costs.t1_cost), budget=200, params=p, seed=1)
        states = [r.state for r in res.trace]
        assert len(states) == len(set(states)) == res.evals == 200
        bests = [r.best for r in res.trace]
        assert all(x >= y for x, y in zip(bests, bests[1:]))
        again = na2c.na2c(sp, gbfs.fn_source(costs.t1_cost), budget=200, params=p, seed=1)
        assert [r.key() for r in again.trace] == [r.key() for r in res.trace]


def test_na2c_locality():
    # every collected state is within T steps of the episode's start state.  With T=3 and
    # batch 1, each episode's start is the incumbent before that batch.
    sp = Spec(64, 64, 64)
    p = na2c.Params(epsilon=0.0, batch=1, steps=3)
    res = na2c.na2c(sp, gbfs.fn_source(costs.t1_cost), budget=60, params=p, seed=9)
    start = res.trace[0].state
    best = res.trace[0].cost
    for r in res.trace[1:]:
        # BFS distance from start <= 3
        frontier, seen = {start}, {start}
        for _ in range(3):
            frontier = {t for s in frontier for t in space.neighbors(sp, s)} - seen
            seen |= frontier
        assert r.state in seen
        if r.cost < best:
            best, start = r.cost, r.state


def _na2c_vs_random(seed):
    sp = Spec(64, 64, 64)
    allst = list(space.enumerate_configs(sp))
    a = na2c.na2c(sp, gbfs.fn_source(costs.t1_cost), budget=988, seed=seed).best_cost
    pick = SplitMix64(1000 + seed).sample_indices(len(allst), 988)
    return a, min(costs.t1_cost(allst[i]) for i in pick)


def test_na2c_beats_random_search():
    # 64^3 T1 preset, budget 988, 10 paired seeds: N-A2C median <= random median and
    # paired wins (<=) in >= 7/10 (seeds run in parallel processes: the oracle is pure Python)
    import multiprocessing as mproc
    with mproc.get_context("spawn").Pool(min(10, os.cpu_count() or 1)) as pool:
        pairs = pool.map(_na2c_vs_random, range(10))
    nres = [a for a, _ in pairs]
    rres = [b for _, b in pairs]
    wins = sum(a <= b for a, b in pairs)
    assert statistics.median(nres) <= statistics.median(rres)
    assert wins >= 7


# ------------------------------------------------------------------ measurement aggregation
def test_aggregate_fake_clock():
    # injected trial durations
    xs = [1.0, 2.0, 3.0, 4.0, 100.0, 5.0, 6.0, 7.0, 8.0, 9.0]
    a = measure.aggregate(xs)
    assert a["mean"] == sum(xs) / 10                       # paper's statistic
    assert a["cost"] == 5.5                                # median of 10 (reading Z10)
    assert a["min"] == 1.0 and a["repeats"] == 10
    assert abs(a["stdev"] - statistics.stdev(xs)) < 1e-12
    assert measure.aggregate([2.5])["stdev"] == 0.0
    assert measure.aggregate([3.0, 1.0, 2.0])["cost"] == 2.0
    assert measure.number_for(100e-6, 500e-6) == 5 and measure.number_for(1.0, 500e-6) == 1
    assert measure.is_slow(0.2, 0.05) and not measure.is_slow(0.01, 0.05)
