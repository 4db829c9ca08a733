"""N-A2C, Algorithm 2 of the paper (oracle; test infra only).

PAPER.md Sec. "N-A2C Method", Algorithm 2:

  1  Initialization: s0, M, H_v, cost_min
  2  for each episode:
  3      while len(B_collect) < len(B_test):
  4          s = s0
  5          for each step until T steps:
  6              if rand() < eps:  a follows pi(s)      else:  a is randomly selected from A
  11             s' = step(s, a)
  12             if s' not in H_v:  Add s' in B_collect
  14             s = s'
  17     for s' in B_collect:
  18         if cost_min > cost(s'):  cost_min = cost(s');  s* = s';  s0 = s*
  22         H_v[s'] = cost(s')
  23         Store (s, a, r(s,a), s') to M, for all s, all a satisfying step(s,a) = s'
  24         Train actor's and critic's neural networks with M
  26 Return s*, cost_min

eps is the *exploitation* probability ("with probability of eps, the agent takes action
a guided by the policy").  Readings (Z18):
  * s0 is measured first and enters H_v; cost_min = cost(s0), s* = s0.
  * an illegitimate step result leaves the agent in place; a state already in
    B_collect is not added twice; whole rollouts run (the while test is between rollouts).
  * at most ``50*batch`` rollouts per collection; if B_collect is still empty, T is
    increased by 1 for this episode ("T can also increase to explore new configuration
    neighborhoods"); after 16 increases the neighbourhood is exhausted and the search stops.
  * B_collect is truncated to budget - evals, measured as one batch, walked in order.
  * reward r = c_ref / cost(s'), c_ref = cost(initial s0): a positive rescale of Eq. 8's 1/cost.
  * M is a FIFO of capacity ``mem_capacity`` holding every predecessor transition.
  * training once per batch (``train_per_candidate=True``: after every candidate, Alg. 2's own
    placement of line 24 inside the line-17 loop): ``epochs`` SGD steps, each on ``minibatch`` transitions drawn
    with replacement via bounded(len(M)) from the network stream.  A = r + gamma V(s') - V(s)
    (V(s') a constant target); critic loss A^2; actor loss -A log pi(a|s) - beta H(pi(.|s)).
  * two SplitMix64 streams: exploration ``seed`` (eps draw, then the action draw), and network
    init + minibatch sampling ``seed ^ 0xA2C0A2C0A2C0A2C0``.
  * policy sampling: u = uniform(); first legitimate action (action order) whose cumulative
    probability exceeds u, else the last legitimate one.
With eps = 0 the policy is never consulted, so the trajectory depends only on the RNG and the
cost source.  With eps > 0 the trajectory also depends on the networks; their arithmetic is
written with every sum left-to-right in index order and C-library tanh / exp / log (mlp.py,
reading Z24), so the whole trajectory is still a fixed function of (seed, costs) and the
library is compared bit for bit in both modes.
"""
from __future__ import annotations

import math
import time
from collections import deque
from typing import Callable, List, Optional

import numpy as np

from . import space
from .gbfs import Result, TraceRow
from .mlp import Mlp, masked_softmax
from .rng import SplitMix64

NN_STREAM_XOR = 0xA2C0A2C0A2C0A2C0


class Params:
    def __init__(self, steps=3, epsilon=0.8, batch=16, mem_capacity=4096, gamma=0.9, beta=0.01,
                 lr=0.01, clip=1.0, epochs=4, minibatch=64, hidden=64, rollout_cap_factor=50,
                 max_t_increase=16, steps_floor=1, decay_every=0, train_per_candidate=False):
        self.steps, self.epsilon, self.batch = steps, epsilon, batch
        self.mem_capacity, self.gamma, self.beta, self.lr, self.clip = mem_capacity, gamma, beta, lr, clip
        self.epochs, self.minibatch, self.hidden = epochs, minibatch, hidden
        self.rollout_cap_factor, self.max_t_increase = rollout_cap_factor, max_t_increase
        # P:336 "the exploration step T can have a decay process": T_e = max(floor, T0 - e // every)
        self.steps_floor, self.decay_every = steps_floor, decay_every
        # Alg. 2 places "Train actor's and critic's neural networks with M" inside the
        # "for s' in B_collect" loop: True trains after every candidate, in that order;
        # False (default, reading Z18 / S:422) trains once after the batch.
        self.train_per_candidate = train_per_candidate


class Agent:
    def __init__(self, spec: space.Spec, p: Params, rng_nn: SplitMix64):
        self.spec, self.p = spec, p
        self.acts = space.actions(spec)
        nin = spec.dm + spec.dk + spec.dn
        self.actor = Mlp([nin, p.hidden, p.hidden, len(self.acts)], rng_nn)
        self.critic = Mlp([nin, p.hidden, p.hidden, 1], rng_nn)

    def legal_mask(self, s) -> np.ndarray:
        """Which actions lead to a legitimate state (a pure function of s, memoised)."""
        cache = self.__dict__.setdefault("_mask_cache", {})
        if s in cache:
            return cache[s]
        m = np.zeros(len(self.acts), dtype=bool)
        for i, a in enumerate(self.acts):
            t = space.step(s, a)
            m[i] = t is not None and space.legitimate(self.spec, t)
        cache[s] = m
        return m

    def policy(self, s) -> np.ndarray:
        x = np.array([space.features(self.spec, s)])
        z, _ = self.actor.forward(x)
        return masked_softmax(z[0], self.legal_mask(s))

    def train(self, memory, rng_nn: SplitMix64):
        p = self.p
        n = len(memory)
        if n == 0:
            return
        for _ in range(p.epochs):
            mb = [memory[rng_nn.bounded(n)] for _ in range(p.minibatch)]
            Xs = np.array([space.features(self.spec, t[0]) for t in mb])
            X2 = np.array([space.features(self.spec, t[3]) for t in mb])
            r = np.array([t[2] for t in mb])
            aidx = np.array([t[1] for t in mb])
            masks = np.array([self.legal_mask(t[0]) for t in mb])
            B = len(mb)
            v, acts_c = self.critic.forward(Xs)
            v2, _ = self.critic.forward(X2)
            adv = r + p.gamma * v2[:, 0] - v[:, 0]
            # critic: mean A^2, dL/dV(s) = -2A / B
            gWc, gbc = self.critic.backward(acts_c, (-2.0 * adv / B)[:, None])
            # actor: mean(-A log pi_a - beta H)
            z, acts_a = self.actor.forward(Xs)
            dz = np.zeros_like(z)
            for b in range(B):
                pi = masked_softmax(z[b], masks[b])
                H = 0.0                                             # entropy, left-to-right
                for i in range(len(pi)):
                    if masks[b][i] and pi[i] > 0:
                        H -= pi[i] * math.log(pi[i])
                for i in range(len(pi)):
                    if not masks[b][i]:
                        continue
                    lp = math.log(pi[i]) if pi[i] > 0 else 0.0
                    g = adv[b] * pi[i]                              # d(-A log pi_a)/dz_i = A (pi_i - [i = a])
                    if i == aidx[b]:
                        g -= adv[b]
                    g += p.beta * pi[i] * (lp + H)                  # d(-beta H)/dz_i
                    dz[b, i] = g / B
            gWa, gba = self.actor.backward(acts_a, dz)
            self.critic.sgd_step(gWc, gbc, p.lr, p.clip)
            self.actor.sgd_step(gWa, gba, p.lr, p.clip)


def na2c(spec: space.Spec,
         cost_batch: Callable[[List[space.State]], List[float]],
         budget: int,
         params: Optional[Params] = None,
         seed: int = 0,
         s0=None,
         t_max: Optional[float] = None) -> Result:
    p = params or Params()
    if s0 is None:
        from .hw import default_s0
        s0 = default_s0(spec)
    if not space.legitimate(spec, s0):
        raise ValueError("s0 is not legitimate (S:256)")
    rng = SplitMix64(seed)
    rng_nn = SplitMix64(seed ^ NN_STREAM_XOR)
    agent = Agent(spec, p, rng_nn)
    acts = agent.acts
    t0 = time.perf_counter()

    c0 = cost_batch([s0])[0]
    H = {s0: c0}
    evals = 1
    best_cost, best_state = c0, s0
    c_ref = c0
    start = s0
    memory = deque(maxlen=p.mem_capacity)
    trace = [TraceRow(0, time.perf_counter() - t0, s0, c0, best_cost)]
    cap = p.rollout_cap_factor * p.batch
    episode = 0

    while evals < budget:
        if t_max is not None and time.perf_counter() - t0 >= t_max:
            break
        T_e = max(p.steps_floor, p.steps - episode // p.decay_every) if p.decay_every > 0 else p.steps
        episode += 1
        T = T_e
        coll: List[space.State] = []
        cset = set()
        exhausted = False
        while True:
            rollouts = 0
            while len(coll) < p.batch and rollouts < cap:          # line 3
                rollouts += 1
                s = start                                           # line 4
                for _ in range(T):                                  # line 5
                    u = rng.uniform()
                    a = None
                    if u < p.epsilon:                               # line 6: follow pi(s)
                        pi = agent.policy(s)
                        if pi.sum() > 0:
                            u2 = rng.uniform()
                            cum = 0.0
                            last = None
                            for i in range(len(acts)):
                                if pi[i] > 0:
                                    last = i
                                    cum += pi[i]
                                    if u2 < cum:
                                        a = i
                                        break
                            if a is None:
                                a = last
                    if a is None:                                   # random a in A
                        a = rng.bounded(len(acts))
                    s2 = space.step(s, acts[a])                     # line 11
                    if s2 is None or not space.legitimate(spec, s2):
                        s2 = s                                      # stay in place
                    if s2 not in H and s2 not in cset:              # line 12
                        coll.append(s2)
                        cset.add(s2)
                    s = s2                                          # line 14
            if coll:
                break
            T += 1
            if T > T_e + p.max_t_increase:
                exhausted = True
                break
        if exhausted:
            break
        coll = coll[:budget - evals]
        costs = cost_batch(coll)
        for s2, c in zip(coll, costs):                              # line 17
            if c < best_cost:                                       # lines 18-21
                best_cost, best_state = c, s2
                start = s2
            H[s2] = c                                               # line 22
            r = c_ref / c if c > 0 else 0.0
            for (pred, a) in space.predecessors(spec, s2):          # line 23
                memory.append((pred, acts.index(a), r, s2))
            trace.append(TraceRow(evals, time.perf_counter() - t0, s2, c, best_cost))
            evals += 1
            if p.train_per_candidate:
                agent.train(memory, rng_nn)                         # line 24, inside the loop
        if not p.train_per_candidate:
            agent.train(memory, rng_nn)                             # line 24, once per batch (Z18)
    return Result(best_state, best_cost, evals, trace, space.count_configs(spec), None)
