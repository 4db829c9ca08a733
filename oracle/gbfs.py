"""G-BFS, Algorithm 1 of the paper (oracle; test infra only).

PAPER.md Sec. "G-BFS Method", Algorithm 1:

  1  Initialization: Q = PriorityQueue(), S_v, s0
  2  Q.push((cost(s0), s0))
  3  Add s0 in S_v
  4  while Q != {} and t_search < T_max:
  5      (cost(s), s) = Q.pop()
  6      B = Take rho neighbors randomly from g(s)
  7      for s' in B:
  8          if s' is legitimate and s' not in S_v:
  9              Q.push((cost(s'), s'));  10  Add s' in S_v
  11             if cost_min > cost(s'):  12 cost_min = cost(s');  13  s* = s'
  16 Return s*, cost_min

Readings:
  Z4  g(s) holds legitimate results only (J = J_prod and J_hw), in action order.
  Z5  rho samples uniformly without replacement (oracle.rng.sample_indices); all if |g| < rho.
  Z6  queue key (cost, insertion sequence) -> FIFO among equal costs.
  Z7  s* = s0, cost_min = cost(s0) initially; strict '<' keeps the earliest of equal costs.
  Z8  ``budget`` = max number of distinct states measured, s0 included, checked before each
      measurement; ``t_max`` (seconds) is checked once per round at the while test.
  Z9  ``width`` W pops per round ("explore from the rho most promising red nodes");
      W = 1 is exactly Algorithm 1.  With W = 1 the candidates of one expansion are tested
      in sample order; their costs never change which of them are tested.
A round's candidates are the concatenation of each popped state's sample, dropping states in
S_v and repeats within the round (first occurrence wins); already-visited draws still consume
a rho slot.  Candidates are then truncated to budget - evals, added to S_v, measured
as one batch (any partition over GPUs is allowed), and pushed in candidate order.
"""
from __future__ import annotations

import heapq
import math
import time
from typing import Callable, List, Optional

from . import space
from .rng import SplitMix64


class TraceRow:
    __slots__ = ("eval_index", "t_wall", "state", "cost", "best")

    def __init__(self, eval_index, t_wall, state, cost, best):
        self.eval_index, self.t_wall, self.state, self.cost, self.best = eval_index, t_wall, state, cost, best

    def key(self):
        return (self.eval_index, self.state, self.cost, self.best)


class Result:
    def __init__(self, best_state, best_cost, evals, trace, space_raw, space_feasible):
        self.best_state, self.best_cost, self.evals, self.trace = best_state, best_cost, evals, trace
        self.space_raw, self.space_feasible = space_raw, space_feasible

    @property
    def frac_raw(self):
        return self.evals / self.space_raw


def gbfs(spec: space.Spec,
         cost_batch: Callable[[List[space.State]], List[float]],
         budget: Optional[int] = None,
         rho: int = 5,
         seed: int = 0,
         s0: Optional[space.State] = None,
         width: int = 1,
         t_max: Optional[float] = None) -> Result:
    if s0 is None:
        from .hw import default_s0
        s0 = default_s0(spec)
    if not space.legitimate(spec, s0):
        raise ValueError("s0 is not legitimate (S:256)")
    if budget is None:
        budget = math.inf
    rng = SplitMix64(seed)
    t0 = time.perf_counter()

    c0 = cost_batch([s0])[0]                              # line 2: test s0
    evals = 1
    seq = 0
    queue = [(c0, seq, s0)]                               # line 2
    visited = {s0}                                        # line 3
    best_cost, best_state = c0, s0                        # reading Z7
    trace = [TraceRow(0, time.perf_counter() - t0, s0, c0, best_cost)]

    while queue and evals < budget:                       # line 4 (+ eval budget, Z8)
        if t_max is not None and time.perf_counter() - t0 >= t_max:
            break
        popped = [heapq.heappop(queue)[2] for _ in range(min(width, len(queue)))]   # line 5
        cands: List[space.State] = []
        round_set = set()
        for s in popped:
            g = space.neighbors(spec, s)                  # Eq. 9 (Z4: legitimate only)
            for idx in rng.sample_indices(len(g), rho):   # line 6 (Z5)
                s2 = g[idx]
                if s2 in visited or s2 in round_set:      # line 8
                    continue
                cands.append(s2)
                round_set.add(s2)
        remaining = budget - evals
        if len(cands) > remaining:
            cands = cands[:int(remaining)]
        if not cands:
            continue
        visited.update(cands)                             # line 10
        costs = cost_batch(cands)                         # "test them in hardware"
        for s2, c in zip(cands, costs):
            seq += 1
            heapq.heappush(queue, (c, seq, s2))           # line 9
            if c < best_cost:                             # lines 11-13, strict (Z7)
                best_cost, best_state = c, s2
            trace.append(TraceRow(evals, time.perf_counter() - t0, s2, c, best_cost))
            evals += 1
    raw = space.count_configs(spec)
    return Result(best_state, best_cost, evals, trace, raw, None)


def table_source(spec: space.Spec, table: List[float]):
    """cost_batch over a rank-indexed table (the TABLE cost source / replay of a device trace)."""
    def f(states):
        return [table[space.rank(spec, s)] for s in states]
    return f


def fn_source(fn):
    def f(states):
        return [fn(s) for s in states]
    return f


def brute_force(spec: space.Spec, fn) -> tuple:
    """Grid search: argmin over every legitimate state; ties -> lowest rank."""
    best = (math.inf, None)
    for s in space.enumerate_configs(spec):
        if not space.legitimate(spec, s):
            continue
        c = fn(s)
        if c < best[0]:
            best = (c, s)
    return best
