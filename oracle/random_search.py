"""Random-search comparator (oracle; test infra only).

PAPER.md P:64: in random search "configurations are randomly selected to be tested"; SPEC S:475-483:
sample legitimate states uniformly without replacement via index sampling over the enumeration
order.  Reading: the feasible states (J_prod and J_hw) in rank order are permuted
by a partial Fisher-Yates shuffle with SplitMix64(seed) (oracle.rng) and the first `budget` are
measured, in batches of `width`, in draw order; strict '<' keeps the earliest best.
"""
from __future__ import annotations

import math
import time

from . import space
from .gbfs import Result, TraceRow
from .rng import SplitMix64


def random_search(spec: space.Spec, cost_batch, budget: int, seed: int = 0, width: int = 1) -> Result:
    feas = [s for s in space.enumerate_configs(spec) if space.legitimate(spec, s)]
    L = len(feas)
    budget = L if (budget is None or budget <= 0 or budget > L) else budget
    order = SplitMix64(seed).sample_indices(L, budget)
    t0 = time.perf_counter()
    best_cost, best_state = math.inf, None
    trace = []
    evals = 0
    while evals < budget:
        batch = [feas[i] for i in order[evals:evals + width]]
        for s, c in zip(batch, cost_batch(batch)):
            if c < best_cost:
                best_cost, best_state = c, s
            trace.append(TraceRow(evals, time.perf_counter() - t0, s, c, best_cost))
            evals += 1
    return Result(best_state, best_cost, evals, trace, space.count_configs(spec), L)
