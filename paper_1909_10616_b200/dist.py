"""Multi-GPU plumbing (B6): one process per GPU, torch.distributed for the exchange.

Two partitions of the hot path:

1. Candidate-batch sharding for the searches.  Every rank runs the identical search (same
   seed, same code, replicated state); a round's candidates are independent measurements, so
   each is measured on exactly one rank and the costs are exchanged.  The traversal depends only
   on (seed, W, rho, cost values), never on G or on which rank measured what.
2. Row-partitioned large GEMM: rank r owns rows [r M/G, (r+1) M/G) of A and C, B is
   replicated, and there is no collective on the math path (``row_shard``).

torch is used for the process group and the tiny timing tensors only; every measurement is a
libtiletune call (``tt_measure_set``: the per-rank half of a round runs in C++, one call per round).
"""
from __future__ import annotations

import itertools
import math
import time
from typing import Callable, List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist

from . import tiletune as tt

# measurement-time model of one candidate for the LPT assignment: a candidate scored by its
# probe costs one launch, a full one ~11 (cold probe, 10 repeats), plus host overhead
_FULL_LAUNCHES = 11
_PER_CANDIDATE_S = 2e-3


class ShardedEvaluator:
    """BATCH cost source for tt.gbfs_search / tt.na2c_search / tt.random_search.

    ``measure_set(states, mine) -> (costs, seconds)`` scores the states whose ``mine`` flag is
    set on this rank (normally ``device_measure_set``: one tt_measure_set call, C++ loop) and
    returns 0 elsewhere.  For host-side tests ``measure_one(state) -> cost`` is accepted instead.

    Assignment of a round's candidates to ranks (``assign``):

    * ``"lpt"`` (default): longest predicted measurement first, each to the least-loaded rank.
      The prediction of a candidate is the lowest known cost among its measured neighbours (a
      neighbour differs by one x2 / /2 move), turned into a measurement time by the
      scoring rules (one launch above the cut, ~11 below).  Every rank holds the same known
      costs, so every rank computes the same assignment with no communication.
    * ``"static"``: candidate j on rank j mod G.
    * ``"dynamic"`` (``store`` given): ranks claim the next unmeasured index from a shared
      counter (``store.add``) whenever they are free.

    Costs are exchanged with one all_reduce(MAX) of an [n] float64 vector whose entries only the
    measuring rank filled (every cost is > 0), so each candidate is measured exactly once and the
    costs come back by index.
    """

    _instances = itertools.count()     # per-process: identical on every rank that builds evaluators in order

    def __init__(self, measure_one: Optional[Callable] = None, group=None, device: Optional[torch.device] = None,
                 store=None, measure_set: Optional[Callable] = None, assign: Optional[str] = None,
                 space: Optional[tt.Space] = None, cut_s: Optional[Callable[[], float]] = None):
        if measure_set is None:
            if measure_one is None:
                raise ValueError("need measure_one or measure_set")

            def measure_set(states, mine):
                costs, secs = [0.0] * len(states), [0.0] * len(states)
                for j, (s, m) in enumerate(zip(states, mine)):
                    if m:
                        t0 = time.perf_counter()
                        costs[j] = float(measure_one(s))
                        secs[j] = time.perf_counter() - t0
                return costs, secs
        self.measure_set = measure_set
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.device = device or torch.device("cpu")
        self.store = store if self.world > 1 else None
        self.assign = "dynamic" if self.store is not None else (assign or "lpt")
        if self.assign == "dynamic" and self.store is None and self.world > 1:
            raise ValueError("dynamic assignment needs a store")
        self.space = space
        self.cut_s = cut_s
        self.ns = f"tt_eval{next(ShardedEvaluator._instances)}"
        self.rounds = 0
        self.local_evals = 0
        self.known: dict = {}
        self._nb_cache: dict = {}
        # per round: (measurement seconds of every candidate on the rank that measured it -- the
        # values are exchanged with the costs --, predicted weights used by the LPT assignment)
        self.round_times: List[List[float]] = []
        self.round_weights: List[List[float]] = []

    # ------------------------------------------------------------------ assignment
    def _neighbors(self, s):
        nb = self._nb_cache.get(s)
        if nb is None:
            nb = self._nb_cache[s] = tt.neighbors(self.space, s)
        return nb

    def _predicted_cost(self, s) -> float:
        best = math.inf
        if self.space is not None:
            for t in self._neighbors(s):
                c = self.known.get(t)
                if c is not None and c < best:
                    best = c
        if not math.isfinite(best):
            best = min(self.known.values()) if self.known else 1.0
        return best

    def weights(self, states) -> List[float]:
        cut = self.cut_s() if self.cut_s is not None else 0.0
        w = []
        for s in states:
            c = self._predicted_cost(s)
            w.append((c if (cut > 0 and c > cut) else _FULL_LAUNCHES * c) + _PER_CANDIDATE_S)
        return w

    @staticmethod
    def lpt_owners(weights: Sequence[float], world: int) -> List[int]:
        """Longest-processing-time-first list scheduling: candidates in decreasing weight (ties by
        index) go to the least-loaded rank (ties: lowest rank).  Deterministic."""
        owner = [0] * len(weights)
        load = [0.0] * world
        for j in sorted(range(len(weights)), key=lambda j: (-weights[j], j)):
            r = min(range(world), key=lambda i: (load[i], i))
            owner[j] = r
            load[r] += weights[j]
        return owner

    # ------------------------------------------------------------------ one round
    def __call__(self, states: Sequence) -> List[float]:
        n = len(states)
        wts = self.weights(states) if self.assign == "lpt" else [1.0] * n
        vals = [0.0] * (2 * n)                                                # costs, then seconds
        if self.assign == "dynamic":
            key = f"{self.ns}_round{self.rounds}"
            while True:
                j = int(self.store.add(key, 1)) - 1
                if j >= n:
                    break
                mine = [i == j for i in range(n)]
                c, t = self.measure_set(states, mine)
                vals[j], vals[n + j] = c[j], t[j]
                self.local_evals += 1
        else:
            owner = self.lpt_owners(wts, self.world) if self.assign == "lpt" else [j % self.world for j in range(n)]
            mine = [o == self.rank for o in owner]
            c, t = self.measure_set(states, mine)
            for j in range(n):
                if mine[j]:
                    vals[j], vals[n + j] = c[j], t[j]
                    self.local_evals += 1
        if self.world > 1:
            buf = torch.tensor(vals, dtype=torch.float64, device=self.device)
            dist.all_reduce(buf, op=dist.ReduceOp.MAX, group=self.group)
            vals = buf.cpu().tolist()
            if self.assign == "dynamic" and self.rank == 0:
                try:                                     # every rank has left its claim loop
                    self.store.delete_key(f"{self.ns}_round{self.rounds}")
                except Exception:  # noqa: BLE001 - older stores: keys are namespaced anyway
                    pass
        out = vals
        costs = out[:n]
        if not all(c > 0 for c in costs):
            raise RuntimeError(f"sharded round {self.rounds}: a candidate came back unmeasured ({costs})")
        self.round_times.append(out[n:])
        self.round_weights.append(wts)
        self.rounds += 1
        for s, c in zip(states, costs):
            self.known[s] = c
        return costs


def default_store():
    """The default process group's TCPStore (for dynamic assignment), or None."""
    try:
        from torch.distributed import distributed_c10d as c10d
        return c10d._get_default_store()
    except Exception:  # noqa: BLE001 - private API moved: fall back to the static assignment
        return None


def device_measure_set(ctx: tt.Context, sp: tt.Space, opts: tt.SearchOpts, device: int = -1):
    """measure_set for ShardedEvaluator on the device: one tt_measure_set call per round with the
    search's scoring options (tt_scoring_opts: slow-candidate cut and racing, reading Z12) at the
    incumbent -- identical on every rank, because it is the minimum of the exchanged costs.
    Returns (measure_set, observe, cut_s) where observe(costs) updates the incumbent and cut_s()
    is the current cut (for the LPT weights)."""
    state = {"best": math.inf}

    def mo():
        return tt.scoring_opts(sp, opts, state["best"], device)

    def measure_set(states, mine):
        return ctx.measure_set(sp, states, mine, mo())

    def observe(costs):
        for c in costs:
            state["best"] = min(state["best"], c)

    return measure_set, observe, lambda: mo().cut_s


def projected_sharded_wall(round_times: Sequence[Sequence[float]], world: int, per_round_s: float = 0.0,
                           dynamic: bool = False, per_claim_s: float = 0.0,
                           weights: Optional[Sequence[Sequence[float]]] = None) -> float:
    """Measurement wall time of the same traversal sharded over ``world`` ranks, from
    per-candidate times recorded on one rank: sum over rounds of the slowest rank's busy time,
    plus ``per_round_s`` (the collective) per round.  Static: candidate j on rank j mod world.
    ``weights`` given: the LPT assignment the evaluator makes from those predicted weights.
    Dynamic: candidates in index order each go to the rank that becomes free first (what the
    counter-claiming evaluator does), each claim costing ``per_claim_s``.  A projection from
    measured times, not a multi-GPU measurement."""
    total = 0.0
    for k, times in enumerate(round_times):
        busy = [0.0] * world
        if weights is not None:
            owner = ShardedEvaluator.lpt_owners(weights[k], world)
        for j, t in enumerate(times):
            if weights is not None:
                r = owner[j]
            else:
                r = min(range(world), key=lambda i: busy[i]) if dynamic else j % world
            busy[r] += t + (per_claim_s if dynamic else 0.0)
        total += max(busy) + (per_round_s if world > 1 else 0.0)
    return total


class TrackingEvaluator(ShardedEvaluator):
    """ShardedEvaluator that feeds the exchanged costs back into the scoring tracker."""

    def __init__(self, measure_one=None, observe=None, **kw):
        super().__init__(measure_one, **kw)
        self.observe = observe

    def __call__(self, states):
        costs = super().__call__(states)
        if self.observe is not None:
            self.observe(costs)
        return costs


def row_shard(M: int, world: int, rank: int) -> Tuple[int, int]:
    """Rows [r0, r1) of the row-partitioned GEMM owned by ``rank`` (exact: M % world == 0)."""
    if M % world:
        raise ValueError("row partition needs M divisible by the number of ranks")
    per = M // world
    return rank * per, (rank + 1) * per


def max_over_ranks(x: float, device=None) -> float:
    """Max of a host float over ranks (timings are reported as the max over ranks)."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device or torch.device("cpu"))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
