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
# one dynamic claim (a TCPStore add round trip); "auto" claims dynamically only in rounds whose
# median predicted measurement time is >= _AUTO_CLAIMS claims, else it uses the LPT plan
_CLAIM_S = 200e-6
_AUTO_CLAIMS = 10


def auto_mode(weights: Sequence[float]) -> str:
    """The "auto" rule for one round (identical on every rank: the weights come from the
    replicated known costs): dynamic claiming when the median predicted measurement time is at
    least _AUTO_CLAIMS claim round trips, else the LPT plan (no per-candidate store traffic)."""
    raw = sorted(w - _PER_CANDIDATE_S for w in weights)
    med = raw[len(raw) // 2] if raw else 0.0
    return "dynamic" if med >= _AUTO_CLAIMS * _CLAIM_S else "lpt"


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
    * ``"dynamic"`` (``store`` given): ranks claim the next unmeasured candidate, in the LPT
      order of the predictions, from a shared counter (``store.add``) whenever they are free.
    * ``"auto"`` (``store`` given): per round, dynamic when the median predicted measurement time
      is at least 10 claim round trips (~2 ms), else the LPT plan -- short candidates (bf16 at
      4096^3, ~1 ms each) do not pay a store round trip apiece, long ones (fp32) balance
      dynamically.

    Speculation (``speculate``, needs ``space``): in round 0 -- s0 alone, so G - 1 ranks would
    idle -- the idle ranks measure s0's neighbourhood g(s0), from which round 1 draws all of its
    candidates; their costs are served from a cache when the search asks for them.  Nothing about
    the traversal changes; ``spec_measured`` / ``spec_used`` count the extra hardware
    measurements and how many the search consumed.

    Costs are exchanged with one all_reduce(MAX) of an [n] float64 vector whose entries only the
    measuring rank filled (every cost is > 0), so each candidate is measured exactly once and the
    costs come back by index.
    """

    _instances = itertools.count()     # per-process: identical on every rank that builds evaluators in order

    def __init__(self, measure_one: Optional[Callable] = None, group=None, device: Optional[torch.device] = None,
                 store=None, measure_set: Optional[Callable] = None, assign: Optional[str] = None,
                 space: Optional[tt.Space] = None, cut_s: Optional[Callable[[], float]] = None,
                 speculate: bool = True):
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
        if assign == "auto":
            self.assign = "auto" if self.store is not None else "lpt"
        else:
            self.assign = "dynamic" if self.store is not None else (assign or "lpt")
        if self.assign == "dynamic" and self.store is None and self.world > 1:
            raise ValueError("dynamic assignment needs a store")
        self.round_modes: List[str] = []
        self.space = space
        self.cut_s = cut_s
        self.ns = f"tt_eval{next(ShardedEvaluator._instances)}"
        self.rounds = 0
        self.local_evals = 0
        self.known: dict = {}
        self._nb_cache: dict = {}
        self.speculate = speculate
        self.cache: dict = {}                # speculative costs not yet requested by the search
        self.spec_measured = 0
        self.spec_used = 0
        self.round_states: List[list] = []
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

    @staticmethod
    def _moves(s):
        """Every state one action away from s (Eq. 6: s_x[i] <- 2 s_x[i], s_x[j] <- s_x[j] / 2, s_x[j]
        even), legitimate or not.  Only measured -- hence legitimate -- states are ever looked up in
        the known costs, so min over these equals min over the legitimate neighbours g(s); pure
        Python, because this runs on every rank for every candidate (a ctypes tt_neighbors call per
        candidate cost ~50 us, a third of a bf16 search's host time)."""
        for a, f in enumerate(s):
            for i in range(len(f)):
                for j in range(len(f)):
                    if i != j and f[j] % 2 == 0:
                        g = list(f)
                        g[i] *= 2
                        g[j] //= 2
                        yield s[:a] + (tuple(g),) + s[a + 1:]

    def _predicted_cost(self, s) -> float:
        best = math.inf
        if self.space is not None:
            for t in self._moves(s):
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
    def _speculative(self, states) -> List:
        """States the idle ranks measure while a round that has fewer candidates than ranks runs:
        the round-0 neighbourhood g(s0) (Eq. 9 under reading Z4), in action order.  Round 1 of
        G-BFS draws its candidates from exactly that set (Alg. 1 line 6), so it then costs no
        measurement; the traversal is unchanged (costs are looked up, never re-drawn)."""
        if not self.speculate or self.rounds != 0 or self.world <= len(states) or self.space is None:
            return []
        seen = set(states) | set(self.known) | set(self.cache)
        out = []
        for s in states:
            for t in self._neighbors(s):
                if t not in seen:
                    seen.add(t)
                    out.append(t)
        return out

    def __call__(self, states: Sequence) -> List[float]:
        n = len(states)
        hit = [s in self.cache for s in states]         # measured speculatively in an earlier round
        todo = [j for j in range(n) if not hit[j]]
        sub = [states[j] for j in todo]
        m = len(sub)
        wts = self.weights(sub) if self.assign in ("lpt", "dynamic", "auto") else [1.0] * m
        mode = auto_mode(wts) if self.assign == "auto" else self.assign
        self.round_modes.append(mode)
        spec = self._speculative(sub)
        S = len(spec)
        vals = [0.0] * (2 * m + 2 * S)          # costs, seconds (this round), then speculative costs, seconds
        if mode == "dynamic" and self.world > 1:
            # claim in longest-predicted-first order (LPT order) from a shared counter
            order = sorted(range(m), key=lambda j: (-wts[j], j))
            key = f"{self.ns}_round{self.rounds}"
            while True:
                q = int(self.store.add(key, 1)) - 1
                if q >= m:
                    break
                j = order[q]
                c, t = self.measure_set(sub, [i == j for i in range(m)])
                vals[j], vals[m + j] = c[j], t[j]
                self.local_evals += 1
            if S:                                        # then the speculative states, same way
                while True:
                    q = int(self.store.add(key + "_spec", 1)) - 1
                    if q >= S:
                        break
                    c, t = self.measure_set(spec, [i == q for i in range(S)])
                    vals[2 * m + q], vals[2 * m + S + q] = c[q], t[q]
            spec_owner = []
        else:
            if mode == "lpt":
                owner = self.lpt_owners(wts, self.world)
            else:
                owner = [j % self.world for j in range(m)]
            mine = [o == self.rank for o in owner]
            if any(mine):
                c, t = self.measure_set(sub, mine)
                for j in range(m):
                    if mine[j]:
                        vals[j], vals[m + j] = c[j], t[j]
                        self.local_evals += 1
            busy = set(owner)
            idle = [r for r in range(self.world) if r not in busy] or list(range(self.world))
            spec_owner = [idle[i % len(idle)] for i in range(S)]
        if S and spec_owner:
            smine = [o == self.rank for o in spec_owner]
            if any(smine):
                c, t = self.measure_set(spec, smine)
                for i in range(S):
                    if smine[i]:
                        vals[2 * m + i], vals[2 * m + S + i] = c[i], t[i]
        if self.world > 1:
            buf = torch.tensor(vals, dtype=torch.float64, device=self.device)
            dist.all_reduce(buf, op=dist.ReduceOp.MAX, group=self.group)
            vals = buf.cpu().tolist()
            if mode == "dynamic" and self.rank == 0:
                for k in (f"{self.ns}_round{self.rounds}", f"{self.ns}_round{self.rounds}_spec"):
                    try:                                 # every rank has left its claim loops
                        self.store.delete_key(k)
                    except Exception:  # noqa: BLE001 - older stores: keys are namespaced anyway
                        pass
        costs = [0.0] * n
        secs = [0.0] * n
        for q, j in enumerate(todo):
            costs[j], secs[j] = vals[q], vals[m + q]
        for j in range(n):
            if hit[j]:
                costs[j] = self.cache.pop(states[j])
                self.spec_used += 1
        if not all(c > 0 for c in costs):
            raise RuntimeError(f"sharded round {self.rounds}: a candidate came back unmeasured ({costs})")
        for i in range(S):
            if vals[2 * m + i] > 0:
                self.cache[spec[i]] = vals[2 * m + i]
                self.spec_measured += 1
        self.round_times.append(secs)
        self.round_weights.append([w for w in wts] if m == n else
                                  [wts[todo.index(j)] if not hit[j] else 0.0 for j in range(n)])
        self.round_states.append(list(states))
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


def _busy(times: Sequence[float], world: int, mode: str, weights: Optional[Sequence[float]], per_claim_s: float):
    """Per-rank busy time of one round's candidates under an assignment rule."""
    busy = [0.0] * world
    if mode == "dynamic":                                  # list scheduling, LPT order if weighted
        order = sorted(range(len(times)), key=lambda j: (-weights[j], j)) if weights is not None else range(len(times))
        for j in order:
            r = min(range(world), key=lambda i: busy[i])
            busy[r] += times[j] + per_claim_s
    else:
        owner = ShardedEvaluator.lpt_owners(weights, world) if mode == "lpt" else [j % world for j in range(len(times))]
        for j, t in enumerate(times):
            busy[owner[j]] += t
    return busy


def projected_sharded_wall(round_times: Sequence[Sequence[float]], world: int, per_round_s: float = 0.0,
                           dynamic: bool = False, per_claim_s: float = 0.0,
                           weights: Optional[Sequence[Sequence[float]]] = None,
                           states: Optional[Sequence[Sequence]] = None, neighbors: Optional[Callable] = None,
                           auto: bool = False) -> float:
    """Measurement wall time of the same traversal sharded over ``world`` ranks, from
    per-candidate times recorded on one rank: sum over rounds of the slowest rank's busy time,
    plus ``per_round_s`` (the exchange) per round.  Static: candidate j on rank j mod world.
    ``weights`` given: the evaluator's LPT assignment from those predicted weights (with
    ``dynamic``: claims in that order).  Dynamic: each candidate goes to the rank that becomes
    free first, each claim costing ``per_claim_s``.  ``states`` + ``neighbors`` given: the
    speculative round 0 (ShardedEvaluator.speculate) -- the idle ranks measure g(s0) while s0 runs,
    each such state costing what it cost when the search measured it (else the dearest of them),
    and later rounds do not re-measure those states.  ``auto`` (needs ``weights``): each round
    dynamic or LPT by the evaluator's auto rule (``auto_mode``).  A projection from measured
    times, not a multi-GPU measurement."""
    mode = "dynamic" if dynamic else ("lpt" if weights is not None else "static")
    if auto:
        mode = "auto"
    spec_t = {}
    if states is not None and neighbors is not None and world > 1 and round_times and len(round_times[0]) < world:
        seen = set(states[0])
        order = []
        for s0 in states[0]:
            for t in neighbors(s0):
                if t not in seen:
                    seen.add(t)
                    order.append(t)
        when = {}
        for k in range(1, len(states)):
            for s, t in zip(states[k], round_times[k]):
                when.setdefault(s, t)
        known = [when[t] for t in order if t in when]
        fallback = max(known) if known else max(round_times[0])
        spec_t = {t: when.get(t, fallback) for t in order}
    total = 0.0
    for k, times in enumerate(round_times):
        w = weights[k] if weights is not None else None
        if spec_t and k > 0:
            keep = [j for j, s in enumerate(states[k]) if s not in spec_t]
            times = [times[j] for j in keep]
            w = [w[j] for j in keep] if w is not None else None
            for s in states[k]:                            # a speculative state is served once
                spec_t.pop(s, None)
        rmode = (auto_mode(weights[k]) if weights is not None else "static") if mode == "auto" else mode
        busy = _busy(times, world, rmode, w, per_claim_s)
        if spec_t and k == 0:
            st = list(spec_t.values())
            if rmode == "dynamic":
                for t in st:
                    r = min(range(world), key=lambda i: busy[i])
                    busy[r] += t + per_claim_s
            else:
                idle = [r for r in range(world) if busy[r] == 0.0] or list(range(world))
                for i, t in enumerate(st):
                    busy[idle[i % len(idle)]] += t
        total += (max(busy) if busy else 0.0) + (per_round_s if world > 1 else 0.0)
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
