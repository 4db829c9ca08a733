"""Multi-GPU plumbing (B6): one process per GPU, torch.distributed for the exchange.

Two partitions of the hot path:

1. Candidate-batch sharding for the searches.  Every rank runs the identical search (same
   seed, same code, replicated state); a round's candidates are independent measurements, so
   candidate j is measured on rank j mod G and the (j, cost) pairs are all-gathered.  The
   traversal depends only on (seed, W, rho, cost values), never on G.
2. Row-partitioned large GEMM: rank r owns rows [r M/G, (r+1) M/G) of A and C, B is
   replicated, and there is no collective on the math path (``row_shard``).

torch is used for the process group and the tiny timing tensors only; every measurement is a
libtiletune call.
"""
from __future__ import annotations

import math
import time
from typing import Callable, List, Optional, Sequence

import torch
import torch.distributed as dist

from . import tiletune as tt


class ShardedEvaluator:
    """BATCH cost source for tt.gbfs_search / tt.na2c_search.

    ``measure_one(state) -> float`` scores one candidate on this rank (normally a
    ``tt.Context.measure``).  Assignment of a round's candidates to ranks:

    * static (default): candidate j on rank j mod G; one all_gather of a [G, n] float64 tensor;
    * dynamic (``store`` given): ranks claim the next unmeasured candidate index from a shared
      counter (``store.add``, the process group's TCPStore) as soon as they are free, so one slow
      candidate does not hold up the others; one all_reduce(MAX) of an [n] float64 tensor whose
      entries only the claiming rank filled (costs are > 0).

    Either way each candidate is measured exactly once and the costs are returned by index, so
    the traversal depends only on (seed, W, rho, costs), never on G or on the assignment.
    """

    def __init__(self, measure_one: Callable, group=None, device: Optional[torch.device] = None, store=None):
        self.measure_one = measure_one
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.device = device or torch.device("cpu")
        self.store = store if self.world > 1 else None
        self.rounds = 0
        self.local_evals = 0
        self.round_times: List[List[float]] = []   # per round: wall time of each local measurement

    def _measure(self, states, j, mine, times):
        t0 = time.perf_counter()
        mine[j] = float(self.measure_one(states[j]))
        times[j] = time.perf_counter() - t0
        self.local_evals += 1

    def __call__(self, states: Sequence) -> List[float]:
        n = len(states)
        mine = torch.zeros(n, dtype=torch.float64, device=self.device)
        times = [0.0] * n
        if self.store is not None:
            key = f"tt_round_{self.rounds}"
            while True:
                j = int(self.store.add(key, 1)) - 1
                if j >= n:
                    break
                self._measure(states, j, mine, times)
        else:
            for j in range(self.rank, n, self.world):
                self._measure(states, j, mine, times)
        self.round_times.append(times)
        self.rounds += 1
        if self.world == 1:
            return mine.tolist()
        if self.store is not None:
            dist.all_reduce(mine, op=dist.ReduceOp.MAX, group=self.group)
            return [float(x) for x in mine.cpu().tolist()]
        out = torch.empty(self.world * n, dtype=torch.float64, device=self.device)
        dist.all_gather_into_tensor(out, mine, group=self.group)
        g = out.view(self.world, n).cpu()
        return [float(g[j % self.world, j]) for j in range(n)]


def default_store():
    """The default process group's TCPStore (for dynamic assignment), or None."""
    try:
        from torch.distributed import distributed_c10d as c10d
        return c10d._get_default_store()
    except Exception:  # noqa: BLE001 - private API moved: fall back to the static assignment
        return None


def device_measure(ctx: tt.Context, sp: tt.Space, opts: Optional[tt.MeasureOpts] = None, cut_factor: float = 20.0,
                   cut_floor_s: float = 0.05):
    """measure_one for ShardedEvaluator: tt_measure with the slow-candidate cut of reading Z12
    driven by the best cost seen so far (identical on every rank: it is computed from the
    gathered costs the search pushes)."""
    state = {"best": math.inf}
    base = opts or tt.measure_opts()

    def f(s):
        mo = tt.MeasureOpts.from_buffer_copy(base)
        if math.isfinite(state["best"]):
            mo.cut_s = max(cut_factor * state["best"], cut_floor_s)
        c = ctx.measure(sp, s, mo).cost_s
        return c

    def observe(costs):
        for c in costs:
            state["best"] = min(state["best"], c)

    return f, observe


def projected_sharded_wall(round_times: Sequence[Sequence[float]], world: int, per_round_s: float = 0.0,
                           dynamic: bool = False, per_claim_s: float = 0.0) -> float:
    """Measurement wall time of the same traversal sharded over ``world`` ranks, from
    per-candidate times recorded on one rank: sum over rounds of the slowest rank's busy time,
    plus ``per_round_s`` (the collective) per round.  Static: candidate j on rank j mod world.
    Dynamic: candidates in index order each go to the rank that becomes free first (what the
    counter-claiming evaluator does), each claim costing ``per_claim_s``.  A projection from
    measured times, not a multi-GPU measurement."""
    total = 0.0
    for times in round_times:
        busy = [0.0] * world
        for j, t in enumerate(times):
            r = min(range(world), key=lambda i: busy[i]) if dynamic else j % world
            busy[r] += t + (per_claim_s if dynamic else 0.0)
        total += max(busy) + (per_round_s if world > 1 else 0.0)
    return total


class TrackingEvaluator(ShardedEvaluator):
    """ShardedEvaluator that feeds the gathered costs back into a cut tracker."""

    def __init__(self, measure_one, observe, **kw):
        super().__init__(measure_one, **kw)
        self.observe = observe

    def __call__(self, states):
        costs = super().__call__(states)
        self.observe(costs)
        return costs


def row_shard(M: int, world: int, rank: int):
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
