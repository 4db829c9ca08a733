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

import bisect
import heapq
import itertools
import math
import time
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist

from . import tiletune as tt

# measurement-time model of one candidate for the LPT assignment (reading Z12's scoring rules): a
# candidate above the slow cut is scored by its probe (1 launch); below it, the probe and R = 10
# repeats (11 launches) unless racing stops it after 2 repeats (3) -- predicted when its predicted
# cost exceeds 1.1 x the incumbent.  Every launch costs the GEMM plus an overhead (L2 flush, events,
# host) that the evaluator calibrates from the exchanged (cost, seconds) of the measured candidates.
_FULL_LAUNCHES = 11
_RACED_LAUNCHES = 3
_RACE_RATIO = 1.1
# racing compares the first repeats (not the cold probe) with 1.1 x the incumbent; a probe up to
# 10 % above that line still often runs the full repeats (measured on the B200: probes sit 1-7 %
# above the final cost), so phase 2 predicts "raced" only beyond it -- predicting a short
# candidate long costs an LPT plan little, the converse leaves one rank running at the round's end
_PROBE_MARGIN = 0.1
# "auto" claims dynamically only in rounds whose median predicted measurement time is >=
# _AUTO_CLAIMS x _CLAIM_S = 2 ms, else it uses the LPT (or two-phase) plan.  _CLAIM_S is a
# conservative budget per claim (a TCPStore add round trip plus one measure call's marshalling:
# 21 us measured on the GPU host, bench.py claim_s); the 2 ms line keeps the bf16 rounds (0.3-2.9
# ms candidates) on the two-phase plan, which the replays rate above dynamic claiming there
# (profiles/r12_replay_sharded_bf16_4096.txt), and sends the long fp32 rounds to dynamic claims.
_CLAIM_S = 200e-6
_AUTO_CLAIMS = 10


def auto_mode(weights: Sequence[float]) -> str:
    """The "auto" rule for one round (identical on every rank: the weights come from the
    replicated known costs): dynamic claiming when the median predicted measurement time is at
    least _AUTO_CLAIMS claim round trips, else the LPT plan (no per-candidate store traffic)."""
    raw = sorted(weights)
    med = raw[len(raw) // 2] if raw else 0.0
    return "dynamic" if med >= _AUTO_CLAIMS * _CLAIM_S else "lpt"


class ShardedEvaluator:
    """BATCH cost source for tt.gbfs_search / tt.na2c_search / tt.random_search.

    ``measure_set(states, mine) -> (costs, seconds)`` scores the states whose ``mine`` flag is
    set on this rank (normally ``device_measure_set``: one tt_measure_set call, C++ loop) and
    returns 0 elsewhere.  For host-side tests ``measure_one(state) -> cost`` is accepted instead.

    Assignment of a round's candidates to ranks (``assign``):

    * ``"lpt"`` (default): longest predicted measurement first, each to the least-loaded rank.
      The predicted cost of a candidate is the geometric mean of the known costs of its measured
      neighbours (a neighbour differs by one x2 / /2 move), turned into seconds by the
      scoring rules (1 launch above the cut, 3 when racing is expected to stop it, else 11) and
      the calibrated per-launch overhead.  Every rank holds the same known costs, so every rank
      computes the same assignment with no communication.
    * ``"static"``: candidate j on rank j mod G.
    * ``"dynamic"`` (``store`` given): ranks claim the next unmeasured candidate, in the LPT
      order of the predictions, from a shared counter (``store.add``) whenever they are free.
    * ``"auto"`` (``store`` given): per round, dynamic when the median predicted measurement time
      is at least 10 claim round trips (~2 ms), else the LPT plan -- short candidates (bf16 at
      4096^3, ~1 ms each) do not pay a store round trip apiece, long ones (fp32) balance
      dynamically.

    Two-phase rounds (``measure_phase`` given, e.g. from ``device_measure_set``): a round with more
    candidates than ranks measures every cold probe first (LPT over predicted probe times), then
    the rest of each unfinished measurement, LPT over predictions made from the exchanged probes.

    Speculation (``speculate``, needs ``space``): in round 0 -- s0 alone, so G - 1 ranks would
    idle -- the idle ranks measure s0's neighbourhood g(s0) (only the cold probes when
    ``measure_phase`` is given), from which round 1 draws all of its candidates; their costs or
    probes are served from caches when the search asks for them.  Nothing about the traversal
    changes; ``spec_measured`` / ``spec_used`` count the extra hardware measurements and how many
    the search consumed.

    Results are exchanged with one all_reduce(MAX) per phase of a float64 vector whose entries
    only the measuring rank filled (every cost is > 0), so each candidate is measured exactly
    once and the costs come back by index.
    """

    _instances = itertools.count()     # per-process: identical on every rank that builds evaluators in order

    def __init__(self, measure_one: Optional[Callable] = None, group=None, device: Optional[torch.device] = None,
                 store=None, measure_set: Optional[Callable] = None, assign: Optional[str] = None,
                 space: Optional[tt.Space] = None, cut_s: Optional[Callable[[], float]] = None,
                 speculate: bool = True, measure_phase: Optional[Callable] = None):
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
        self.measure_phase = measure_phase
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
        self._known_code: dict = {}              # packed-exponent key -> cost (see _code)
        self._kc_arrays = None                   # (sorted codes, log costs) for _predicted_costs
        self._best = math.inf                    # min(known.values())
        self._move_deltas = None
        self.plan_s = 0.0                        # host seconds spent planning rounds (replicated work)
        self._over = 0.0                         # calibrated per-launch overhead (weights)
        self._over_obs: List[float] = []
        self._over1 = 0.0                        # calibrated overhead of a phase-1 probe call
        self._over1_obs: List[float] = []
        self._nb_cache: dict = {}
        self.speculate = speculate
        self.cache: dict = {}                # speculative costs not yet requested by the search
        self.probe_cache: dict = {}          # speculative cold probes (phase 1) not yet requested
        self.spec_measured = 0
        self.spec_used = 0
        self.round_states: List[list] = []
        self.round_spec: List[tuple] = []        # per round: (speculative states, their seconds)
        # per round, two-phase rounds only (else empty lists): phase-1 seconds, probe values, and
        # whether the probe alone decided the score
        self.round_phase1: List[tuple] = []
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
        the known costs, so the known costs among these are those of the measured part of g(s)."""
        for a, f in enumerate(s):
            for i in range(len(f)):
                for j in range(len(f)):
                    if i != j and f[j] % 2 == 0:
                        g = list(f)
                        g[i] *= 2
                        g[j] //= 2
                        yield s[:a] + (tuple(g),) + s[a + 1:]

    _codes: dict = {}                          # state -> packed code (None: not all powers of two)

    @classmethod
    def _code(cls, s):
        """Packed log2 exponents (5 bits per factor, outer to inner, m then k then n) when every
        factor is a power of two (the paper's square 2^j problems), else None.  An action of Eq. 6
        is then one integer add: +1 on exponent i, -1 on exponent j of the same axis."""
        code = cls._codes.get(s, -1)
        if code != -1:
            return code
        code, sh = 0, 0
        for f in s:
            for v in f:
                if v & (v - 1):
                    cls._codes[s] = None
                    return None
                code |= (v.bit_length() - 1) << sh
                sh += 5
        if len(cls._codes) > 1 << 20:
            cls._codes.clear()
        cls._codes[s] = code
        return code

    def _deltas(self, s):
        d = self._move_deltas
        if d is None:
            d, base = [], 0
            for f in s:
                L = len(f)
                for i in range(L):
                    for j in range(L):
                        if i != j:
                            d.append(((1 << 5 * (base + i)) - (1 << 5 * (base + j)), 5 * (base + j)))
                base += L
            self._move_deltas = d
        return d

    def _predicted_cost(self, s) -> float:
        """Geometric mean of the known costs of the states one action away from s (measured
        states are legitimate, so these are its measured neighbours in g(s)); the minimum known
        cost if none is known.  On the measured bf16 4096^3 costs it classifies racing correctly
        for 83 % of the candidates, the neighbours' minimum for 74 % (tools/spec_study.py).  Pure
        Python over packed exponents: this runs on every rank for every candidate (a ctypes
        tt_neighbors call per candidate costs ~50 us)."""
        acc, n = 0.0, 0
        if self.space is not None:
            c = self._code(s)
            if c is not None:
                get = self._known_code.get
                log = math.log
                for d, sh in self._deltas(s):
                    if (c >> sh) & 31:
                        v = get(c + d)
                        if v is not None:
                            acc += log(v)
                            n += 1
            else:
                for t in self._moves(s):
                    v = self.known.get(t)
                    if v is not None:
                        acc += math.log(v)
                        n += 1
        if n:
            return math.exp(acc / n)
        return min(self.known.values()) if self.known else 1.0

    def _predicted_costs(self, states) -> List[float]:
        """_predicted_cost of every state at once: on packed codes the neighbour lookups of a whole
        round are one sorted search over the known codes (numpy); the planning of a round is host
        work every rank repeats, so it stays off the round's critical path as far as possible."""
        codes = [self._code(s) for s in states] if self.space is not None else [None]
        if not states or any(c is None for c in codes) or not self._known_code:
            return [self._predicted_cost(s) for s in states]
        if self._kc_arrays is None:
            ks = sorted(self._known_code)
            self._kc_arrays = (np.array(ks, dtype=np.int64),
                               np.array([math.log(self._known_code[k]) for k in ks], dtype=np.float64))
        K, L = self._kc_arrays
        dl = self._deltas(states[0])
        D = np.array([d for d, _ in dl], dtype=np.int64)
        SH = np.array([sh for _, sh in dl], dtype=np.int64)
        C = np.array(codes, dtype=np.int64)[:, None]
        valid = ((C >> SH[None, :]) & 31) != 0
        nbr = C + D[None, :]
        idx = np.minimum(np.searchsorted(K, nbr), len(K) - 1)
        found = valid & (K[idx] == nbr)
        n = found.sum(axis=1)
        acc = np.where(found, L[idx], 0.0).sum(axis=1)
        fallback = min(self.known.values())
        return [math.exp(a / k) if k else fallback for a, k in zip(acc.tolist(), n.tolist())]

    def set_known(self, known: dict):
        """Replace the known costs (tests; the search fills them round by round)."""
        self.known = {}
        self._known_code = {}
        self._kc_arrays = None
        self._best = math.inf
        for s, c in known.items():
            self._remember(s, c)

    def _remember(self, s, c):
        self.known[s] = c
        if c < self._best:
            self._best = c
        k = self._code(s)
        if k is not None:
            self._known_code[k] = c
            self._kc_arrays = None

    @staticmethod
    def launches(c: float, best: float, cut: float) -> int:
        """Launches the scoring rules (reading Z12) spend on a candidate of cost c at incumbent
        ``best`` and slow cut ``cut`` (0 = none)."""
        if cut > 0 and c > cut:
            return 1
        if math.isfinite(best) and c > _RACE_RATIO * best:
            return _RACED_LAUNCHES
        return _FULL_LAUNCHES

    def weights(self, states, preds: Optional[Sequence[float]] = None) -> List[float]:
        """Predicted measurement seconds of each state: launches(predicted cost) x (predicted cost +
        calibrated per-launch overhead).  Identical on every rank (exchanged costs only)."""
        cut = self.cut_s() if self.cut_s is not None else 0.0
        best = self._best
        o = self._over
        if preds is None:
            preds = self._predicted_costs(states)
        return [self.launches(c, best, cut) * (c + o) for c in preds]

    def _calibrate(self, costs, secs, best, cut):
        """Per-launch overhead = median over measured candidates of secs / launches - cost."""
        v = self._over_obs                      # kept sorted
        for c, t in zip(costs, secs):
            if c > 0 and t > 0:
                bisect.insort(v, max(0.0, t / self.launches(c, best, cut) - c))
        if v:
            self._over = v[len(v) // 2]

    @staticmethod
    def lpt_owners(weights: Sequence[float], world: int) -> List[int]:
        """Longest-processing-time-first list scheduling: candidates in decreasing weight (ties by
        index) go to the least-loaded rank (ties: lowest rank).  Deterministic."""
        owner = [0] * len(weights)
        heap = [(0.0, r) for r in range(world)]
        for j in sorted(range(len(weights)), key=lambda j: (-weights[j], j)):
            load, r = heapq.heappop(heap)
            owner[j] = r
            heapq.heappush(heap, (load + weights[j], r))
        return owner

    # ------------------------------------------------------------------ one round
    def _speculative(self, sub, wts, owner):
        """States measured speculatively in this round, and their ranks.

        Round 0 (s0 alone, fewer candidates than ranks): the idle ranks measure g(s0) (Eq. 9
        under reading Z4), from which round 1 of G-BFS draws all of its candidates (Alg. 1 line
        6) -- every state, spread over the idle ranks; with a phase measurer only their cold
        probes (``_measure_spec``), and round 1 finishes the ones it draws.
        (Speculating later rounds -- the unmeasured neighbours of the states the next G-BFS round
        is expected to pop, filling each rank's idle time -- was simulated on the measured bf16
        4096^3 costs, tools/spec_study.py: with W = 16 the ranks' idle time rarely fits a whole
        candidate and it bought nothing, so it is not built.)
        The traversal is unchanged either way: a speculative cost is only looked up when the
        search requests that state (never re-drawn)."""
        if not self.speculate or self.space is None or self.world <= 1:
            return [], []
        if self.rounds == 0:
            if self.world <= len(sub):
                return [], []
            seen = set(sub) | set(self.known) | set(self.cache) | set(self.probe_cache)
            out = []
            for s in sub:
                for t in self._neighbors(s):
                    if t not in seen:
                        seen.add(t)
                        out.append(t)
            if owner is None:
                return out, None
            busy = set(owner)
            idle = [r for r in range(self.world) if r not in busy] or list(range(self.world))
            return out, [idle[i % len(idle)] for i in range(len(out))]
        return [], []

    def plan(self, states):
        """The round's plan, identical on every rank (it depends only on the exchanged costs):
        (hit, todo, wts, mode, owner, spec, spec_owner).  ``owner`` is None for dynamic claims;
        ``spec_owner`` is None when speculative states are claimed dynamically."""
        hit = [s in self.cache for s in states]         # measured speculatively in an earlier round
        todo = [j for j in range(len(states)) if not hit[j]]
        sub = [states[j] for j in todo]
        m = len(sub)
        preds = self._predicted_costs(sub) if self.assign in ("lpt", "dynamic", "auto") else None
        wts = self.weights(sub, preds) if preds is not None else [1.0] * m
        mode = auto_mode(wts) if self.assign == "auto" else self.assign
        cached = [s in self.probe_cache for s in sub]
        if self.two_phase(m, mode) or (self.measure_phase is not None and any(cached)):
            # phase 1 = the cold probes, balanced by the predicted probe time (one launch each);
            # a candidate whose probe was taken speculatively skips it (owner None)
            mode = "two-phase"
            o = self._over1 if self._over1_obs else self._over
            idx = [j for j in range(m) if not cached[j]]
            own = self.lpt_owners([preds[j] + o for j in idx], self.world) if preds is not None else \
                [q % self.world for q in range(len(idx))]
            owner = [None] * m
            for q, j in enumerate(idx):
                owner[j] = own[q]
            return hit, todo, sub, wts, mode, owner, [], []
        if mode == "dynamic" and self.world > 1:
            owner = None
        elif mode == "lpt":
            owner = self.lpt_owners(wts, self.world)
        else:
            owner = [j % self.world for j in range(m)]
        spec, spec_owner = self._speculative(sub, wts, owner)
        return hit, todo, sub, wts, mode, owner, spec, spec_owner

    def two_phase(self, m: int, mode: str) -> bool:
        """A round runs in two phases (probes, exchange, then the rest of each measurement balanced
        with the probes known; tt_measure_phase) when the evaluator has a phase measurer, the round
        has more candidates than ranks, and its candidates are not claimed dynamically."""
        return self.measure_phase is not None and m > self.world and mode != "dynamic" and self.assign != "static"

    def phase2_plan(self, probes, final, cut):
        """Owners of the phase-2 work (None for candidates the probe finished) and its predicted
        seconds: (launches(probe) - 1) x (probe + overhead) -- the racing prediction now uses the
        measured probe instead of the neighbours' costs."""
        best = self._best
        o = self._over
        idx = [j for j in range(len(probes)) if not final[j]]
        w2 = [(self.launches(probes[j] / (1 + _PROBE_MARGIN), best, cut) - 1) * (probes[j] + o) for j in idx]
        own = self.lpt_owners(w2, self.world)
        owner2 = [None] * len(probes)
        for q, j in enumerate(idx):
            owner2[j] = own[q]
        return owner2, w2

    def warm_up(self, states):
        """Run the planning code once on ``states`` with throw-away costs and forget it, so the
        first timed round does not pay Python's and numpy's first-call costs (measured ~3 ms on
        the GPU hosts: more than a whole bf16 round's planning)."""
        saved = (self.known, self._known_code, self._kc_arrays, self._best, self._over, self._over_obs,
                 self._over1, self._over1_obs)
        self.set_known({s: 1.0 + 1e-3 * i for i, s in enumerate(states)})
        self._over_obs = []
        self._over1_obs = []
        self.calibrate_probes([1.0], [1.5])
        self._predicted_costs(list(states))
        self.weights(list(states))
        self.lpt_owners([1.0] * len(states), max(1, self.world))
        self.phase2_plan([1.0] * len(states), [False] * len(states), 0.0)
        self._calibrate([1.0], [2.0], 1.0, 0.0)
        (self.known, self._known_code, self._kc_arrays, self._best, self._over, self._over_obs,
         self._over1, self._over1_obs) = saved

    def _measure_spec(self, spec, mine):
        """(values, final flags, seconds) of the speculative states this rank owns.  With a phase
        measurer only their cold probes: in round 0 there is no incumbent yet, so racing could not
        shorten whole measurements (a 0.4 ms bf16 config would run all 11 launches); the round
        that requests a state finishes it with the incumbent known (phase 2).  A probe the slow
        cut decides is final.  Without a phase measurer: whole measurements."""
        if self.measure_phase is not None:
            return self.measure_phase(spec, mine, 1, None)
        c, t = self.measure_set(spec, mine)
        return c, [True] * len(spec), t

    def _exchange(self, vals):
        """all_reduce(MAX) of a host float vector whose entries only the owning rank filled."""
        buf = torch.tensor(vals, dtype=torch.float64, device=self.device)
        dist.all_reduce(buf, op=dist.ReduceOp.MAX, group=self.group)
        return buf.cpu().tolist()

    def _two_phase(self, sub, owner, cut, vals):
        """Measure a round in two phases; fills vals[:m] (costs) and vals[m:2m] (seconds, both
        phases) like the one-phase path and returns per candidate (phase-1 seconds, probe or
        final value, final?).  Phase 1: each rank probes its LPT share, one exchange.  Phase 2:
        the unfinished candidates' remaining launches, LPT over the probe-based predictions, a
        second exchange.  A candidate's repeats may run on another rank than its probe (same GPU
        model; under the L2 flush every timed launch starts cold, and the probe only decides the
        cut and the prediction)."""
        m = len(sub)
        mine = [o == self.rank for o in owner]
        v1 = [0.0] * (3 * m)                   # value, final flag, seconds
        for j, s in enumerate(sub):
            if owner[j] is None:                 # probed speculatively in an earlier round
                v1[j] = self.probe_cache.pop(s)
                self.spec_used += 1
        if any(mine):
            val, fin, sec = self.measure_phase(sub, mine, 1, None)
            for j in range(m):
                if mine[j]:
                    v1[j], v1[m + j], v1[2 * m + j] = val[j], 1.0 if fin[j] else 0.0, sec[j]
        if self.world > 1:
            v1 = self._exchange(v1)           # cached entries are identical on every rank
        probes = v1[:m]
        final = [v1[m + j] > 0.5 for j in range(m)]
        self.calibrate_probes(probes, v1[2 * m:])
        t0 = time.perf_counter()
        owner2, _ = self.phase2_plan(probes, final, cut)
        self.plan_s += time.perf_counter() - t0
        mine2 = [o == self.rank for o in owner2]
        v2 = [0.0] * (2 * m)
        for j in range(m):
            if final[j] and owner[j] == self.rank:
                v2[j] = probes[j]
        if any(mine2):
            val, _, sec = self.measure_phase(sub, mine2, 2, probes)
            for j in range(m):
                if mine2[j]:
                    v2[j], v2[m + j] = val[j], sec[j]
                    self.local_evals += 1
        for j in range(m):
            if final[j] and owner[j] == self.rank:
                self.local_evals += 1
        if self.world > 1:
            v2 = self._exchange(v2)
        for j in range(m):
            vals[j] = v2[j]
            vals[m + j] = v1[2 * m + j] + v2[m + j]
        return [(v1[2 * m + j], probes[j], final[j]) for j in range(m)]

    def calibrate_probes(self, probes, secs1):
        """Phase-1 overhead = median over probed candidates of (seconds - probe): a probe call
        also pays the candidate's first-launch host setup (plan, tensor maps)."""
        v = self._over1_obs
        for p, t in zip(probes, secs1):
            if p > 0 and t > 0:
                bisect.insort(v, max(0.0, t - p))
        if v:
            self._over1 = v[len(v) // 2]

    def absorb(self, states, costs, spec, spec_costs, secs=None, cut=0.0, spec_final=None):
        """Record a finished round: requested costs become known, their measurement seconds
        calibrate the weight model, speculative costs (final) or probes wait in their caches until
        requested."""
        if secs is not None:
            self._calibrate(costs, secs, self._best, cut)
        for i, t in enumerate(spec):
            if spec_costs[i] > 0:
                if spec_final is None or spec_final[i]:
                    self.cache[t] = spec_costs[i]
                else:
                    self.probe_cache[t] = spec_costs[i]
                self.spec_measured += 1
        for s, c in zip(states, costs):
            self._remember(s, c)
        self.round_states.append(list(states))
        self.rounds += 1

    def __call__(self, states: Sequence) -> List[float]:
        n = len(states)
        t0 = time.perf_counter()
        cut = self.cut_s() if self.cut_s is not None else 0.0
        hit, todo, sub, wts, mode, owner, spec, spec_owner = self.plan(states)
        self.plan_s += time.perf_counter() - t0
        m = len(sub)
        self.round_modes.append(mode)
        S = len(spec)
        # costs, seconds (this round), then speculative values, seconds, final flags
        vals = [0.0] * (2 * m + 3 * S)
        p1 = None
        if mode == "two-phase":
            p1 = self._two_phase(sub, owner, cut, vals)
        elif owner is None:
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
                    c, f, t = self._measure_spec(spec, [i == q for i in range(S)])
                    vals[2 * m + q], vals[2 * m + S + q], vals[2 * m + 2 * S + q] = c[q], t[q], float(f[q])
        else:
            mine = [o == self.rank for o in owner]
            if any(mine):
                c, t = self.measure_set(sub, mine)
                for j in range(m):
                    if mine[j]:
                        vals[j], vals[m + j] = c[j], t[j]
                        self.local_evals += 1
            smine = [o == self.rank for o in spec_owner]
            if any(smine):
                c, f, t = self._measure_spec(spec, smine)
                for i in range(S):
                    if smine[i]:
                        vals[2 * m + i], vals[2 * m + S + i], vals[2 * m + 2 * S + i] = c[i], t[i], float(f[i])
        if self.world > 1 and p1 is None:
            vals = self._exchange(vals)
        if self.world > 1:
            if owner is None and self.rank == 0:
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
        self.round_times.append(secs)
        self.round_weights.append([w for w in wts] if m == n else
                                  [wts[todo.index(j)] if not hit[j] else 0.0 for j in range(n)])
        self.round_spec.append((list(spec), vals[2 * m + S:2 * m + 2 * S]))
        if p1 is not None:
            ph = [(0.0, 0.0, False)] * n
            for q, j in enumerate(todo):
                ph[j] = p1[q]
            self.round_phase1.append(tuple(zip(*ph)))
        else:
            self.round_phase1.append(([], [], []))
        self.absorb(states, costs, spec, vals[2 * m:2 * m + S], secs=secs, cut=cut,
                    spec_final=[v > 0.5 for v in vals[2 * m + 2 * S:2 * m + 3 * S]])
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
    Returns (measure_set, observe, cut_s, measure_phase) where observe(costs) updates the
    incumbent, cut_s() is the current cut (for the weights) and measure_phase(states, mine, phase,
    probes) is the two-phase form (tt_measure_phase)."""
    state = {"best": math.inf, "mo": None, "mo_best": None}

    def mo():                                # one tt_scoring_opts call per incumbent value
        if state["mo_best"] != state["best"]:
            state["mo"] = tt.scoring_opts(sp, opts, state["best"], device)
            state["mo_best"] = state["best"]
        return state["mo"]

    def measure_set(states, mine):
        return ctx.measure_set(sp, states, mine, mo())

    def measure_phase(states, mine, phase, probes):
        return ctx.measure_phase(sp, states, mine, phase, probes, mo())

    def observe(costs):
        for c in costs:
            state["best"] = min(state["best"], c)

    return measure_set, observe, lambda: mo().cut_s, measure_phase


def simulate_sharded(round_states: Sequence[Sequence], round_costs: Sequence[Sequence[float]],
                     round_times: Sequence[Sequence[float]], world: int, *, space: Optional[tt.Space],
                     assign: str = "lpt", speculate: bool = True, two_phase: bool = False,
                     round_phase1: Optional[Sequence[tuple]] = None,
                     cut_of: Optional[Callable[[float], float]] = None, spec_time: Optional[Callable] = None,
                     per_round_s: float = 50e-6, per_claim_s: float = 200e-6) -> dict:
    """Projection of a recorded search (rounds of requested states, their costs and the seconds
    each took to measure on one GPU) onto ``world`` ranks by running the evaluator's own planning
    code (``ShardedEvaluator.plan`` / ``phase2_plan`` / ``absorb``: weights, assignment,
    speculation, two-phase rounds) with the recorded costs.  Per round: the slowest rank's busy
    time (its candidates' recorded seconds, plus ``per_claim_s`` per dynamic claim) +
    ``per_round_s`` per exchange (two in a two-phase round).  Two-phase rounds split a candidate's
    seconds at its probe: the recorded phase-1 seconds and probe value when the one-GPU run was
    two-phase too (``round_phase1``, ShardedEvaluator.round_phase1), else one launch's share
    (seconds / launches(cost)) with probe = cost.  ``cut_of(incumbent)`` gives the slow cut the weights assume
    (tt.scoring_opts), none if omitted.  Speculation and assignment cannot change the traversal,
    so the recorded rounds are exactly what the sharded run requests.  Round-0 speculation costs
    each state its probe with ``two_phase`` (recorded phase-1 seconds, else their median), else a
    whole measurement without an incumbent (11 launches of recorded cost + the calibrated
    per-launch overhead; ``spec_time(state)`` overrides).  Returns {"wall_s",
    "plan_host_s" (the planning code's own host time), "spec_measured", "spec_used", "modes"}.
    A projection from one-GPU times, not a multi-GPU measurement."""
    ev = ShardedEvaluator(measure_set=lambda st, mi: ([0.0] * len(st), [0.0] * len(st)), space=space,
                          speculate=speculate, assign=assign if assign in ("lpt", "static") else "lpt",
                          measure_phase=(lambda *a: None) if two_phase else None)
    ev.world, ev.rank = world, 0
    if cut_of is not None:
        ev.cut_s = lambda: cut_of(min(ev.known.values())) if ev.known else 0.0
    if assign in ("dynamic", "auto") and world > 1:
        ev.assign = assign
    rec, rec_cost, rec_p1 = {}, {}, {}
    for k, (rs, rt) in enumerate(zip(round_states, round_times)):
        ph = round_phase1[k] if round_phase1 is not None and k < len(round_phase1) else None
        for j, (s, t) in enumerate(zip(rs, rt)):
            rec.setdefault(s, t)
            rec_cost.setdefault(s, round_costs[k][j])
            if ph is not None and len(ph[0]):
                rec_p1.setdefault(s, ph[0][j])
    allt = sorted(t for rt in round_times for t in rt)
    med = allt[len(allt) // 2] if allt else 0.0
    allc = sorted(rec_cost.values())
    med_c = allc[len(allc) // 2] if allc else 0.0
    allp = sorted(rec_p1.values())
    med_p1 = allp[len(allp) // 2] if allp else med / 11
    # per-launch overhead of the recorded run (the evaluator's calibration rule over every round)
    est = ShardedEvaluator(measure_set=lambda st, mi: None)
    if cut_of is not None:
        est.cut_s = lambda: cut_of(est._best) if math.isfinite(est._best) else 0.0
    for k, rs in enumerate(round_states):
        c_ = est.cut_s() if est.cut_s is not None else 0.0
        est._calibrate(list(round_costs[k]), list(round_times[k]), est._best, c_)
        for s, c in zip(rs, round_costs[k]):
            est._remember(s, c)
    o_est = est._over

    def t_of(s):
        """Seconds of a speculative (round-0) measurement: its cold probe with a phase measurer
        (the recorded phase-1 seconds, else the median), else the whole measurement, which in
        round 0 has no incumbent to race against: 11 launches of (cost + overhead)."""
        if spec_time is not None:
            return spec_time(s)
        if two_phase:
            return rec_p1.get(s, med_p1)
        return _FULL_LAUNCHES * (rec_cost.get(s, med_c) + o_est)

    def lpt_busy(owner, times):
        busy = [0.0] * world
        for j, r in enumerate(owner):
            if r is not None:
                busy[r] += times[j]
        return max(busy)

    wall = host = 0.0
    modes = []
    for k, states in enumerate(round_states):
        t0 = time.perf_counter()
        cut = ev.cut_s() if ev.cut_s is not None else 0.0
        best = min(ev.known.values()) if ev.known else math.inf
        hit, todo, sub, wts, mode, owner, spec, spec_owner = ev.plan(list(states))
        host += time.perf_counter() - t0
        modes.append(mode)
        times = [round_times[k][j] for j in todo]
        if mode == "two-phase":
            ph = round_phase1[k] if round_phase1 is not None and k < len(round_phase1) else None
            if ph is not None and len(ph[0]):
                t1 = [ph[0][j] for j in todo]
                probes = [ph[1][j] for j in todo]
                final = [bool(ph[2][j]) for j in todo]
            else:
                cs = [round_costs[k][j] for j in todo]
                nl = [ev.launches(c, best, cut) for c in cs]
                t1 = [t / n for t, n in zip(times, nl)]
                probes = cs
                final = [n == 1 for n in nl]
            for j, s in enumerate(sub):
                if owner[j] is None:                        # probe taken speculatively in round 0
                    ev.probe_cache.pop(s)
                    ev.spec_used += 1
            t0 = time.perf_counter()
            ev.calibrate_probes(probes, [0.0 if owner[j] is None else t1[j] for j in range(len(sub))])
            owner2, _ = ev.phase2_plan(probes, final, cut)
            host += time.perf_counter() - t0
            t2 = [t - a for t, a in zip(times, t1)]
            wall += lpt_busy(owner, t1) + lpt_busy(owner2, t2) + (2 * per_round_s if world > 1 else 0.0)
        else:
            busy = [0.0] * world
            if owner is None:                               # dynamic claims in LPT order
                for j in sorted(range(len(sub)), key=lambda j: (-wts[j], j)):
                    r = min(range(world), key=lambda i: busy[i])
                    busy[r] += times[j] + per_claim_s
                for s in spec:
                    r = min(range(world), key=lambda i: busy[i])
                    busy[r] += t_of(s) + per_claim_s
            else:
                for j, r in enumerate(owner):
                    busy[r] += times[j]
                for s, r in zip(spec, spec_owner):
                    busy[r] += t_of(s)
            wall += max(busy) + (per_round_s if world > 1 else 0.0)
        for j, s in enumerate(states):
            if hit[j]:
                ev.cache.pop(s)
                ev.spec_used += 1
        ev.absorb(list(states), list(round_costs[k]), spec, [1.0] * len(spec),
                  secs=[0.0 if hit[j] else round_times[k][j] for j in range(len(states))], cut=cut,
                  spec_final=[not two_phase] * len(spec))
    return {"wall_s": wall, "plan_host_s": host, "spec_measured": ev.spec_measured, "spec_used": ev.spec_used,
            "modes": modes}


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
