"""Deterministic cost sources for table-driven search parity (oracle; test infra only).

T1 -- SPEC S:172-180 synthetic landscape:  cost = 1 + sum_{x,i} w_{x,i} (log2 s_x[i] - c_{x,i})^2.
      The 64^3 preset uses targets m (2,2,1,1), k (3,3), n (2,2,1,1) and unit weights.
T2 -- the "randomly generated reward function" of Fig. 5(c)/6(c), made
      reproducible (reading O11): cost = 1 + 2^-53 * (mix((seed_T << 32 ^ rank) + GAMMA) >> 11),
      i.e. the first SplitMix64 output of a stream seeded with (seed_T << 32) xor rank(s).
"""
from __future__ import annotations

import math

from . import space
from .rng import SplitMix64

PRESET_64 = ((2.0, 2.0, 1.0, 1.0), (3.0, 3.0), (2.0, 2.0, 1.0, 1.0))


def t1_cost(s, targets=PRESET_64, weights=None) -> float:
    c = 1.0
    for a in range(3):
        for i, f in enumerate(s[a]):
            w = 1.0 if weights is None else weights[a][i]
            d = math.log2(f) - targets[a][i]
            c += w * d * d
    return c


def t2_cost(spec, s, seed_t: int = 7) -> float:
    r = space.rank(spec, s)
    g = SplitMix64(((seed_t << 32) ^ r))
    return 1.0 + (g.next() >> 11) * (1.0 / 9007199254740992.0)


def table(spec, fn) -> list:
    """Cost indexed by rank over the whole raw space (J_prod); infeasible states get +inf."""
    out = []
    for s in space.enumerate_configs(spec):
        out.append(fn(s) if space.legitimate(spec, s) else math.inf)
    return out
