"""Cost aggregation over repeated trials (oracle; test infra only).

PAPER.md P:369: "the computation time for each configuration is the arithmetic mean for 10
repeated trials".  The north star asks for a median of repeats; reading Z10 reports
cost = median of the R per-repeat means (mean of the two middle values for even R) and also
mean, min and the sample standard deviation (0 when R = 1).  Pinned by injected samples
("fake clock").
"""
from __future__ import annotations

import math
from typing import Sequence


def aggregate(per_repeat: Sequence[float]) -> dict:
    xs = sorted(float(x) for x in per_repeat)
    R = len(xs)
    if R == 0:
        raise ValueError("no repeats")
    med = xs[R // 2] if R % 2 else 0.5 * (xs[R // 2 - 1] + xs[R // 2])
    mean = sum(per_repeat) / R
    sd = math.sqrt(sum((x - mean) ** 2 for x in per_repeat) / (R - 1)) if R > 1 else 0.0
    return {"cost": med, "mean": mean, "min": xs[0], "stdev": sd, "repeats": R}


def number_for(probe_s: float, min_repeat_s: float) -> int:
    """Launches per repeat so that one repeat lasts >= min_repeat_s (reading Z11)."""
    if probe_s <= 0:
        return 1
    return max(1, int(math.ceil(min_repeat_s / probe_s)))


def is_slow(probe_s: float, cut_s: float) -> bool:
    """Reading Z12: a candidate whose single probe exceeds the cut is scored by the probe."""
    return cut_s > 0 and probe_s > cut_s
