"""SplitMix64 random stream and the sampling rules of the searches (oracle; test infra only).

The paper only says "randomly select rho states from g(s)" (Alg. 1 line 6 P:250) and
"rand() < epsilon" / "a is randomly selected from A" (Alg. 2).  Reading Z5 / O7
 pins the generator so that library and oracle traverse identically:

  next():  state += 0x9E3779B97F4A7C15
           z = state; z = (z ^ z>>30) * 0xBF58476D1CE4E5B9; z = (z ^ z>>27) * 0x94D049BB133111EB
           return z ^ z>>31                                   (Steele/Lea/Flood SplitMix64)
  bounded(n) = (next() * n) >> 64                             (Lemire multiply-shift, no rejection)
  uniform()  = (next() >> 11) * 2^-53
  sample(L, r): partial Fisher-Yates over idx = [0..L-1]: for t < r: j = t + bounded(L - t),
                swap idx[t], idx[j]; emit idx[0..r) in t order.
"""
from __future__ import annotations

MASK = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


def mix(z: int) -> int:
    """SplitMix64 output function (finaliser)."""
    z &= MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


class SplitMix64:
    def __init__(self, seed: int):
        self.state = seed & MASK

    def next(self) -> int:
        self.state = (self.state + GAMMA) & MASK
        return mix(self.state)

    def bounded(self, n: int) -> int:
        return (self.next() * n) >> 64

    def uniform(self) -> float:
        return (self.next() >> 11) * (1.0 / 9007199254740992.0)

    def sample_indices(self, length: int, r: int):
        """r distinct indices of range(length), uniformly without replacement (reading Z5)."""
        r = min(r, length)
        idx = list(range(length))
        for t in range(r):
            j = t + self.bounded(length - t)
            idx[t], idx[j] = idx[j], idx[t]
        return idx[:r]
