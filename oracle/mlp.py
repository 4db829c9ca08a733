"""Actor / critic networks of N-A2C (oracle; test infra only).

PAPER.md P:284: "both actor and critic initialize their neural networks with random weights";
P:327 "Train actor's and critic's neural networks with M".  The architecture, initialisation
and optimiser are unspecified (reading Z18); SPEC S:332-334 defaults are used:

  * two hidden layers of ``hidden`` (64) tanh units; actor head = masked softmax over the
    |A| = 26 actions, critic head = one linear unit;
  * W ~ U(+-sqrt(6/(fan_in+fan_out))) drawn row-major ([out][in]) from a SplitMix64 stream,
    biases 0; init order: actor W1, W2, W3 then critic W1, W2, W3;
  * plain SGD, gradient clipped to global L2 norm ``clip`` (1.0) per network.

Plain numpy in float64.  Pinned by central finite differences in the tests.
"""
from __future__ import annotations

import math
from typing import List, Optional, Sequence

import numpy as np


class Mlp:
    def __init__(self, sizes: Sequence[int], rng=None):
        self.sizes = list(sizes)
        self.W: List[np.ndarray] = []
        self.b: List[np.ndarray] = []
        for fi, fo in zip(self.sizes[:-1], self.sizes[1:]):
            w = np.zeros((fo, fi))
            if rng is not None:
                lim = math.sqrt(6.0 / (fi + fo))
                for o in range(fo):
                    for i in range(fi):
                        w[o, i] = (2.0 * rng.uniform() - 1.0) * lim
            self.W.append(w)
            self.b.append(np.zeros(fo))

    def n_params(self) -> int:
        return sum(w.size + b.size for w, b in zip(self.W, self.b))

    # forward over a batch X [B, in]; returns output (pre-head) and activation cache
    def forward(self, X: np.ndarray):
        acts = [X]
        h = X
        L = len(self.W)
        for l in range(L):
            z = h @ self.W[l].T + self.b[l]
            h = np.tanh(z) if l < L - 1 else z
            acts.append(h)
        return h, acts

    def backward(self, acts, dout: np.ndarray):
        """Gradients of sum_b <dout_b, out_b> w.r.t. every parameter (no averaging here)."""
        L = len(self.W)
        gW = [None] * L
        gb = [None] * L
        d = dout
        for l in range(L - 1, -1, -1):
            gW[l] = d.T @ acts[l]
            gb[l] = d.sum(axis=0)
            if l > 0:
                d = (d @ self.W[l]) * (1.0 - acts[l] ** 2)   # tanh' = 1 - tanh^2
        return gW, gb

    def sgd_step(self, gW, gb, lr: float, clip: Optional[float]):
        norm = math.sqrt(sum(float((g * g).sum()) for g in gW) + sum(float((g * g).sum()) for g in gb))
        scale = 1.0
        if clip is not None and norm > clip:
            scale = clip / norm
        for l in range(len(self.W)):
            self.W[l] -= lr * scale * gW[l]
            self.b[l] -= lr * scale * gb[l]
        return norm


def masked_softmax(z: np.ndarray, mask: np.ndarray) -> np.ndarray:
    """Softmax over entries with mask True (max-subtracted); masked entries exactly 0."""
    out = np.zeros_like(z)
    if not mask.any():
        return out
    zz = z[mask]
    e = np.exp(zz - zz.max())
    out[mask] = e / e.sum()
    return out
