"""Actor / critic networks of N-A2C (oracle; test infra only).

PAPER.md P:284: "both actor and critic initialize their neural networks with random weights";
P:327 "Train actor's and critic's neural networks with M".  The architecture, initialisation
and optimiser are unspecified (reading Z18); SPEC S:332-334 defaults are used:

  * two hidden layers of ``hidden`` (64) tanh units; actor head = masked softmax over the
    |A| = 26 actions, critic head = one linear unit;
  * W ~ U(+-sqrt(6/(fan_in+fan_out))) drawn row-major ([out][in]) from a SplitMix64 stream,
    biases 0; init order: actor W1, W2, W3 then critic W1, W2, W3;
  * plain SGD, gradient clipped to global L2 norm ``clip`` (1.0) per network.

float64 throughout.  Every sum is written as the plain left-to-right sum of its definition
(index order, starting from 0.0; a bias is added after the weighted sum; a batch gradient is
accumulated sample by sample), and tanh / exp / log are the C library's (``math``), so the
values are a fixed function of the inputs that any implementation summing in the same order
reproduces bit for bit (reading Z24).  Arrays only vectorise over the
*non-reduced* index; numpy's own reductions (pairwise sums, BLAS) are not used.
Pinned by central finite differences in the tests.
"""
from __future__ import annotations

import math
from typing import List, Optional, Sequence

import numpy as np

_tanh = np.frompyfunc(math.tanh, 1, 1)


def _affine(H: np.ndarray, W: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Z[:, r] = (sum_{c ascending} H[:, c] W[r, c]) + b[r]."""
    Z = np.zeros((H.shape[0], W.shape[0]))
    for c in range(W.shape[1]):
        Z = Z + H[:, c:c + 1] * W[None, :, c]
    return Z + b[None, :]


def seq_sum(values: np.ndarray, axis: int = 0) -> np.ndarray:
    """Left-to-right sum along ``axis`` (np.cumsum accumulates sequentially; 0.0 + x = x)."""
    values = np.asarray(values, dtype=float)
    if values.shape[axis] == 0:
        return np.zeros(np.delete(values.shape, axis))
    return np.take(np.cumsum(values, axis=axis), -1, axis=axis)


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
        acts = [np.asarray(X, dtype=float)]
        h = acts[0]
        L = len(self.W)
        for l in range(L):
            z = _affine(h, self.W[l], self.b[l])
            h = _tanh(z).astype(float) if l < L - 1 else z
            acts.append(h)
        return h, acts

    def backward(self, acts, dout: np.ndarray):
        """Gradients of sum_b <dout_b, out_b> w.r.t. every parameter (no averaging here),
        accumulated over the samples in batch order."""
        L = len(self.W)
        B = dout.shape[0]
        gW = [np.zeros_like(w) for w in self.W]
        gb = [np.zeros_like(b) for b in self.b]
        d = np.asarray(dout, dtype=float)
        for l in range(L - 1, -1, -1):
            gb[l] = seq_sum(d)                                   # sample by sample, batch order
            gW[l] = seq_sum(d[:, :, None] * acts[l][:, None, :])
            if l > 0:
                dn = np.zeros((B, self.W[l].shape[1]))
                for r in range(self.W[l].shape[0]):          # (d W)[:, c] = sum_r d[:, r] W[r, c]
                    dn = dn + d[:, r:r + 1] * self.W[l][None, r, :]
                d = dn * (1.0 - acts[l] * acts[l])           # tanh' = 1 - tanh^2
        return gW, gb

    def sgd_step(self, gW, gb, lr: float, clip: Optional[float]):
        flat = np.concatenate([np.ravel(g) for g in list(gW) + list(gb)])   # weights, then biases
        norm = math.sqrt(float(seq_sum(flat * flat)))
        scale = 1.0
        if clip is not None and clip > 0 and norm > clip:
            scale = clip / norm
        for l in range(len(self.W)):
            self.W[l] = self.W[l] - lr * scale * gW[l]
            self.b[l] = self.b[l] - lr * scale * gb[l]
        return norm


def masked_softmax(z: np.ndarray, mask: np.ndarray) -> np.ndarray:
    """Softmax over entries with mask True (max-subtracted); masked entries exactly 0."""
    out = np.zeros(len(z))
    if not np.any(mask):
        return out
    mx = max(float(z[i]) for i in range(len(z)) if mask[i])
    tot = 0.0
    for i in range(len(z)):
        if mask[i]:
            out[i] = math.exp(float(z[i]) - mx)
            tot += out[i]
    return out / tot
