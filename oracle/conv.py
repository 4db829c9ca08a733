"""Convolution layer reference (oracle; test infra only).  PAPER.md P:105: a Conv layer "can be
computed with matrix multiplication after rearranging data in a matrix format".  The oracle is the
direct definition (oracle_conv2d_f64 in gemm_ref.c), not the rearrangement."""
from __future__ import annotations

import ctypes

import numpy as np

from . import gemm as _g


def conv2d_f64(x: np.ndarray, w: np.ndarray, stride: int = 1, pad: int = 0) -> np.ndarray:
    """x [Nb, C, H, W], w [F, C, R, S] -> y [Nb, F, P, Q] in double."""
    lib = _g._load()
    f = lib.oracle_conv2d_f64
    I, P_ = ctypes.c_int64, ctypes.c_void_p
    f.argtypes = [I] * 9 + [P_, P_, P_]
    x = np.ascontiguousarray(x, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    Nb, C, H, W = x.shape
    F, C2, R, S = w.shape
    assert C == C2
    P = (H + 2 * pad - R) // stride + 1
    Q = (W + 2 * pad - S) // stride + 1
    y = np.empty((Nb, F, P, Q), dtype=np.float64)
    f(Nb, C, H, W, F, R, S, stride, pad, _g._p(x), _g._p(w), _g._p(y))
    return y


def im2col_ref(x: np.ndarray, R: int, S: int, stride: int = 1, pad: int = 0) -> np.ndarray:
    """The rearrangement of P:105 written out: row (n, p, q), column (c, r, s), zero outside."""
    Nb, C, H, W = x.shape
    P = (H + 2 * pad - R) // stride + 1
    Q = (W + 2 * pad - S) // stride + 1
    A = np.zeros((Nb * P * Q, C * R * S), dtype=x.dtype)
    for n in range(Nb):
        for p in range(P):
            for q in range(Q):
                row = (n * P + p) * Q + q
                for c in range(C):
                    for r in range(R):
                        for s in range(S):
                            ih, iw = p * stride - pad + r, q * stride - pad + s
                            if 0 <= ih < H and 0 <= iw < W:
                                A[row, (c * R + r) * S + s] = x[n, c, ih, iw]
    return A


def kernel_matrix(w: np.ndarray) -> np.ndarray:
    """Each kernel as a column: Wm[(c R + r) S + s, f] = w[f, c, r, s]."""
    F = w.shape[0]
    return np.ascontiguousarray(w.reshape(F, -1).T)
