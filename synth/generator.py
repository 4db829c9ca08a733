"""Counter-based U[-1,1) operand generator (see package docstring)."""
from __future__ import annotations

import numpy as np

SEED_A = 1
SEED_B = 2
_G = np.uint64(0x9E3779B97F4A7C15)
_H = np.uint64(0xD1B54A32D192ED03)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def _finalise(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _C1
    z = (z ^ (z >> np.uint64(27))) * _C2
    return z ^ (z >> np.uint64(31))


def uniform_f32(seed: int, rows: int, cols: int, row0: int = 0, chunk: int = 1 << 22) -> np.ndarray:
    """fp32 [rows, cols] block of the matrix with ``seed`` whose first row is global row ``row0``
    (row-major, ``cols`` columns in the full matrix)."""
    n = rows * cols
    out = np.empty(n, dtype=np.float32)
    base = np.uint64((int(seed) * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF)
    start = row0 * cols
    with np.errstate(over="ignore"):
        for s in range(0, n, chunk):
            e = min(n, s + chunk)
            idx = np.arange(start + s + 1, start + e + 1, dtype=np.uint64)
            z = _finalise(base + idx * _H)
            u = (z >> np.uint64(40)).astype(np.int64) - (1 << 23)
            out[s:e] = u.astype(np.float32) * np.float32(2.0 ** -23)
    return out.reshape(rows, cols)


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit patterns (uint16).  Inputs are finite."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))
    return (u >> np.uint64(16)).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32)
