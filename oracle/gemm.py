"""ctypes front for oracle/gemm_ref.c (oracle; test infra only).  See gemm_ref.c for the
definition and citations.  ``build()`` compiles the shared object with gcc; it is also built
lazily on first use."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "gemm_ref.c")
LIB = os.path.join(HERE, "_gemm_ref.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O3", "-mavx2", "-mfma", "-ffp-contract=off", "-fopenmp",
                               "-shared", "-fPIC", SRC, "-o", LIB, "-lm"])
    return LIB


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(LIB)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        _lib.oracle_gemm_f64.argtypes = [I, I, I, P, P, P]
        _lib.oracle_gemm_fmaf.argtypes = [I, I, I, P, P, P]
        _lib.oracle_gemm_f64_rows.argtypes = [I, I, P, P, P, I, P]
        _lib.oracle_gemm_f64_entries.argtypes = [I, I, P, P, P, P, I, P]
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def gemm_f64(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """R = A.B in double, sequential k (O1)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    m, k = A.shape
    k2, n = B.shape
    assert k == k2
    C = np.empty((m, n), dtype=np.float64)
    _load().oracle_gemm_f64(m, n, k, _p(A), _p(B), _p(C))
    return C


def gemm_fmaf(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """C = A.B as one sequential fmaf chain per entry in float (O1 secondary mode)."""
    A = np.ascontiguousarray(A, dtype=np.float32)
    B = np.ascontiguousarray(B, dtype=np.float32)
    m, k = A.shape
    _, n = B.shape
    C = np.empty((m, n), dtype=np.float32)
    _load().oracle_gemm_fmaf(m, n, k, _p(A), _p(B), _p(C))
    return C


def gemm_f64_rows(A: np.ndarray, B: np.ndarray, rows) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    k, n = B.shape
    out = np.empty((len(rows), n), dtype=np.float64)
    _load().oracle_gemm_f64_rows(n, k, _p(A), _p(B), _p(rows), len(rows), _p(out))
    return out


def gemm_f64_entries(A: np.ndarray, B: np.ndarray, ii, jj) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    ii = np.ascontiguousarray(ii, dtype=np.int64)
    jj = np.ascontiguousarray(jj, dtype=np.int64)
    k, n = B.shape
    out = np.empty(len(ii), dtype=np.float64)
    _load().oracle_gemm_f64_entries(n, k, _p(A), _p(B), _p(ii), _p(jj), len(ii), _p(out))
    return out


def normwise_error(C: np.ndarray, R: np.ndarray) -> float:
    """Reading Z15: max_ij |C_ij - R_ij| / max_ij |R_ij|."""
    den = float(np.max(np.abs(R)))
    return float(np.max(np.abs(C.astype(np.float64) - R))) / (den if den > 0 else 1.0)
