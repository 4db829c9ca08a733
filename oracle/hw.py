"""J_hw: per-family launch limits added to the paper's legitimacy flag (oracle; test infra only).

PAPER.md P:191 (footnote to Eq. 5): "Other constraints can be crafted to limit the search
space and accelerate the search."  Reading Z2/Z3 maps the d = (4,2,4) factors
onto B200 kernel levels and states the limits below.  The table is shared with the CUDA
library *by specification only* (DESIGN.md §4 "J_hw table"); this file is an independent
transcription of that table and imports nothing from the product package.

Families (tt_family in include/tiletune.h):
  0 NONE        J_hw = true
  1 F32_SIMT    fp32 CUDA-core kernel K1
  2 TF32_UMMA   tcgen05 kind::tf32 kernel K2
  3 BF16_UMMA   tcgen05 kind::f16 (bf16) kernel K3
"""
from __future__ import annotations

FAM_NONE, FAM_F32_SIMT, FAM_TF32_UMMA, FAM_BF16_UMMA = 0, 1, 2, 3

# DESIGN.md §4 constants
SMEM_PER_CTA = 232448          # 227 KB opt-in dynamic shared memory per CTA on sm_100
SIMT_SMEM_PAD = 4               # floats of padding per smem tile row (bank-conflict-free stores)
SIMT_MAX_GROUP = 32             # m2*n2 threads form one warp-level thread group
SIMT_MAX_ACC = 128              # m3*n3 fp32 accumulators per thread
SIMT_MAX_REG_DIM = 64           # m3, n3 <= 64 and powers of two (compiled register tiles)
SIMT_MAX_GRID_Y = 65535         # m0 is grid.y
SIMT_STAGES = 2
UMMA_M_ATOM = 128               # m3: UMMA_M per CTA
UMMA_MAX_TMEM_COLS = 512
UMMA_PIPE_SMEM = SMEM_PER_CTA - 2048 - 32768   # barriers/alignment + epilogue staging reserve
UMMA_MIN_STAGES = 2
UMMA_MAX_BK = 256               # TMA box dimension limit


def _elem_bytes(family: int) -> int:
    return 4 if family == FAM_TF32_UMMA else 2


def _umma_k(family: int) -> int:
    return 8 if family == FAM_TF32_UMMA else 16


def simt_max_threads(acc: int) -> int:
    """Threads per CTA allowed for a register tile of ``acc`` = m3*n3 accumulators: the kernel
    instance is compiled with __launch_bounds__ of this size so that threads x registers fits
    the 64K-register file (255 registers at 256 threads)."""
    return 1024 if acc <= 16 else (512 if acc <= 64 else 256)


def umma_stage_bytes(fam: int, s) -> int:
    """Shared memory of one pipeline stage: the A tile (m2*128 rows x k1, K-major) plus the B
    tile (k1 rows x n2*n3/m1 columns, MN-major) rounded up to 1024 B (swizzle-atom alignment)."""
    (m0, m1, m2, m3), (k0, k1), (n0, n1, n2, n3) = s
    elem = _elem_bytes(fam)
    a = m2 * UMMA_M_ATOM * k1 * elem
    b = n2 * (n3 // m1) * k1 * elem
    return a + (b + 1023) // 1024 * 1024


def j_hw(spec, s) -> bool:
    fam = spec.family
    if fam == FAM_NONE:
        return True
    if spec.depths != (4, 2, 4):
        return False
    (m0, m1, m2, m3), (k0, k1), (n0, n1, n2, n3) = s
    if fam == FAM_F32_SIMT:
        threads = m1 * n1 * m2 * n2
        if threads > simt_max_threads(m3 * n3):
            return False
        if m2 * n2 > SIMT_MAX_GROUP:
            return False
        if m3 * n3 > SIMT_MAX_ACC or m3 > SIMT_MAX_REG_DIM or n3 > SIMT_MAX_REG_DIM:
            return False
        if m3 & (m3 - 1) or n3 & (n3 - 1):   # register tiles are compiled for powers of two
            return False
        if m0 > SIMT_MAX_GRID_Y:
            return False
        bm, bn = m1 * m2 * m3, n1 * n2 * n3
        return SIMT_STAGES * (bm + bn + 2 * SIMT_SMEM_PAD) * k1 * 4 <= SMEM_PER_CTA
    if fam in (FAM_TF32_UMMA, FAM_BF16_UMMA):
        elem = _elem_bytes(fam)
        if m3 != UMMA_M_ATOM or m1 not in (1, 2) or m2 not in (1, 2):
            return False
        if n1 not in (1, 2) or n2 not in (1, 2):      # n1 = clusters of n1 pairs sharing A (multicast)
            return False
        if n3 % 16 != 0 or not (16 <= n3 <= 256):
            return False
        nb = n3 // m1                      # B columns per CTA per MMA (cta_group::2 splits N)
        # smallest MN-major B swizzle atom: 32 B for bf16; MN-major tf32 exists only in the
        # 128B-swizzle-with-32B-atoms layout, so a CTA's B columns must span 128 B
        if nb * elem < (128 if fam == FAM_TF32_UMMA else 32):
            return False
        if m2 * n2 * n3 > UMMA_MAX_TMEM_COLS:
            return False
        if k1 % _umma_k(fam) != 0 or k1 > UMMA_MAX_BK:
            return False
        if n3 & (n3 - 1) or k1 & (k1 - 1):   # TMA / UMMA swizzle widths are 32, 64 or 128 B
            return False
        return UMMA_PIPE_SMEM // umma_stage_bytes(fam, s) >= UMMA_MIN_STAGES
    return False


def default_s0(spec):
    """Start state per family.  F32_SIMT / NONE: the paper's untiled s0.  UMMA: the
    untiled s0 is infeasible (m3 must be 128), so a hand-crafted 128x128xBK tile is used
    ("a random or hand-crafted starting state"; reading Z3)."""
    from .space import initial_state
    if spec.family in (FAM_NONE, FAM_F32_SIMT):
        return initial_state(spec)
    bk = 32 if spec.family == FAM_TF32_UMMA else 64
    return ((spec.m // 128, 1, 1, 128), (spec.k // bk, bk), (spec.n // 128, 1, 1, 128))
