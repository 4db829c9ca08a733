"""Seeded synthetic operands shared by the oracle tests and the product's host-buffer path.

This module holds none of the method's arithmetic (no GEMM, no search, no tiling): it is
only the counter-based input recipe of DESIGN.md §5 (reading O2), written in numpy.  The
CUDA library implements the same recipe independently (kernel K4, ``tt_fill_uniform``); the
tests check the two agree bit for bit.

Recipe for matrix X with seed sigma (A: 1, B: 2) at logical row-major index idx:
  z = SplitMix64 finaliser of (sigma * 0x9E3779B97F4A7C15 + (idx + 1) * 0xD1B54A32D192ED03) mod 2^64
  u = z >> 40                      (24 bits)
  x = (u - 2^23) * 2^-23           in [-1, 1), exactly representable in fp32
  bf16 operands: x_bf = round-to-nearest-even of x to bfloat16.
Row shards use global indices, so a shard is bit-identical to the rows of the full matrix.
"""
from .generator import SEED_A, SEED_B, uniform_f32, to_bf16_bits, bf16_bits_to_f32  # noqa: F401
