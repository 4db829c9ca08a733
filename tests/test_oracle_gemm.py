"""Pins for oracle.gemm (O1), synth (O2 input recipe) and oracle.hw (J_hw table)."""
from fractions import Fraction

import numpy as np
import pytest

import synth
from oracle import gemm, hw, space
from oracle.space import Spec


def _rand(m, n, seed):
    return synth.uniform_f32(seed, m, n)


# ------------------------------------------------------------------ O1 double reference
def test_identity_and_permutation():
    B = _rand(48, 40, 2)
    I = np.eye(48)
    assert np.array_equal(gemm.gemm_f64(I, B), B.astype(np.float64))          # pin 1
    perm = np.random.default_rng(0).permutation(48)
    P = np.eye(48)[perm]
    assert np.array_equal(gemm.gemm_f64(P, B), B.astype(np.float64)[perm])   # pin 2
    assert np.array_equal(gemm.gemm_fmaf(I.astype(np.float32), B), B)
    assert np.array_equal(gemm.gemm_fmaf(P.astype(np.float32), B), B[perm])


def test_rank1_integers_and_ones():
    rng = np.random.default_rng(3)
    u, v = rng.integers(-2, 3, 33), rng.integers(-2, 3, 70)
    w, z = rng.integers(-2, 3, 70), rng.integers(-2, 3, 21)
    A, B = np.outer(u, v).astype(np.float64), np.outer(w, z).astype(np.float64)
    exact = np.outer(u, z) * int(v @ w)                                      # pin 3: u (v^T w) z^T
    assert np.array_equal(gemm.gemm_f64(A, B), exact)
    assert np.array_equal(gemm.gemm_fmaf(A.astype(np.float32), B.astype(np.float32)), exact.astype(np.float32))
    K = 1000
    ones = gemm.gemm_fmaf(np.ones((5, K), np.float32), np.ones((K, 7), np.float32))
    assert (ones == K).all()                                                 # pin 4


def test_matches_numpy_float64():
    A, B = _rand(70, 130, 1).astype(np.float64), _rand(130, 50, 2).astype(np.float64)
    R = gemm.gemm_f64(A, B)
    assert gemm.normwise_error(R, A @ B) < 1e-12                              # pin 5


def _round_f32(x: Fraction) -> np.float32:
    """Correctly rounded (nearest-even) float32 of an exact rational, by bracketing."""
    f = np.float32(float(x))
    lo, hi = (np.nextafter(f, np.float32(-np.inf)), f) if Fraction(float(f)) > x else (f, np.nextafter(f, np.float32(np.inf)))
    if Fraction(float(lo)) <= x <= Fraction(float(hi)) and lo != hi:
        dl, dh = x - Fraction(float(lo)), Fraction(float(hi)) - x
        if dl < dh:
            return lo
        if dh < dl:
            return hi
        return lo if (lo.view(np.uint32) & 1) == 0 else hi
    return f


def test_fmaf_exact_rational_bruteforce():
    # fmaf(a, b, c) = round_f32(a*b + c) exactly; brute force with rationals on a tiny case
    A, B = _rand(3, 17, 5), _rand(17, 4, 6)
    C = gemm.gemm_fmaf(A, B)
    for i in range(3):
        for j in range(4):
            acc = np.float32(0.0)
            for l in range(17):
                acc = _round_f32(Fraction(float(A[i, l])) * Fraction(float(B[l, j])) + Fraction(float(acc)))
            assert acc == C[i, j]


def test_fmaf_within_fp32_bound():
    A, B = _rand(64, 4096, 1), _rand(4096, 32, 2)
    err = gemm.normwise_error(gemm.gemm_fmaf(A, B), gemm.gemm_f64(A, B))
    assert err < 1e-4                                                          # pin 6 (fp32 1e-4)


def test_rows_and_entries_match_full():
    A, B = _rand(40, 64, 1).astype(np.float64), _rand(64, 24, 2).astype(np.float64)
    R = gemm.gemm_f64(A, B)
    rows = [0, 7, 39]
    assert np.array_equal(gemm.gemm_f64_rows(A, B, rows), R[rows])
    ii, jj = np.array([0, 5, 39]), np.array([23, 0, 11])
    assert np.array_equal(gemm.gemm_f64_entries(A, B, ii, jj), R[ii, jj])


# ------------------------------------------------------------------ O2 generator recipe
def test_generator_grid_range_and_shards():
    X = synth.uniform_f32(1, 256, 512)
    assert X.min() >= -1.0 and X.max() < 1.0
    assert np.array_equal(X * 2 ** 23, np.round(X * 2 ** 23))                  # on the 2^-23 grid
    hist, _ = np.histogram(X, bins=16, range=(-1, 1))
    assert (abs(hist - X.size / 16) < 5 * np.sqrt(X.size / 16)).all()          # uniform
    assert abs(float(X.mean())) < 0.01
    assert np.array_equal(synth.uniform_f32(1, 64, 512, row0=100), X[100:164])  # global-index shards
    assert not np.array_equal(synth.uniform_f32(2, 256, 512), X)


def test_bf16_rne_matches_torch():
    import torch
    X = synth.uniform_f32(2, 64, 300)
    bits = synth.to_bf16_bits(X)
    ref = torch.from_numpy(X).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(bits, ref)
    # tie case: 1 + 2^-8 is halfway between bf16 neighbours 1 and 1 + 2^-7 -> even (1.0)
    t = np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8], np.float32)
    assert list(synth.bf16_bits_to_f32(synth.to_bf16_bits(t))) == [1.0, 1.0 + 2 ** -6]


# ------------------------------------------------------------------ J_hw table
def test_jhw_simt_boundaries():
    sp = Spec(512, 512, 512, family=hw.FAM_F32_SIMT)
    assert space.legitimate(sp, space.initial_state(sp))                       # untiled s0 feasible
    good = ((4, 2, 8, 8), (64, 8), (4, 4, 4, 8))                               # 128x128 tile, 256 thr
    assert space.legitimate(sp, good)
    assert not space.legitimate(sp, ((1, 2, 16, 16), (64, 8), (2, 4, 16, 4)))  # lanes 16*16 > 32
    assert not space.legitimate(sp, ((1, 32, 2, 8), (64, 8), (2, 16, 16, 1)))  # 32*16*2*16 threads > 1024
    assert space.legitimate(sp, ((4, 2, 4, 16), (64, 8), (4, 4, 4, 8)))       # m3*n3 = 128 allowed
    assert not space.legitimate(sp, ((4, 2, 4, 16), (64, 8), (2, 4, 4, 16)))  # m3*n3 = 256 > 128
    assert space.legitimate(sp, ((4, 2, 4, 16), (64, 8), (8, 4, 8, 2)))
    assert not space.legitimate(sp, ((1, 1, 1, 512), (512, 1), (512, 1, 1, 1)))  # m3 > 64
    # smem: 2*(BM+BN)*BK*4 <= 232448: BM=BN=1, BK=512 -> 8192 ok; BM=512, BN=512, BK=32 -> 262144 no
    assert not space.legitimate(sp, ((1, 8, 4, 16), (16, 32), (1, 8, 4, 16)))


def test_jhw_umma_boundaries():
    sp = Spec(4096, 4096, 4096, family=hw.FAM_BF16_UMMA)
    s0 = hw.default_s0(sp)
    assert s0 == ((32, 1, 1, 128), (64, 64), (32, 1, 1, 128)) and space.legitimate(sp, s0)
    assert not space.legitimate(sp, space.initial_state(sp))                   # untiled s0 infeasible
    assert space.legitimate(sp, ((8, 2, 2, 128), (64, 64), (16, 1, 1, 256)))   # 2-CTA, 256x256 per CTA
    assert not space.legitimate(sp, ((8, 2, 2, 128), (16, 256), (16, 1, 1, 256)))  # 1 stage only
    assert not space.legitimate(sp, ((16, 1, 2, 128), (64, 64), (4, 1, 4, 256)))   # n2 = 4
    assert not space.legitimate(sp, ((16, 2, 1, 128), (64, 64), (256, 1, 1, 16)))  # 2-CTA N=16: 8 cols < 32 B
    assert not space.legitimate(sp, ((32, 1, 1, 128), (512, 8), (32, 1, 1, 128)))  # BK % 16
    tf = Spec(2048, 2048, 2048, family=hw.FAM_TF32_UMMA)
    assert space.legitimate(tf, hw.default_s0(tf))
    assert space.legitimate(tf, ((16, 1, 1, 128), (256, 8), (64, 1, 1, 32)))
    assert not space.legitimate(tf, ((16, 1, 1, 128), (256, 8), (128, 1, 1, 16)))  # tf32 MN-major needs 128 B
    assert not space.legitimate(tf, ((8, 2, 1, 128), (256, 8), (64, 1, 1, 32)))    # 2-CTA: 16 cols = 64 B
    assert not space.legitimate(tf, ((16, 1, 1, 128), (2048, 1), (128, 1, 1, 16)))


def test_jhw_requires_d424():
    sp = Spec(64, 64, 64, 2, 2, 2, family=hw.FAM_F32_SIMT)
    assert not space.legitimate(sp, ((64, 1), (64, 1), (64, 1)))
