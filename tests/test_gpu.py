"""GPU parity of the CUDA path (through the C-ABI) against the oracle.  Run with -m gpu on a B200.

Tolerances (north star; reading Z15 normwise max|C - R| / max|R|): fp32 SIMT bit-exact vs the
sequential fmaf oracle and <= 1e-4 vs double; TF32 / BF16 <= 5e-3 vs double on the operands
the device consumed (bf16-rounded for BF16, reading Z16; fp32 for TF32, reading Z17).
"""
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import synth  # noqa: E402
from oracle import na2c as ona2c, costs, gbfs as ogbfs, gemm as og, hw, space  # noqa: E402
from oracle.rng import SplitMix64  # noqa: E402
from oracle.space import Spec  # noqa: E402
from paper_1909_10616_b200 import tiletune as tt  # noqa: E402

DEV = torch.device("cuda:0")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def host_inputs(M, N, K, bf16=False, row0=0):
    A = synth.uniform_f32(synth.SEED_A, M, K, row0=row0)
    B = synth.uniform_f32(synth.SEED_B, K, N)
    if bf16:
        A = synth.bf16_bits_to_f32(synth.to_bf16_bits(A))
        B = synth.bf16_bits_to_f32(synth.to_bf16_bits(B))
    return A, B


def to_dev(X, bf16=False):
    t = torch.from_numpy(np.ascontiguousarray(X)).to(DEV)
    return t.to(torch.bfloat16) if bf16 else t


def run(fam, cfg, A, B):
    bf16 = fam == tt.FAM_BF16_UMMA
    Ad, Bd = to_dev(A, bf16), to_dev(B, bf16)
    C = torch.full((A.shape[0], B.shape[1]), float("nan"), device=DEV)
    tt.gemm(Ad, Bd, C, fam, cfg)
    torch.cuda.synchronize()
    return C.cpu().numpy()


# ------------------------------------------------------------------ K4 generator
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_generator_bit_exact(dtype):
    n, idx0 = 1 << 20, 12345
    t = torch.empty(n, device=DEV, dtype=torch.float32 if dtype == "f32" else torch.bfloat16)
    tt.fill_uniform(t, seed=2, idx0=idx0)
    torch.cuda.synchronize()
    ref = synth.uniform_f32(2, 1, n + idx0)[0, idx0:]
    if dtype == "f32":
        assert np.array_equal(t.cpu().numpy(), ref)
    else:
        got = t.cpu().view(torch.int16).numpy().view(np.uint16)
        assert np.array_equal(got, synth.to_bf16_bits(ref))


# ------------------------------------------------------------------ K1 fp32 SIMT
def _random_feasible(sp, n, seed):
    allst = [s for s in space.enumerate_configs(sp) if space.legitimate(sp, s)]
    r = SplitMix64(seed)
    return [allst[i] for i in r.sample_indices(len(allst), n)]


@pytest.mark.parametrize("dims,n", [((64, 64, 64), 50), ((256, 256, 256), 20), ((256, 128, 64), 20)])
def test_simt_random_configs_bit_exact(dims, n):
    # S:533 acceptance 3: 50 random legitimate configs at 64^3, 20 at 256^3 (+ a non-square shape)
    m, k, nn = dims
    sp = Spec(m, k, nn, family=hw.FAM_F32_SIMT)
    A, B = host_inputs(m, nn, k)
    ref32 = og.gemm_fmaf(A, B)
    R = og.gemm_f64(A, B)
    for s in _random_feasible(sp, n, seed=m + k + nn):
        C = run(tt.FAM_F32_SIMT, s, A, B)
        assert np.array_equal(C, ref32), s
        assert og.normwise_error(C, R) <= 1e-4


def test_simt_fixed_slab_instances_bit_exact():
    # register tiles of <= 32 accumulators with BK in {32, 64, 128} run compile-time-BK instances
    # (gemm_simt.cu kFixed): same fmaf chain, so still bit-identical to the sequential oracle
    m, k, n = 512, 256, 384
    sp = Spec(m, k, n, family=hw.FAM_F32_SIMT)
    A, B = host_inputs(m, n, k)
    ref32 = og.gemm_fmaf(A, B)
    picked = [s for s in (c for c in space.enumerate_configs(sp) if space.legitimate(sp, c))
              if s[1][1] in (32, 64, 128) and (s[0][3], s[2][3]) in ((4, 4), (4, 8), (8, 4))]
    pick = [picked[i] for i in SplitMix64(11).sample_indices(len(picked), 24)]
    assert {s[1][1] for s in pick} == {32, 64, 128}
    for s in pick:
        assert np.array_equal(run(tt.FAM_F32_SIMT, s, A, B), ref32), s


def test_simt_s0_identity_ones_degenerate():
    B = synth.uniform_f32(2, 128, 96)
    I = np.eye(128, dtype=np.float32)
    for s in [((128, 1, 1, 1), (128, 1), (96, 1, 1, 1)),        # the paper's untiled s0
              ((2, 2, 8, 4), (16, 8), (3, 2, 4, 4))]:
        assert np.array_equal(run(1, s, I, B), B)                  # pin 1
    ones = run(1, ((2, 2, 8, 4), (16, 8), (2, 1, 4, 4)), np.ones((128, 128), np.float32),
               np.ones((128, 32), np.float32))
    assert (ones == 128).all()                                     # pin 4
    # degenerate shapes: single row / column / k
    for (M, N, K), s in [((1, 64, 32), ((1, 1, 1, 1), (4, 8), (4, 2, 8, 1))),
                         ((64, 1, 16), ((8, 1, 8, 1), (1, 16), (1, 1, 1, 1))),
                         ((32, 32, 1), ((2, 2, 8, 1), (1, 1), (2, 2, 4, 2)))]:
        A, B = host_inputs(M, N, K)
        assert np.array_equal(run(1, s, A, B), og.gemm_fmaf(A, B)), (M, N, K)


def test_simt_large_sampled_rows():
    # full size of the C2/C3 workloads: sampled rows against the oracle, one launch config
    M = N = K = 2048
    A, B = host_inputs(M, N, K)
    s = ((16, 2, 8, 8), (256, 8), (16, 4, 4, 8))
    C = run(1, s, A, B)
    rows = np.array([0, 1, 127, 128, 1023, 2047])
    R = og.gemm_f64_rows(A, B, rows)
    assert og.normwise_error(C[rows], R) <= 1e-4
    assert np.array_equal(C[rows], og.gemm_fmaf(A[rows], B))


# ------------------------------------------------------------------ K2/K3 tcgen05
@pytest.mark.parametrize("fam", [tt.FAM_BF16_UMMA, tt.FAM_TF32_UMMA])
def test_umma_every_feasible_config_512(fam):
    m = 512
    sp = Spec(m, m, m, family=fam)
    bf16 = fam == tt.FAM_BF16_UMMA
    A, B = host_inputs(m, m, m, bf16=bf16)
    R = og.gemm_f64(A, B)
    bad = []
    for s in space.enumerate_configs(sp):
        if not space.legitimate(sp, s):
            continue
        C = run(fam, s, A, B)
        err = og.normwise_error(C, R)
        if not err <= 5e-3:
            bad.append((s, err))
    assert not bad, bad[:5]


def test_umma_non_square_and_identity():
    # (M, N, K) = (512, 256, 1024): several tiles on each axis, K loop of many stages
    M, N, K = 512, 256, 1024
    A, B = host_inputs(M, N, K, bf16=True)
    R = og.gemm_f64(A, B)
    for s in [((4, 1, 1, 128), (16, 64), (2, 1, 1, 128)), ((1, 2, 2, 128), (8, 128), (1, 1, 2, 128)),
              ((2, 2, 1, 128), (64, 16), (8, 1, 1, 32)), ((4, 1, 1, 128), (4, 256), (16, 1, 1, 16))]:
        assert og.normwise_error(run(3, s, A, B), R) <= 5e-3, s
    I = np.eye(256, dtype=np.float32)
    Bq = synth.bf16_bits_to_f32(synth.to_bf16_bits(synth.uniform_f32(2, 256, 256)))
    assert np.array_equal(run(3, ((2, 1, 1, 128), (4, 64), (1, 1, 1, 256)), I, Bq), Bq)      # pin 1, exact
    ones = run(3, ((1, 2, 1, 128), (16, 64), (2, 1, 1, 128)), np.ones((256, 1024), np.float32),
               np.ones((1024, 256), np.float32))
    assert (ones == 1024).all()                                                               # pin 4


def test_tf32_rounding_mode_probe():
    # reading Z17: which TF32 conversion does tcgen05 apply?  A = I, B with low mantissa bits
    I = np.eye(128, dtype=np.float32)
    B = synth.uniform_f32(2, 128, 128)
    C = run(2, ((1, 1, 1, 128), (4, 32), (1, 1, 1, 128)), I, B)
    bits = B.view(np.uint32)
    trunc = (bits & np.uint32(0xFFFFE000)).view(np.float32)
    rna = ((bits + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32)
    mode = "exact" if np.array_equal(C, B) else ("trunc" if np.array_equal(C, trunc) else
                                                  ("rna" if np.array_equal(C, rna) else "other"))
    print("TF32 operand conversion:", mode)
    assert mode in ("trunc", "rna", "exact")


def test_bf16_4096_sampled():
    M = N = K = 4096
    A, B = host_inputs(M, N, K, bf16=True)
    rows = np.array([0, 129, 2048, 4095])
    R = og.gemm_f64_rows(A, B, rows)
    for s in [hw.default_s0(Spec(M, K, N, family=3)), ((16, 1, 2, 128), (64, 64), (16, 1, 1, 256)),
              ((8, 2, 2, 128), (64, 64), (16, 1, 1, 256)), ((16, 2, 1, 128), (32, 128), (32, 1, 1, 128)),
              ((16, 2, 1, 128), (32, 128), (8, 2, 1, 256)), ((16, 1, 2, 128), (64, 64), (8, 2, 1, 256))]:
        C = run(3, s, A, B)
        assert og.normwise_error(C[rows], R) <= 5e-3, s
        ii = np.array([5, 1000, 3000, 4095])
        jj = np.array([4095, 17, 2222, 0])
        assert og.normwise_error(C[ii, jj], og.gemm_f64_entries(A, B, ii, jj)) <= 5e-3


@pytest.mark.parametrize("fam,cfg", [
    (3, ((16, 1, 1, 128), (8, 64), (16, 1, 1, 128))),     # 256 tiles: 108-tile tail over 148 CTAs
    (3, ((8, 2, 1, 128), (8, 64), (8, 1, 1, 256))),       # 64 pair tiles < 74 pairs: all split
    (3, ((4, 2, 2, 128), (16, 32), (8, 1, 2, 128))),      # 2 x 2 atoms per CTA
    (3, ((16, 1, 1, 128), (32, 16), (128, 1, 1, 16))),    # n3 = 16: direct-store epilogue adds
    (2, ((16, 1, 1, 128), (16, 32), (16, 1, 1, 128))),    # tf32
    (2, ((8, 2, 1, 128), (64, 8), (16, 1, 1, 128))),
    (3, ((8, 2, 1, 128), (8, 64), (4, 2, 1, 256))),       # n1 = 2: clusters of two pairs, A multicast
    (2, ((16, 1, 1, 128), (16, 32), (8, 2, 1, 128))),     # n1 = 2 with single-CTA MMAs
])
def test_umma_tail_split(fam, cfg, monkeypatch):
    # DESIGN.md §6 tail split: tiles % co-resident clusters != 0, so the last tiles' k-blocks are
    # shared by up to 4 clusters (TMA store, then descending-k TMA reduce-adds).  Parity vs the
    # double oracle, bit-reproducible across launches and streams (the flags reset themselves).
    # TT_TAIL_SPLIT=2 forces the split on these small shapes (the default policy would not).
    monkeypatch.setenv("TT_TAIL_SPLIT", "2")
    M = N = 2048
    K = 512
    sp = tt.make_space(M, N, K, family=fam)
    info = tt.binding(sp, cfg)
    assert info.split_tiles > 0 and 0 < info.split_workers <= 4 * info.split_tiles
    bf16 = fam == tt.FAM_BF16_UMMA
    A, B = host_inputs(M, N, K, bf16=bf16)
    R = og.gemm_f64(A, B)
    Ad, Bd = to_dev(A, bf16), to_dev(B, bf16)
    outs = []
    s2 = torch.cuda.Stream()
    for stream in (None, None, s2):
        C = torch.full((M, N), float("nan"), device=DEV)
        if stream is None:
            tt.gemm(Ad, Bd, C, fam, cfg)
        else:
            with torch.cuda.stream(stream):
                tt.gemm(Ad, Bd, C, fam, cfg, stream=stream)
        torch.cuda.synchronize()
        outs.append(C.cpu().numpy())
    assert og.normwise_error(outs[0], R) <= 5e-3
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


@pytest.mark.parametrize("fam,cfg", [
    (3, ((16, 1, 1, 128), (8, 64), (16, 1, 1, 128))),     # 256 tiles, 148 clusters: 108 + 148 split
    (3, ((8, 2, 1, 128), (8, 64), (16, 1, 1, 128))),      # 128 pair tiles on 74 pairs: all stream-K
    (3, ((16, 1, 1, 128), (8, 64), (16, 2, 1, 64))),      # n1 = 2 clusters (A multicast): 34 + 74 split
    (2, ((16, 1, 1, 128), (16, 32), (16, 1, 1, 128))),    # tf32
])
def test_umma_wave_remainder_split(fam, cfg, monkeypatch):
    # Round-2 default split shape: the last full wave plus the remainder by
    # stream-K over all clusters.  TT_TAIL_SPLIT=4 forces it at this small K; parity vs the double
    # oracle, bit-reproducible across launches and streams.
    monkeypatch.setenv("TT_TAIL_SPLIT", "4")
    M = N = 2048
    K = 512
    sp = tt.make_space(M, N, K, family=fam)
    info = tt.binding(sp, cfg)
    tiles = cfg[0][0] * cfg[2][0]
    assert info.split_tiles > 0 and info.split_tiles == tiles % info.split_workers + info.split_workers
    bf16 = fam == tt.FAM_BF16_UMMA
    A, B = host_inputs(M, N, K, bf16=bf16)
    R = og.gemm_f64(A, B)
    Ad, Bd = to_dev(A, bf16), to_dev(B, bf16)
    outs = []
    s2 = torch.cuda.Stream()
    for stream in (None, None, s2):
        C = torch.full((M, N), float("nan"), device=DEV)
        if stream is None:
            tt.gemm(Ad, Bd, C, fam, cfg)
        else:
            with torch.cuda.stream(stream):
                tt.gemm(Ad, Bd, C, fam, cfg, stream=stream)
        torch.cuda.synchronize()
        outs.append(C.cpu().numpy())
    assert og.normwise_error(outs[0], R) <= 5e-3
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


# ------------------------------------------------------------------ evaluator and search
def test_measure_and_errors():
    ctx = tt.Context(0)
    sp = tt.make_space(512, 512, 512, family=1)
    ctx.prepare(sp)                                       # one-time setup: operands + kernels loaded
    smp = ctx.measure(sp, ((4, 2, 8, 8), (64, 8), (4, 4, 4, 8)))
    assert smp.cost_s > 0 and smp.repeats == 10 and smp.min_s <= smp.cost_s and smp.number >= 1
    assert smp.number * smp.cost_s >= 4e-4
    with pytest.raises(tt.TileTuneError) as e:
        ctx.measure(sp, ((4, 2, 8, 8), (64, 8), (4, 4, 4, 4)))
    assert e.value.status == tt.E_ILLEGITIMATE
    with pytest.raises(tt.TileTuneError) as e:
        ctx.measure(sp, ((1, 1, 1, 512), (512, 1), (512, 1, 1, 1)))
    assert e.value.status == tt.E_INFEASIBLE
    cut = ctx.measure(sp, space.initial_state(Spec(512, 512, 512)), tt.measure_opts(cut_s=1e-6))
    assert cut.slow_cut in (1, 2) and cut.repeats == 1             # 2: partial-grid estimate (Z12)
    fl = ctx.measure(sp, ((4, 2, 8, 8), (64, 8), (4, 4, 4, 8)), tt.measure_opts(l2_flush=1, repeats=3))
    assert fl.number == 1 and fl.repeats == 3 and fl.graph_nodes == 0


def test_measure_graph_replay():
    # default: repeats replay a captured CUDA graph (device time only); graph=0: host launch loop.
    # On a ~5 us bf16 GEMM the host path (tensor maps, cluster launch) can exceed the kernel, so
    # the graph score must not be slower, and both must agree on a long kernel.
    ctx = tt.Context(0)
    small = tt.make_space(1024, 1024, 1024, family=3)
    cfg = ((8, 1, 1, 128), (8, 128), (16, 1, 1, 64))
    g = ctx.measure(small, cfg)
    d = ctx.measure(small, cfg, tt.measure_opts(graph=0))
    assert g.graph_nodes > 0 and d.graph_nodes == 0 and g.number % g.graph_nodes == 0
    assert g.cost_s <= d.cost_s * 1.05, (g.cost_s, d.cost_s)
    big = tt.make_space(4096, 4096, 4096, family=3)
    cfg = ((16, 2, 1, 128), (32, 128), (16, 1, 1, 256))
    g = ctx.measure(big, cfg, tt.measure_opts(repeats=5))
    d = ctx.measure(big, cfg, tt.measure_opts(repeats=5, graph=0))
    assert abs(g.cost_s / d.cost_s - 1) < 0.05, (g.cost_s, d.cost_s)
    ctx.close()


class _Raw:
    """Expose a raw device pointer to torch (CUDA array interface) without copying."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr, False), "version": 3}


def test_ctx_operands_are_the_recipe():
    ctx = tt.Context(0, input_seed=1)
    a, b, c = ctx.operands(64, 32, 16, tt.FAM_BF16_UMMA)
    torch.cuda.synchronize()
    A = torch.as_tensor(_Raw(a, (64, 16), "<i2"), device=DEV).cpu().numpy().view(np.uint16)
    B = torch.as_tensor(_Raw(b, (16, 32), "<i2"), device=DEV).cpu().numpy().view(np.uint16)
    assert np.array_equal(A, synth.to_bf16_bits(synth.uniform_f32(1, 64, 16)))
    assert np.array_equal(B, synth.to_bf16_bits(synth.uniform_f32(2, 16, 32)))
    ctx.close()


def test_gemm_host_matches_device():
    ctx = tt.Context(0)
    M, N, K = 256, 256, 512
    A, B = host_inputs(M, N, K)
    Ah, Bh = torch.from_numpy(A).pin_memory(), torch.from_numpy(B).pin_memory()
    Ch = torch.empty(M, N).pin_memory()
    s = ((2, 2, 8, 8), (64, 8), (2, 4, 4, 8))      # 2 x 2 blocks of the host pipeline
    ctx.gemm_host(Ah, Bh, Ch, 1, s)
    assert np.array_equal(Ch.numpy(), og.gemm_fmaf(A, B))
    # bf16 tcgen05 through the 2-D block pipeline (4 x 2 blocks, packed B column chunks)
    M, N, K = 1024, 1024, 512
    A, B = host_inputs(M, N, K, bf16=True)
    Ah = torch.from_numpy(synth.to_bf16_bits(A).view(np.int16)).view(torch.bfloat16).pin_memory()
    Bh = torch.from_numpy(synth.to_bf16_bits(B).view(np.int16)).view(torch.bfloat16).pin_memory()
    Ch = torch.full((M, N), float("nan")).pin_memory()
    ctx.gemm_host(Ah, Bh, Ch, 3, ((4, 2, 1, 128), (8, 64), (4, 1, 1, 256)))
    assert og.normwise_error(Ch.numpy(), og.gemm_f64(A, B)) <= 5e-3
    ctx.close()


def test_gbfs_device_search_replay_parity():
    # live G-BFS on the SIMT space of 512^3; replaying its (state -> cost) table through the
    # oracle reproduces the identical sequence of evaluated states (O8 "live-GPU parity by replay")
    ctx = tt.Context(0)
    res = tt.gbfs_search(512, 512, 512, 120, tt.search_opts(family=1, seed=3), ctx=ctx)
    ctx.close()
    assert res.evals == 120 and res.best_cost < res.trace[0]["cost"]
    table = {r["state"]: r["cost"] for r in res.trace}
    sp = Spec(512, 512, 512, family=1)
    o = ogbfs.gbfs(sp, lambda states: [table[s] for s in states], budget=120, rho=5, seed=3)
    assert [r.state for r in o.trace] == [r["state"] for r in res.trace]
    assert res.frac_raw == 120 / 484000


def test_gbfs_two_phase_evaluator_replay_parity():
    # the bench's tuning path: G-BFS (W = 16) with the sharded evaluator, device two-phase rounds
    # (probes, then the rest, tt_measure_phase) on one rank; the traversal replays exactly through
    # the oracle with the recorded costs, and every round with more than one candidate ran in two
    # phases
    from paper_1909_10616_b200 import dist as tdist
    ctx = tt.Context(0)
    sp = tt.make_space(2048, 2048, 2048, family=3)
    sopts = tt.search_opts(family=3, seed=1, width=16, measure={"l2_flush": 1})
    ms, observe, cut, mp = tdist.device_measure_set(ctx, sp, sopts)
    ev = tdist.TrackingEvaluator(observe=observe, measure_set=ms, measure_phase=mp, space=sp, cut_s=cut)
    res = tt.gbfs_search(2048, 2048, 2048, 48, sopts, batch=ev)
    ctx.close()
    assert res.evals == 48
    assert [md == "two-phase" for md in ev.round_modes] == [len(r) > 1 for r in ev.round_states]
    table = {r["state"]: r["cost"] for r in res.trace}
    o = ogbfs.gbfs(Spec(2048, 2048, 2048, family=3), lambda states: [table[s] for s in states], budget=48, rho=5,
                   seed=1, width=16)
    assert [r.state for r in o.trace] == [r["state"] for r in res.trace]


def test_na2c_device_search():
    # live N-A2C (eps = 0.8: policy sampled, networks trained every batch) on the SIMT space of
    # 512^3; replaying its (state -> cost) table through the oracle's Algorithm 2 reproduces the
    # identical sequence of evaluated states (reading Z24 makes the network arithmetic exact)
    ctx = tt.Context(0)
    res = tt.na2c_search(512, 512, 512, 64, tt.search_opts(family=1, seed=1), ctx=ctx)
    ctx.close()
    assert res.evals == 64 and res.best_cost < res.trace[0]["cost"]
    states = [r["state"] for r in res.trace]
    assert len(set(states)) == 64
    table = {r["state"]: r["cost"] for r in res.trace}
    sp = Spec(512, 512, 512, family=1)
    o = ona2c.na2c(sp, lambda batch: [table[s] for s in batch], budget=64, params=ona2c.Params(), seed=1)
    assert [r.state for r in o.trace] == states


def test_bf16_exhaustive_vs_gbfs_4096():
    # every feasible BF16 config at 4096^3 measured once; G-BFS at <= 1% of the raw space must
    # land within 5% of the exhaustive best (reading O10 machine-relative pin)
    ctx = tt.Context(0)
    sp = tt.make_space(4096, 4096, 4096, family=3)
    cfgs, _ = tt.enumerate_feasible(sp)
    mo = tt.measure_opts(repeats=5)
    best = min(ctx.measure(sp, s, mo).cost_s for s in cfgs)
    res = tt.gbfs_search(4096, 4096, 4096, 100, tt.search_opts(family=3, seed=0, measure={"repeats": 5}), ctx=ctx)
    ctx.close()
    assert res.frac_raw <= 0.01
    assert res.best_cost <= best * 1.05, (res.best_cost, best)


# ------------------------------------------------------------------ TN layout (P:372 Y = W^T X)
@pytest.mark.parametrize("fam", [tt.FAM_F32_SIMT, tt.FAM_BF16_UMMA, tt.FAM_TF32_UMMA])
def test_tn_layout_perceptron(fam):
    # the paper's perceptron workload: W in R^(k x m), X in R^(k x n), Y = W^T X;
    # (m, k, n) = (512, 256, 384) non-square so a swapped axis cannot pass
    m, k, n = 512, 256, 384
    bf16 = fam == tt.FAM_BF16_UMMA
    W = synth.uniform_f32(synth.SEED_A, k, m)
    X = synth.uniform_f32(synth.SEED_B, k, n)
    if bf16:
        W = synth.bf16_bits_to_f32(synth.to_bf16_bits(W))
        X = synth.bf16_bits_to_f32(synth.to_bf16_bits(X))
    A = np.ascontiguousarray(W.T)
    R = og.gemm_f64(A, X)
    sp = Spec(m, k, n, family=fam)
    cfgs = [s for s in space.enumerate_configs(sp) if space.legitimate(sp, s)]
    pick = [cfgs[i] for i in SplitMix64(5).sample_indices(len(cfgs), 12)]
    if fam != tt.FAM_F32_SIMT:                         # A multicast (n1 = 2) with MN-major A boxes
        pick += [c for c in cfgs if c[2][1] == 2][:3]
    Wd, Xd = to_dev(W, bf16), to_dev(X, bf16)
    for s in pick:
        C = torch.full((m, n), float("nan"), device=DEV)
        tt.gemm(Wd, Xd, C, fam, s, layout=tt.LAYOUT_TN)
        torch.cuda.synchronize()
        Cn = C.cpu().numpy()
        if fam == tt.FAM_F32_SIMT:
            assert np.array_equal(Cn, og.gemm_fmaf(A, X)), s
        else:
            assert og.normwise_error(Cn, R) <= 5e-3, s


# ------------------------------------------------------------------ conv layer as GEMM
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_im2col_bit_exact(dtype):
    from oracle import conv
    x = synth.uniform_f32(1, 2 * 3 * 9 * 10, 1).reshape(2, 3, 9, 10)
    if dtype == "bf16":
        x = synth.bf16_bits_to_f32(synth.to_bf16_bits(x))
    xd = to_dev(x, dtype == "bf16")
    for (R, S, st, pad) in [(3, 3, 1, 1), (5, 2, 2, 0), (1, 1, 1, 0)]:
        A = tt.im2col(xd, R, S, st, pad)
        torch.cuda.synchronize()
        ref = conv.im2col_ref(x, R, S, st, pad)
        assert np.array_equal(A.float().cpu().numpy(), ref)


@pytest.mark.parametrize("fam", [tt.FAM_F32_SIMT, tt.FAM_BF16_UMMA, tt.FAM_TF32_UMMA])
def test_conv2d_via_gemm(fam):
    # a ResNet-style 3x3 layer: Nb=2, C=64, 16x16, F=128, pad 1 -> GEMM (M, N, K) = (512, 128, 576)
    from oracle import conv
    Nb, C, H, W, F, R, S = 2, 64, 16, 16, 128, 3, 3
    bf16 = fam == tt.FAM_BF16_UMMA
    x = synth.uniform_f32(1, Nb * C * H * W, 1).reshape(Nb, C, H, W)
    w = synth.uniform_f32(2, F * C * R * S, 1).reshape(F, C, R, S)
    if bf16:
        x = synth.bf16_bits_to_f32(synth.to_bf16_bits(x))
        w = synth.bf16_bits_to_f32(synth.to_bf16_bits(w))
    M, N, K = tt.conv_gemm_dims(x.shape, F, R, S, 1, 1)
    assert (M, N, K) == (512, 128, 576)
    sp = Spec(M, K, N, family=fam)
    s = hw.default_s0(sp) if fam != tt.FAM_F32_SIMT else ((4, 2, 8, 8), (72, 8), (1, 4, 4, 8))
    assert space.legitimate(sp, s)
    y = tt.conv2d(to_dev(x, bf16), to_dev(conv.kernel_matrix(w), bf16), fam, s, R, S, 1, 1)
    torch.cuda.synchronize()
    ref = conv.conv2d_f64(x, w, 1, 1)
    got = y.cpu().numpy().reshape(Nb, H, W, F).transpose(0, 3, 1, 2)
    assert og.normwise_error(got, ref) <= (1e-4 if fam == tt.FAM_F32_SIMT else 5e-3)


@pytest.mark.parametrize("M,N,K,s", [
    (8192, 8192, 8192, ((16, 2, 2, 128), (128, 64), (32, 1, 1, 256))),     # bench bf16_8192 config
    (1024, 8192, 8192, ((4, 2, 1, 128), (128, 64), (32, 1, 1, 256))),      # C5 shard at 8 GPUs
    (8192, 8192, 8192, ((16, 2, 2, 128), (128, 64), (32, 1, 2, 128))),     # r13_workloads bf16_8192
    (1024, 8192, 8192, ((2, 2, 2, 128), (128, 64), (32, 1, 2, 128))),      # r13_workloads shard8
])
def test_bf16_max_sizes_sampled(M, N, K, s):
    # BASELINE configs[4] sizes, in the launch configuration bench.py times; sampled entries
    Ab = synth.to_bf16_bits(synth.uniform_f32(synth.SEED_A, M, K))
    Bb = synth.to_bf16_bits(synth.uniform_f32(synth.SEED_B, K, N))
    Ad = torch.from_numpy(Ab.view(np.int16)).to(DEV).view(torch.bfloat16)
    Bd = torch.from_numpy(Bb.view(np.int16)).to(DEV).view(torch.bfloat16)
    C = torch.full((M, N), float("nan"), device=DEV)
    tt.gemm(Ad, Bd, C, tt.FAM_BF16_UMMA, s)
    torch.cuda.synchronize()
    assert not torch.isnan(C).any()
    rng = np.random.default_rng(0)
    ii, jj = rng.integers(0, M, 512), rng.integers(0, N, 512)
    A32, B32 = synth.bf16_bits_to_f32(Ab), synth.bf16_bits_to_f32(Bb)
    R = og.gemm_f64_entries(A32, B32, ii, jj)
    got = C[torch.from_numpy(ii).to(DEV), torch.from_numpy(jj).to(DEV)].cpu().numpy()
    assert og.normwise_error(got, R) <= 5e-3


def test_simt_unaligned_views():
    # views whose data pointer is only 4-byte aligned take the scalar load/store paths
    M, N, K = 64, 64, 32
    A, B = host_inputs(M, N, K)
    Abuf = torch.zeros(M * K + 1, device=DEV)
    Bbuf = torch.zeros(K * N + 1, device=DEV)
    Cbuf = torch.full((M * N + 1,), float("nan"), device=DEV)
    Abuf[1:].copy_(torch.from_numpy(A).reshape(-1))
    Bbuf[1:].copy_(torch.from_numpy(B).reshape(-1))
    Av, Bv, Cv = Abuf[1:].view(M, K), Bbuf[1:].view(K, N), Cbuf[1:].view(M, N)
    tt.gemm(Av, Bv, Cv, tt.FAM_F32_SIMT, ((2, 2, 4, 4), (4, 8), (2, 2, 4, 4)))
    torch.cuda.synchronize()
    assert np.array_equal(Cv.cpu().numpy(), og.gemm_fmaf(A, B))
    with pytest.raises(tt.TileTuneError):
        tt.gemm(to_dev(A, True)[:, :].contiguous(), Bbuf[1:].view(K, N).to(torch.bfloat16), torch.empty(M, N, device=DEV),
                tt.FAM_BF16_UMMA, ((1, 1, 1, 128), (2, 16), (1, 1, 1, 64)))


# ------------------------------------------------------------------ round 2: full-size parity holes
def _tail_rows(sp_lib, cfg, M):
    """Rows to check for a config at full size: the first / last row and one row of every row
    block that holds a tile of the tail split (the last split_tiles tiles)."""
    info = tt.binding(sp_lib, cfg)
    m0 = cfg[0][0]
    tiles = m0 * cfg[2][0]
    rows = {0, M - 1}
    for t in range(tiles - info.split_tiles, tiles):
        tm = t % m0
        rows.add(tm * info.tile_m + (37 * t) % info.tile_m)
    return info, np.array(sorted(rows))


@pytest.mark.parametrize("fam,cfg", [
    (3, ((16, 2, 1, 128), (32, 128), (16, 1, 1, 256))),    # bf16 4096^3 driver-bench config (r1 BENCH)
    (3, ((8, 2, 2, 128), (64, 64), (16, 1, 1, 256))),      # bf16 4096^3 round-2 baseline best
    (2, ((8, 2, 2, 128), (128, 32), (16, 1, 1, 256))),     # tf32 4096^3 best (profiles/r7_workloads)
    (2, ((16, 2, 1, 128), (64, 64), (16, 1, 1, 256))),     # tf32 4096^3 round-2 best (wave+remainder split)
])
def test_umma_best_configs_4096_default_policy(fam, cfg):
    # the reported 4096^3 launches under the DEFAULT tail-split policy, rows crossing the split tiles
    M = N = K = 4096
    bf16 = fam == tt.FAM_BF16_UMMA
    sp_lib = tt.make_space(M, N, K, family=fam)
    info, rows = _tail_rows(sp_lib, cfg, M)
    A, B = host_inputs(M, N, K, bf16=bf16)
    C = run(fam, cfg, A, B)
    R = og.gemm_f64_rows(A, B, rows)
    assert og.normwise_error(C[rows], R) <= 5e-3, (cfg, info.split_tiles)
    assert not np.isnan(C).any()
    if cfg[0] == (16, 2, 1, 128) and cfg[2] == (16, 1, 1, 256):
        assert info.split_tiles == 256 % 74 + 74          # the headline launches split the last wave + tail


@pytest.mark.parametrize("fam,cfg", [
    (3, ((8, 2, 1, 128), (16, 128), (8, 1, 2, 128))),      # r13_workloads bf16_2048
    (3, ((16, 1, 1, 128), (32, 64), (8, 1, 1, 256))),      # r11_workloads bf16_2048
    (2, ((8, 2, 1, 128), (32, 64), (8, 1, 2, 128))),       # r13_workloads tf32_2048
    (2, ((8, 2, 1, 128), (32, 64), (8, 1, 1, 256))),       # r13_bench_final.json tf32 record
])
def test_umma_best_configs_2048_default_policy(fam, cfg):
    # the reported 2048^3 launches (BASELINE config 3's TF32 half, bf16 at the paper's 2048 shape)
    # under the default split policy, rows crossing any split tiles
    M = N = K = 2048
    sp_lib = tt.make_space(M, N, K, family=fam)
    info, rows = _tail_rows(sp_lib, cfg, M)
    A, B = host_inputs(M, N, K, bf16=fam == tt.FAM_BF16_UMMA)
    C = run(fam, cfg, A, B)
    assert not np.isnan(C).any()
    assert og.normwise_error(C[rows], og.gemm_f64_rows(A, B, rows)) <= 5e-3, (cfg, info.split_tiles)


@pytest.mark.parametrize("M,s", [
    (4096, ((64, 2, 2, 16), (128, 32), (16, 16, 2, 8))),   # profiles/r7_workloads, r13_bench_final.json
    (4096, ((64, 2, 2, 16), (128, 32), (16, 32, 1, 8))),   # found by the re-entry bench's f32_4096 search
    (2048, ((16, 4, 2, 16), (32, 64), (8, 8, 4, 8))),      # r13_bench_final.json fp32 (f32_2048)
    (2048, ((16, 2, 4, 16), (32, 64), (8, 16, 2, 8))),     # found by an r13 f32_2048 search
    (1024, ((16, 4, 2, 8), (8, 128), (8, 16, 2, 4))),      # r13_workloads f32_1024 (width 4)
])
def test_simt_best_config_sampled_rows(M, s):
    # K1's reported configs at full size, in the launch configuration bench.py times (TMA-fed B
    # slabs, one barrier per slab for the 128-accumulator tiles): fmaf-bit-exact rows
    N = K = M
    A, B = host_inputs(M, N, K)
    C = run(tt.FAM_F32_SIMT, s, A, B)
    rows = np.array([0, 1, 63, 64, M // 2 - 1, M - 96, M - 1])
    assert np.array_equal(C[rows], og.gemm_fmaf(A[rows], B))
    assert og.normwise_error(C[rows], og.gemm_f64_rows(A, B, rows)) <= 1e-4


@pytest.mark.parametrize("fam,cfg,split", [
    (1, ((8, 2, 4, 4), (512, 32), (8, 2, 4, 4)), "1"),
    (1, ((4, 4, 2, 8), (128, 128), (16, 2, 4, 2)), "1"),
    (3, ((2, 1, 1, 128), (256, 64), (2, 1, 1, 128)), "1"),
    (3, ((1, 2, 1, 128), (128, 128), (1, 1, 1, 256)), "2"),   # forced split: 1 pair tile over many clusters
    (2, ((2, 1, 1, 128), (512, 32), (2, 1, 1, 128)), "1"),
    (2, ((1, 2, 1, 128), (256, 64), (2, 1, 1, 128)), "2"),
])
def test_k16384_all_families(fam, cfg, split, monkeypatch):
    # the north star's tolerance clause holds "at K <= 16384": the longest K, full oracle
    monkeypatch.setenv("TT_TAIL_SPLIT", split)
    M, N, K = 256, 256, 16384
    assert space.legitimate(Spec(M, K, N, family=fam), cfg)
    bf16 = fam == tt.FAM_BF16_UMMA
    A, B = host_inputs(M, N, K, bf16=bf16)
    C = run(fam, cfg, A, B)
    R = og.gemm_f64(A, B)
    if fam == tt.FAM_F32_SIMT:
        assert np.array_equal(C, og.gemm_fmaf(A, B))
        assert og.normwise_error(C, R) <= 1e-4
    else:
        assert og.normwise_error(C, R) <= 5e-3
        if split == "2":
            assert tt.binding(tt.make_space(M, N, K, family=fam), cfg).split_tiles > 0


def test_na2c_T_decay_device_replay():
    # f1 ("the exploration step T can have a decay process"): live N-A2C with T decaying
    # 4 -> 1 every 2 episodes, and Alg. 2's in-loop training, on the device cost source;
    # the oracle's Algorithm 2 replayed on the recorded (state -> cost) table takes the same path
    sp = Spec(512, 512, 512, family=1)
    ctx = tt.Context(0)
    for kw, okw in ((dict(steps_T=4, steps_T_floor=1, steps_T_decay_every=2, batch=8),
                     dict(steps=4, steps_floor=1, decay_every=2, batch=8)),
                    (dict(train_per_candidate=1, batch=8), dict(train_per_candidate=True, batch=8))):
        res = tt.na2c_search(512, 512, 512, 40, tt.search_opts(family=1, seed=4, **kw), ctx=ctx)
        assert res.evals == 40
        table = {r["state"]: r["cost"] for r in res.trace}
        o = ona2c.na2c(sp, lambda batch: [table[s] for s in batch], budget=40, params=ona2c.Params(**okw), seed=4)
        assert [r.state for r in o.trace] == [r["state"] for r in res.trace]
        assert o.best_cost == res.best_cost
    ctx.close()


def test_random_search_device_replay():
    # f3 ("configurations are randomly selected to be tested"): the live random-search
    # comparator on the bf16 tcgen05 space of 512^3; the oracle draws the same states in order
    from oracle import random_search as ors
    ctx = tt.Context(0)
    res = tt.random_search(512, 512, 512, 40, tt.search_opts(family=3, seed=6, width=8), ctx=ctx)
    ctx.close()
    assert res.evals == 40 and res.space_feasible == 279
    table = {r["state"]: r["cost"] for r in res.trace}
    o = ors.random_search(Spec(512, 512, 512, family=3), lambda b: [table[s] for s in b], 40, seed=6, width=8)
    assert [r.state for r in o.trace] == [r["state"] for r in res.trace]
    assert o.best_cost == res.best_cost


def test_umma_tail_split_beside_concurrent_kernel(monkeypatch):
    # The tail split's pieces wait only on lower-index clusters, so it needs no
    # co-residency of its whole grid.  Launch it while a long SIMT kernel on another stream holds
    # the SMs (launched before and after it): it must complete, bit-identical to a lone launch.
    monkeypatch.setenv("TT_TAIL_SPLIT", "2")
    M = N = 2048
    K = 512
    cfg = ((16, 1, 1, 128), (8, 64), (16, 1, 1, 128))
    A, B = host_inputs(M, N, K, bf16=True)
    Ad, Bd = to_dev(A, True), to_dev(B, True)
    alone = torch.full((M, N), float("nan"), device=DEV)
    tt.gemm(Ad, Bd, alone, 3, cfg)
    torch.cuda.synchronize()
    assert tt.binding(tt.make_space(M, N, K, family=3), cfg).split_tiles > 0
    # blocker: the untiled s0 of 1024^3 fp32: 2^20 one-thread CTAs, tens of milliseconds
    Xb = torch.ones(1024, 1024, device=DEV)
    Yb = torch.ones(1024, 1024, device=DEV)
    Zb = torch.empty(1024, 1024, device=DEV)
    s0 = ((1024, 1, 1, 1), (1024, 1), (1024, 1, 1, 1))
    sb, sg = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for blocker_first in (True, False):
        C = torch.full((M, N), float("nan"), device=DEV)
        torch.cuda.synchronize()
        if blocker_first:
            tt.gemm(Xb, Yb, Zb, 1, s0, stream=sb)
        tt.gemm(Ad, Bd, C, 3, cfg, stream=sg)
        tt.gemm(Xb, Yb, Zb, 1, s0, stream=sb)
        tt.gemm(Ad, Bd, C, 3, cfg, stream=sg)
        torch.cuda.synchronize()
        outs.append(C.cpu().numpy())
    ref = alone.cpu().numpy()
    assert all(np.array_equal(o, ref) for o in outs)
    assert (Zb == 1024).all()


def test_measure_racing_and_measure_set():
    # reading Z12 racing: a candidate whose first race_repeats repeats exceed race_s stops there;
    # tt_measure_set = tt_measure per owned candidate, zeros elsewhere
    ctx = tt.Context(0)
    sp = tt.make_space(512, 512, 512, family=1)
    cfg = ((4, 2, 8, 8), (64, 8), (4, 4, 4, 8))
    lost = ctx.measure(sp, cfg, tt.measure_opts(race_s=1e-9))
    assert lost.raced == 1 and lost.repeats == 2 and lost.cost_s > 0
    won = ctx.measure(sp, cfg, tt.measure_opts(race_s=10.0))
    assert won.raced == 0 and won.repeats == 10
    fl = ctx.measure(sp, cfg, tt.measure_opts(l2_flush=1, race_s=1e-9, race_repeats=3))
    assert fl.raced == 1 and fl.repeats == 3 and fl.number == 1
    other = ((8, 2, 4, 8), (64, 8), (4, 4, 4, 8))
    costs, secs = ctx.measure_set(sp, [cfg, other, cfg], mine=[True, False, True])
    assert costs[1] == 0.0 and secs[1] == 0.0 and costs[0] > 0 and costs[2] > 0 and secs[0] > 0
    assert abs(costs[0] / won.cost_s - 1) < 0.2
    ctx.close()


def test_measure_phase_splits_one_measurement():
    # tt_measure_phase (two-phase sharded rounds, §8e): phase 1 = the cold probe (final only when
    # the slow cut decides the score), phase 2 = the repeats given that probe; together they give
    # the statistic of one tt_measure, and phase 2 honours racing and the cut with the given probe
    ctx = tt.Context(0)
    for fam, M, cfg in ((1, 512, ((4, 2, 8, 8), (64, 8), (4, 4, 4, 8))),
                        (3, 2048, ((16, 1, 1, 128), (16, 128), (16, 1, 1, 128)))):
        sp = tt.make_space(M, M, M, family=fam)
        mo = tt.measure_opts(l2_flush=1)
        whole = ctx.measure(sp, cfg, mo)
        v1, f1, s1 = ctx.measure_phase(sp, [cfg, cfg], [True, False], 1, None, mo)
        assert f1 == [False, False] and v1[1] == 0.0 and s1[1] == 0.0 and v1[0] > 0 and s1[0] > 0
        assert 0.5 < v1[0] / whole.probe_s < 2.0
        v2, f2, s2 = ctx.measure_phase(sp, [cfg], [True], 2, [v1[0]], mo)
        assert f2 == [True] and s2[0] > s1[0]
        assert abs(v2[0] / whole.cost_s - 1) < 0.2
        # the cut decides in phase 1 (final), and phase 2 with a probe above the cut returns it
        cut = tt.measure_opts(l2_flush=1, cut_s=1e-9)
        v1c, f1c, _ = ctx.measure_phase(sp, [cfg], [True], 1, None, cut)
        assert f1c == [True] and v1c[0] > 0
        v2c, _, _ = ctx.measure_phase(sp, [cfg], [True], 2, [0.5], cut)
        assert v2c == [0.5]
        # racing in phase 2: stops after race_repeats like tt_measure
        r2, _, sr = ctx.measure_phase(sp, [cfg], [True], 2, [v1[0]], tt.measure_opts(l2_flush=1, race_s=1e-9))
        assert r2[0] > 0 and sr[0] < s2[0]
    with pytest.raises(tt.TileTuneError):
        ctx.measure_phase(sp, [cfg], [True], 2, [0.0], tt.measure_opts(l2_flush=1))
    with pytest.raises(tt.TileTuneError):
        ctx.measure_phase(sp, [cfg], [True], 3, None, tt.measure_opts(l2_flush=1))
    ctx.close()


def test_gemm_plan_matches_gemm():
    # tt_plan: the same launch as tt_gemm_ex, bound once; bit-identical output
    M, N, K = 512, 256, 384
    A, B = host_inputs(M, N, K, bf16=True)
    Ad, Bd = to_dev(A, True), to_dev(B, True)
    cfg = ((2, 2, 1, 128), (6, 64), (1, 1, 1, 256))
    C1 = torch.full((M, N), float("nan"), device=DEV)
    tt.gemm(Ad, Bd, C1, 3, cfg)
    C2 = torch.full((M, N), float("nan"), device=DEV)
    plan = tt.GemmPlan(Ad, Bd, C2, 3, cfg)
    plan.launch()
    plan.launch(torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    plan.close()
    assert torch.equal(C1, C2)
    with pytest.raises(tt.TileTuneError):
        tt.GemmPlan(Ad, Bd, C2, 3, ((2, 2, 1, 128), (6, 64), (1, 1, 1, 128)))    # J_prod false


def test_partial_grid_probe_estimates_slow_simt():
    # reading Z12: the untiled s0 of 1024^3 fp32 (2^20 one-thread CTAs) is scored from its first
    # ~2 waves when that estimate exceeds the cut; the estimate must be close to a full launch
    ctx = tt.Context(0)
    sp = tt.make_space(1024, 1024, 1024, family=1)
    s0 = ((1024, 1, 1, 1), (1024, 1), (1024, 1, 1, 1))
    full = ctx.measure(sp, s0, tt.measure_opts(repeats=1, warmup=0))
    est = ctx.measure(sp, s0, tt.measure_opts(cut_s=1e-3))
    assert full.slow_cut == 0 and est.slow_cut == 2
    assert 0.6 < est.cost_s / full.cost_s < 1.4, (est.cost_s, full.cost_s)
    assert est.probe_s < full.cost_s / 10                  # the probe ran a small part of the grid
    fast = ((8, 2, 8, 8), (64, 16), (8, 4, 4, 8))          # 64 CTAs: never probed partially
    assert ctx.measure(sp, fast, tt.measure_opts(cut_s=1e-3)).slow_cut == 0
    ctx.close()


def _trace_lib():
    """The trace build of the library, built on first use."""
    lib = os.path.join(ROOT, "build", "variants", "trace", "libtiletune.so")
    if not os.path.exists(lib):
        from paper_1909_10616_b200 import build as b
        lib = b.build_variant("trace", ["TT_UMMA_TRACE_BUILD"])
    return lib


@pytest.mark.parametrize("mode,M,N,K,cfg", [
    ("1", 4096, 4096, 4096, ((16, 2, 1, 128), (32, 128), (16, 1, 1, 256))),   # bench launch: wave + remainder
    ("2", 2048, 2048, 512, ((16, 1, 1, 128), (8, 64), (16, 1, 1, 128))),      # round-1 tail split, forced
    ("4", 2048, 2048, 512, ((16, 1, 1, 128), (8, 64), (16, 2, 1, 64))),       # wave + remainder, n1 = 2
])
def test_device_schedule_matches_host(mode, M, N, K, cfg, tmp_path):
    # The items every cluster's epilogue actually processed (trace build, TT_UMMA_TRACE) are, in
    # order, the ones tt_umma_schedule computes on the host -- so the CPU schedule-invariant test
    # (coverage, ascending-k combine, lower-index-only waits) is a statement about the device.
    import subprocess
    import sys as _sys
    out = tmp_path / "trace.bin"
    env = dict(os.environ, TT_LIB_PATH=_trace_lib(), TT_UMMA_TRACE=str(out), TT_TAIL_SPLIT=mode)
    code = ("import torch, json, sys; sys.path.insert(0, %r); from paper_1909_10616_b200 import tiletune as tt; "
            "M, N, K = %d, %d, %d; cfg = %r; "
            "A = torch.randn(M, K, device='cuda').to(torch.bfloat16); B = torch.randn(K, N, device='cuda').to(torch.bfloat16); "
            "C = torch.empty(M, N, device='cuda'); tt.gemm(A, B, C, tt.FAM_BF16_UMMA, cfg); torch.cuda.synchronize()"
            % (ROOT, M, N, K, cfg))
    subprocess.run([_sys.executable, "-c", code], env=env, check=True, timeout=600)
    raw = np.fromfile(out, dtype=np.uint64)
    ncl, nit = int(raw[0]), int(raw[1])
    tr = raw[4:4 + ncl * nit * 8].reshape(ncl, nit, 8).astype(np.int64)
    os.environ["TT_TAIL_SPLIT"] = mode
    try:
        k0, per = tt.umma_schedule(tt.make_space(M, N, K, family=tt.FAM_BF16_UMMA), cfg)
    finally:
        del os.environ["TT_TAIL_SPLIT"]
    # the trace is sized grid / cta_group; with n1 = 2 only the first grid / cluster-size rows
    # (one per cluster, cluster_id = blockIdx / cluster size) are written
    assert len(per) <= ncl and not tr[len(per):, :, 2].any()
    for c in range(len(per)):
        dev = []
        for i in range(nit):
            if tr[c, i, 2] == 0:                       # slot 2 = MMA start time: 0 = no such item
                break
            w = int(tr[c, i, 1])
            dev.append((int(tr[c, i, 0]), w & 0xFFFF, (w >> 16) & 0xFFFF, w >> 32))
        host = [(t, a, b, o) for (t, a, b, o, _) in per[c]][:nit]
        assert dev == host, (c, dev, host)
