"""Thin ctypes binding of libtiletune (include/tiletune.h).  Argument marshalling only: every
step of the hot path runs inside the C++/CUDA library.  Names follow the ABI without the
``tt_`` prefix.  Device tensors are passed as raw pointers (``tensor.data_ptr()``) and the
torch current stream (``torch.cuda.current_stream().cuda_stream``); torch is plumbing only.

There is no fallback: if ``libtiletune.so`` is missing or fails to load, importing this module
raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Callable, List, Optional, Sequence, Tuple

HERE = os.path.dirname(os.path.abspath(__file__))
# TT_LIB_PATH: an alternative in-tree build of the same sources (kernel A/B experiments)
LIB_PATH = os.environ.get("TT_LIB_PATH") or os.path.join(HERE, "libtiletune.so")

OK, E_INVAL, E_ILLEGITIMATE, E_INFEASIBLE, E_OVERFLOW, E_CAPACITY, E_CUDA, E_EVALUATOR, E_UNSUPPORTED = range(9)
FAM_NONE, FAM_F32_SIMT, FAM_TF32_UMMA, FAM_BF16_UMMA = 0, 1, 2, 3
LAYOUT_NN, LAYOUT_TN = 0, 1
COST_DEVICE, COST_CALLBACK, COST_TABLE, COST_BATCH = 0, 1, 2, 3
MAXD = 4

i32, i64, u32, u64, dbl, vp = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double, C.c_void_p


class Space(C.Structure):
    _fields_ = [("M", i64), ("N", i64), ("K", i64), ("dm", i32), ("dk", i32), ("dn", i32), ("family", i32),
                ("layout", i32)]


class Config(C.Structure):
    _fields_ = [("m", i64 * MAXD), ("k", i64 * MAXD), ("n", i64 * MAXD)]


class Sample(C.Structure):
    _fields_ = [("cost_s", dbl), ("mean_s", dbl), ("min_s", dbl), ("stdev_s", dbl), ("probe_s", dbl),
                ("repeats", i32), ("number", i32), ("device", i32), ("slow_cut", i32), ("graph_nodes", i32),
                ("raced", i32)]


class MeasureOpts(C.Structure):
    _fields_ = [("warmup", i32), ("repeats", i32), ("min_repeat_s", dbl), ("cut_s", dbl), ("l2_flush", i32),
                ("max_number", i32), ("graph", i32),
                ("race_s", dbl), ("race_repeats", i32)]


class TraceRow(C.Structure):
    _fields_ = [("eval_index", u64), ("t_wall_s", dbl), ("cfg", Config), ("cost_s", dbl), ("best_so_far_s", dbl)]


class Result(C.Structure):
    _fields_ = [("best", Config), ("best_cost_s", dbl), ("evals", u64), ("space_raw", u64),
                ("space_feasible", u64), ("frac_raw", dbl), ("frac_feasible", dbl), ("wall_s", dbl),
                ("trace_len", u64)]


COST_FN = C.CFUNCTYPE(dbl, C.POINTER(Config), vp)
BATCH_FN = C.CFUNCTYPE(i32, C.POINTER(Config), i32, C.POINTER(dbl), vp)


class SearchOpts(C.Structure):
    _fields_ = [("family", i32), ("dm", i32), ("dk", i32), ("dn", i32), ("seed", u64), ("has_s0", i32),
                ("s0", Config), ("budget_seconds", dbl), ("cost_source", i32), ("cost_fn", COST_FN),
                ("batch_fn", BATCH_FN), ("user", vp), ("table", C.POINTER(dbl)), ("table_len", u64),
                ("measure", MeasureOpts), ("rho", i32), ("width", i32), ("steps_T", i32), ("epsilon", dbl),
                ("batch", i32), ("mem_capacity", i32), ("gamma", dbl), ("beta", dbl), ("lr", dbl), ("clip", dbl),
                ("epochs", i32), ("minibatch", i32), ("hidden", i32), ("rollout_cap_factor", i32),
                ("max_t_increase", i32), ("steps_T_floor", i32), ("steps_T_decay_every", i32), ("layout", i32),
                ("train_per_candidate", i32), ("cut_roofline_x", dbl), ("race_factor", dbl)]


class LaunchInfo(C.Structure):
    _fields_ = [("family", i32), ("grid_x", i64), ("grid_y", i64), ("grid_z", i64), ("block_x", i32),
                ("cluster_x", i32), ("smem_bytes", i32), ("stages", i32), ("tile_m", i32), ("tile_n", i32),
                ("tile_k", i32), ("tmem_cols", i32), ("acc_buffers", i32), ("idesc", u32), ("reg_tile_m", i32),
                ("reg_tile_n", i32), ("split_tiles", i32), ("split_workers", i32)]


EXPORTS = {
    "tt_version": (i32, []),
    "tt_last_error": (C.c_char_p, []),
    "tt_search_opts_default": (None, [C.POINTER(SearchOpts)]),
    "tt_measure_opts_default": (None, [C.POINTER(MeasureOpts)]),
    "tt_count_configs": (i32, [C.POINTER(Space), C.POINTER(u64), C.POINTER(u64)]),
    "tt_enumerate_configs": (i32, [C.POINTER(Space), u64, u64, C.POINTER(Config), C.POINTER(u64)]),
    "tt_enumerate_feasible": (i32, [C.POINTER(Space), u64, C.POINTER(Config), C.POINTER(u64), C.POINTER(u64)]),
    "tt_rank": (i32, [C.POINTER(Space), C.POINTER(Config), C.POINTER(u64)]),
    "tt_unrank": (i32, [C.POINTER(Space), u64, C.POINTER(Config)]),
    "tt_is_legitimate": (i32, [C.POINTER(Space), C.POINTER(Config), C.POINTER(i32), C.POINTER(i32)]),
    "tt_step": (i32, [C.POINTER(Space), C.POINTER(Config), i32, i32, i32, C.POINTER(Config), C.POINTER(i32)]),
    "tt_neighbors": (i32, [C.POINTER(Space), C.POINTER(Config), C.POINTER(Config), i32, C.POINTER(i32)]),
    "tt_binding": (i32, [C.POINTER(Space), C.POINTER(Config), C.POINTER(LaunchInfo)]),
    "tt_umma_schedule": (i32, [C.POINTER(Space), C.POINTER(Config), i32, C.POINTER(i32), i32, C.POINTER(i32),
                               C.POINTER(i32), C.POINTER(i32)]),
    "tt_fill_uniform": (i32, [vp, i32, u64, u64, u64, vp]),
    "tt_gemm": (i32, [i64, i64, i64, i32, vp, vp, vp, C.POINTER(Config), vp]),
    "tt_gemm_ex": (i32, [i64, i64, i64, i32, i32, vp, vp, vp, C.POINTER(Config), vp]),
    "tt_plan_create": (i32, [i64, i64, i64, i32, i32, vp, vp, vp, C.POINTER(Config), C.POINTER(vp)]),
    "tt_plan_launch": (i32, [vp, vp]),
    "tt_plan_destroy": (i32, [vp]),
    "tt_gemm_host": (i32, [vp, i64, i64, i64, i32, i32, vp, vp, vp, C.POINTER(Config)]),
    "tt_ctx_create": (i32, [i32, u64, C.POINTER(vp)]),
    "tt_ctx_destroy": (i32, [vp]),
    "tt_ctx_stream": (i32, [vp, C.POINTER(vp)]),
    "tt_ctx_prepare": (i32, [vp, C.POINTER(Space)]),
    "tt_ctx_operands": (i32, [vp, i64, i64, i64, i32, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]),
    "tt_aggregate": (i32, [C.POINTER(dbl), i32, C.POINTER(Sample)]),
    "tt_roofline_seconds": (i32, [C.POINTER(Space), i32, C.POINTER(dbl)]),
    "tt_scoring_opts": (i32, [C.POINTER(Space), i32, C.POINTER(SearchOpts), dbl, C.POINTER(MeasureOpts)]),
    "tt_measure_set": (i32, [vp, C.POINTER(Space), C.POINTER(Config), i32, C.POINTER(C.c_uint8),
                             C.POINTER(MeasureOpts), C.POINTER(dbl), C.POINTER(dbl)]),
    "tt_measure_phase": (i32, [vp, C.POINTER(Space), C.POINTER(Config), i32, C.POINTER(C.c_uint8),
                               C.POINTER(MeasureOpts), i32, C.POINTER(dbl), C.POINTER(dbl), C.POINTER(C.c_uint8),
                               C.POINTER(dbl)]),
    "tt_measure": (i32, [vp, C.POINTER(Space), C.POINTER(Config), C.POINTER(MeasureOpts), C.POINTER(Sample)]),
    "tt_gbfs_search": (i32, [vp, i64, i64, i64, u64, C.POINTER(SearchOpts), C.POINTER(Result),
                             C.POINTER(TraceRow), u64]),
    "tt_na2c_search": (i32, [vp, i64, i64, i64, u64, C.POINTER(SearchOpts), C.POINTER(Result),
                             C.POINTER(TraceRow), u64]),
    "tt_im2col": (i32, [i32, vp, i64, i64, i64, i64, i32, i32, i32, i32, vp, vp]),
    "tt_conv2d": (i32, [i32, vp, i64, i64, i64, i64, vp, i64, i32, i32, i32, i32, vp, vp, u64, C.POINTER(Config), vp]),
    "tt_random_search": (i32, [vp, i64, i64, i64, u64, C.POINTER(SearchOpts), C.POINTER(Result),
                               C.POINTER(TraceRow), u64]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1909_10616_b200.build` "
                          "(there is no CPU or Python fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in EXPORTS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


class TileTuneError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = lib.tt_last_error().decode(errors="replace")
        super().__init__(f"{where}: status {status}: {msg}")


def _check(st: int, where: str):
    if st != OK:
        raise TileTuneError(st, where)


# ------------------------------------------------------------------------------------ helpers
State = Tuple[Tuple[int, ...], Tuple[int, ...], Tuple[int, ...]]


def make_space(M: int, N: int, K: int, dm: int = 4, dk: int = 2, dn: int = 4, family: int = FAM_NONE,
               layout: int = LAYOUT_NN) -> Space:
    return Space(M, N, K, dm, dk, dn, family, layout)


def to_config(s: State) -> Config:
    """tt_config of a state (unused inner slots = 1).  A fresh object every call (callers may
    keep it), built from padded tuples in one constructor call: searches marshal every candidate."""
    pad = (1,) * MAXD
    return Config((tuple(s[0]) + pad)[:MAXD], (tuple(s[1]) + pad)[:MAXD], (tuple(s[2]) + pad)[:MAXD])


def from_config(c: Config, depths=(4, 2, 4)) -> State:
    return (tuple(c.m[:depths[0]]), tuple(c.k[:depths[1]]), tuple(c.n[:depths[2]]))


def _depths(sp: Space):
    return (sp.dm, sp.dk, sp.dn)


# ------------------------------------------------------------------------------------ space
def count_configs(sp: Space, feasible: bool = False):
    raw, fz = u64(), u64()
    _check(lib.tt_count_configs(C.byref(sp), C.byref(raw), C.byref(fz) if feasible else None), "count_configs")
    return (raw.value, fz.value) if feasible else raw.value


def enumerate_configs(sp: Space, first_rank: int = 0, cap: Optional[int] = None) -> List[State]:
    raw = count_configs(sp)
    cap = raw - first_rank if cap is None else cap
    buf = (Config * max(cap, 1))()
    n = u64()
    _check(lib.tt_enumerate_configs(C.byref(sp), first_rank, cap, buf, C.byref(n)), "enumerate_configs")
    d = _depths(sp)
    return [from_config(buf[i], d) for i in range(n.value)]


def enumerate_feasible(sp: Space) -> Tuple[List[State], List[int]]:
    n = u64()
    _check(lib.tt_enumerate_feasible(C.byref(sp), 0, None, None, C.byref(n)), "enumerate_feasible(count)")
    cfgs = (Config * max(n.value, 1))()
    ranks = (u64 * max(n.value, 1))()
    _check(lib.tt_enumerate_feasible(C.byref(sp), n.value, cfgs, ranks, C.byref(n)), "enumerate_feasible")
    d = _depths(sp)
    return [from_config(cfgs[i], d) for i in range(n.value)], [ranks[i] for i in range(n.value)]


def rank(sp: Space, s: State) -> int:
    r = u64()
    _check(lib.tt_rank(C.byref(sp), C.byref(to_config(s)), C.byref(r)), "rank")
    return r.value


def unrank(sp: Space, r: int) -> State:
    c = Config()
    _check(lib.tt_unrank(C.byref(sp), r, C.byref(c)), "unrank")
    return from_config(c, _depths(sp))


def is_legitimate(sp: Space, s: State) -> Tuple[bool, bool]:
    jp, jh = i32(), i32()
    _check(lib.tt_is_legitimate(C.byref(sp), C.byref(to_config(s)), C.byref(jp), C.byref(jh)), "is_legitimate")
    return bool(jp.value), bool(jh.value)


def step(sp: Space, s: State, axis: int, i: int, j: int) -> Optional[State]:
    out, legit = Config(), i32()
    _check(lib.tt_step(C.byref(sp), C.byref(to_config(s)), axis, i, j, C.byref(out), C.byref(legit)), "step")
    return from_config(out, _depths(sp)) if legit.value else None


def neighbors(sp: Space, s: State) -> List[State]:
    buf = (Config * 64)()
    n = i32()
    _check(lib.tt_neighbors(C.byref(sp), C.byref(to_config(s)), buf, 64, C.byref(n)), "neighbors")
    d = _depths(sp)
    return [from_config(buf[i], d) for i in range(n.value)]


def umma_schedule(sp: Space, s: State):
    """tt_umma_schedule for every cluster: (k0, [[(tile, kb0, kb1, order, split), ...] per cluster])."""
    n, workers, k0 = i32(), i32(), i32()
    cfg = to_config(s)
    _check(lib.tt_umma_schedule(C.byref(sp), C.byref(cfg), 0, None, 0, C.byref(n), C.byref(workers), C.byref(k0)),
           "umma_schedule")
    out = []
    for w in range(workers.value):
        _check(lib.tt_umma_schedule(C.byref(sp), C.byref(cfg), w, None, 0, C.byref(n), C.byref(workers),
                                    C.byref(k0)), "umma_schedule")
        buf = (i32 * max(5 * n.value, 1))()
        _check(lib.tt_umma_schedule(C.byref(sp), C.byref(cfg), w, buf, n.value, C.byref(n), C.byref(workers),
                                    C.byref(k0)), "umma_schedule")
        out.append([tuple(buf[5 * i:5 * i + 5]) for i in range(n.value)])
    return k0.value, out


def binding(sp: Space, s: State) -> LaunchInfo:
    info = LaunchInfo()
    _check(lib.tt_binding(C.byref(sp), C.byref(to_config(s)), C.byref(info)), "binding")
    return info


# ------------------------------------------------------------------------------------ device
def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if hasattr(stream, "cuda_stream"):                   # torch.cuda.Stream
        return stream.cuda_stream
    return int(stream)


def fill_uniform(tensor, seed: int, idx0: int = 0, stream=None):
    """K4 into a contiguous fp32 / bf16 CUDA tensor (global index of element 0 = idx0)."""
    import torch
    dt = {torch.float32: 0, torch.bfloat16: 1}[tensor.dtype]
    assert tensor.is_cuda and tensor.is_contiguous()
    _check(lib.tt_fill_uniform(tensor.data_ptr(), dt, seed, idx0, tensor.numel(), _stream(stream)), "fill_uniform")


def _operand_dtype(family: int):
    import torch
    if family == FAM_BF16_UMMA:
        return torch.bfloat16
    if family in (FAM_F32_SIMT, FAM_TF32_UMMA):
        return torch.float32
    raise ValueError(f"family {family} has no kernel")


def _check_gemm_operands(A, B, C_out, family: int, layout: int, on_device: bool):
    """The C-ABI sees raw pointers only, so this binding is the one place that can reject a wrong
    dtype (a bf16 buffer read as fp32 runs past its end), a strided view, a mismatched shape or a
    tensor on another device before the library reads or writes it.  Returns (M, N, K)."""
    import torch
    want = _operand_dtype(family)
    named = (("A", A, want), ("B", B, want), ("C", C_out, torch.float32))
    for name, t, dt in named:
        if t.dtype != dt:
            raise TypeError(f"{name} must be {dt} for family {family}, got {t.dtype}")
    for name, t, _ in named:
        if t.dim() != 2 or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous 2-D tensor (row-major), got shape "
                             f"{tuple(t.shape)} strides {t.stride()}")
        if on_device and not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor")
        if not on_device and t.is_cuda:
            raise ValueError(f"{name} must be a host tensor")
    if on_device and not (A.device == B.device == C_out.device):
        raise ValueError(f"A, B, C on different devices: {A.device}, {B.device}, {C_out.device}")
    if layout == LAYOUT_TN:
        K, M = A.shape
    else:
        M, K = A.shape
    K2, N = B.shape
    if K != K2 or tuple(C_out.shape) != (M, N):
        raise ValueError(f"shapes do not chain: A {tuple(A.shape)} (layout {layout}), B {tuple(B.shape)}, "
                         f"C {tuple(C_out.shape)}")
    return M, N, K


def gemm(A, B, C_out, family: int, s: State, stream=None, layout: int = LAYOUT_NN):
    """C_out[M,N] (fp32) = A[M,K] . B[K,N] with config s on the device (tt_gemm_ex).  With
    layout=LAYOUT_TN, A is passed as W = A^T of shape [K, M] (P:372 Y = W^T X)."""
    M, N, K = _check_gemm_operands(A, B, C_out, family, layout, on_device=True)
    _check(lib.tt_gemm_ex(M, N, K, family, layout, A.data_ptr(), B.data_ptr(), C_out.data_ptr(),
                          C.byref(to_config(s)), _stream(stream)), "gemm")


def aggregate(per_repeat: Sequence[float]) -> Sample:
    """The cost statistic tt_measure applies to its per-repeat means (tt_aggregate, reading Z10)."""
    arr = (dbl * max(len(per_repeat), 1))(*per_repeat)
    out = Sample()
    _check(lib.tt_aggregate(arr, len(per_repeat), C.byref(out)), "aggregate")
    return out


def roofline_seconds(sp: Space, device: int = -1) -> float:
    """One GEMM of sp at the family's nominal device peak (tt_roofline_seconds)."""
    t = dbl()
    _check(lib.tt_roofline_seconds(C.byref(sp), device, C.byref(t)), "roofline_seconds")
    return t.value


def scoring_opts(sp: Space, opts: "SearchOpts", cost_min: float, device: int = -1) -> "MeasureOpts":
    """Per-candidate measurement options of a search at incumbent cost_min (tt_scoring_opts, Z12)."""
    mo = MeasureOpts()
    _check(lib.tt_scoring_opts(C.byref(sp), device, C.byref(opts), cost_min, C.byref(mo)), "scoring_opts")
    return mo


class GemmPlan:
    """tt_plan: one GEMM bound to its buffers once (checked here and in the library), then
    ``launch()`` is a single library call -- for launching the same GEMM many times."""

    def __init__(self, A, B, C_out, family: int, s: State, layout: int = LAYOUT_NN):
        M, N, K = _check_gemm_operands(A, B, C_out, family, layout, on_device=True)
        self._keep = (A, B, C_out)                         # the plan holds raw pointers
        self.h = vp()
        _check(lib.tt_plan_create(M, N, K, family, layout, A.data_ptr(), B.data_ptr(), C_out.data_ptr(),
                                  C.byref(to_config(s)), C.byref(self.h)), "plan_create")

    def launch(self, stream=None):
        """stream: None (torch's current stream), a torch.cuda.Stream or a raw cudaStream_t int."""
        st = lib.tt_plan_launch(self.h, _stream(stream))
        if st != OK:
            raise TileTuneError(st, "plan_launch")

    def close(self):
        if self.h:
            lib.tt_plan_destroy(self.h)
            self.h = vp()
            self._keep = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def measure_opts(**kw) -> MeasureOpts:
    mo = MeasureOpts()
    lib.tt_measure_opts_default(C.byref(mo))
    for k, v in kw.items():
        setattr(mo, k, v)
    return mo


class Context:
    """tt_ctx: device measurement context (B2)."""

    def __init__(self, device: int = 0, input_seed: int = 1):
        self.h = vp()
        _check(lib.tt_ctx_create(device, input_seed, C.byref(self.h)), "ctx_create")

    def close(self):
        if self.h:
            lib.tt_ctx_destroy(self.h)
            self.h = vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        s = vp()
        _check(lib.tt_ctx_stream(self.h, C.byref(s)), "ctx_stream")
        return s.value or 0

    def operands(self, M, N, K, family):
        a, b, c = vp(), vp(), vp()
        _check(lib.tt_ctx_operands(self.h, M, N, K, family, C.byref(a), C.byref(b), C.byref(c)), "ctx_operands")
        return a.value, b.value, c.value

    def prepare(self, sp: Space):
        """tt_ctx_prepare: operands, flush buffer and the family's kernels loaded (one-time setup)."""
        _check(lib.tt_ctx_prepare(self.h, C.byref(sp)), "ctx_prepare")

    def measure(self, sp: Space, s: State, opts: Optional[MeasureOpts] = None) -> Sample:
        out = Sample()
        _check(lib.tt_measure(self.h, C.byref(sp), C.byref(to_config(s)), C.byref(opts) if opts else None,
                              C.byref(out)), "measure")
        return out

    def measure_set(self, sp: Space, states: Sequence[State], mine: Optional[Sequence[bool]] = None,
                    opts: Optional[MeasureOpts] = None):
        """tt_measure_set: costs (and host seconds) of the states with mine[j] true, 0 elsewhere."""
        n = len(states)
        cfgs = (Config * max(n, 1))(*[to_config(s) for s in states])
        mk = (C.c_uint8 * max(n, 1))(*[1 if m else 0 for m in mine]) if mine is not None else None
        costs = (dbl * max(n, 1))()
        secs = (dbl * max(n, 1))()
        _check(lib.tt_measure_set(self.h, C.byref(sp), cfgs, n, mk, C.byref(opts) if opts else None, costs, secs),
               "measure_set")
        return [costs[j] for j in range(n)], [secs[j] for j in range(n)]

    def measure_phase(self, sp: Space, states: Sequence[State], mine: Optional[Sequence[bool]], phase: int,
                      probes: Optional[Sequence[float]] = None, opts: Optional[MeasureOpts] = None):
        """tt_measure_phase: (values, final, secs) of the states with mine[j] true (phase 1: the
        cold probe, or the final score when the probe decides it; phase 2: the rest given probes)."""
        n = len(states)
        cfgs = (Config * max(n, 1))(*[to_config(s) for s in states])
        mk = (C.c_uint8 * max(n, 1))(*[1 if m else 0 for m in mine]) if mine is not None else None
        pr = (dbl * max(n, 1))(*[float(p) for p in probes]) if probes is not None else None
        vals = (dbl * max(n, 1))()
        fin = (C.c_uint8 * max(n, 1))()
        secs = (dbl * max(n, 1))()
        _check(lib.tt_measure_phase(self.h, C.byref(sp), cfgs, n, mk, C.byref(opts) if opts else None, phase, pr,
                                    vals, fin, secs), "measure_phase")
        return [vals[j] for j in range(n)], [bool(fin[j]) for j in range(n)], [secs[j] for j in range(n)]

    def gemm_host(self, A_host, B_host, C_host, family: int, s: State, layout: int = LAYOUT_NN):
        M, N, K = _check_gemm_operands(A_host, B_host, C_host, family, layout, on_device=False)
        _check(lib.tt_gemm_host(self.h, M, N, K, family, layout, A_host.data_ptr(), B_host.data_ptr(),
                                C_host.data_ptr(), C.byref(to_config(s))), "gemm_host")


# ------------------------------------------------------------------------------------ searches
def search_opts(**kw) -> SearchOpts:
    o = SearchOpts()
    lib.tt_search_opts_default(C.byref(o))
    for k, v in kw.items():
        if k == "measure" and isinstance(v, dict):
            for mk, mv in v.items():
                setattr(o.measure, mk, mv)
        else:
            setattr(o, k, v)
    return o


class SearchResult:
    """A search's result.  ``trace`` (one dict per evaluated state, in evaluation order) is built
    from the library's tt_trace_row array on first access: a sharded search runs on every rank,
    and the conversion is presentation, not search work."""

    def __init__(self, res: Result, rows, n: int, depths):
        self.best = from_config(res.best, depths)
        self.best_cost = res.best_cost_s
        self.evals = res.evals
        self.space_raw = res.space_raw
        self.space_feasible = res.space_feasible
        self.frac_raw = res.frac_raw
        self.frac_feasible = res.frac_feasible
        self.wall_s = res.wall_s
        self._rows, self._n, self._depths = rows, n, depths
        self._trace = None

    @property
    def trace(self) -> List[dict]:
        if self._trace is None:
            r, d = self._rows, self._depths
            self._trace = [dict(eval_index=r[i].eval_index, t_wall_s=r[i].t_wall_s, state=from_config(r[i].cfg, d),
                                cost=r[i].cost_s, best=r[i].best_so_far_s) for i in range(self._n)]
            self._rows = None
        return self._trace


def _search(fn, name, M, N, K, budget, opts: SearchOpts, ctx: Optional[Context], cost=None, table=None,
            batch=None, trace_cap: Optional[int] = None) -> SearchResult:
    keep = []
    if cost is not None:
        cb = COST_FN(lambda cfgp, user: float(cost(from_config(cfgp[0], (opts.dm, opts.dk, opts.dn)))))
        keep.append(cb)
        opts.cost_fn = cb
        opts.cost_source = COST_CALLBACK
    if table is not None:
        arr = (dbl * len(table))(*table)
        keep.append(arr)
        opts.table = C.cast(arr, C.POINTER(dbl))
        opts.table_len = len(table)
        opts.cost_source = COST_TABLE
    if batch is not None:
        d = (opts.dm, opts.dk, opts.dn)

        def _b(cfgs, n, costs, user):
            try:
                vals = batch([from_config(cfgs[i], d) for i in range(n)])
                for i in range(n):
                    costs[i] = float(vals[i])
                return 0
            except Exception:  # noqa: BLE001 - reported as TT_E_EVALUATOR
                import traceback
                traceback.print_exc()
                return 1

        bb = BATCH_FN(_b)
        keep.append(bb)
        opts.batch_fn = bb
        opts.cost_source = COST_BATCH
    cap = trace_cap if trace_cap is not None else (budget if budget else 1 << 20)
    trace = (TraceRow * max(cap, 1))()
    res = Result()
    st = fn(ctx.h if ctx else None, M, N, K, budget, C.byref(opts), C.byref(res), trace, cap)
    _check(st, name)
    d = (opts.dm, opts.dk, opts.dn)
    return SearchResult(res, trace, res.trace_len, d)


def gbfs_search(M: int, N: int, K: int, budget: int, opts: Optional[SearchOpts] = None,
                ctx: Optional[Context] = None, **kw) -> SearchResult:
    """G-BFS (Alg. 1).  Cost source: ctx (DEVICE), or one of cost= / table= / batch=."""
    return _search(lib.tt_gbfs_search, "gbfs_search", M, N, K, budget, opts or search_opts(), ctx, **kw)


def na2c_search(M: int, N: int, K: int, budget: int, opts: Optional[SearchOpts] = None,
                ctx: Optional[Context] = None, **kw) -> SearchResult:
    """N-A2C (Alg. 2).  Same contract as gbfs_search."""
    return _search(lib.tt_na2c_search, "na2c_search", M, N, K, budget, opts or search_opts(), ctx, **kw)


def random_search(M: int, N: int, K: int, budget: int, opts: Optional[SearchOpts] = None,
                  ctx: Optional[Context] = None, **kw) -> SearchResult:
    """Random-search comparator.  Same contract as gbfs_search."""
    return _search(lib.tt_random_search, "random_search", M, N, K, budget, opts or search_opts(), ctx, **kw)


# ------------------------------------------------------------------------------------ conv
def conv_out_hw(H, W, R, S, stride=1, pad=0):
    return (H + 2 * pad - R) // stride + 1, (W + 2 * pad - S) // stride + 1


def conv_gemm_dims(x_shape, Kf, R, S, stride=1, pad=0):
    """(M, N, K) of the GEMM a conv layer becomes: (Nb*P*Q, Kf, C*R*S)."""
    Nb, Cc, H, W = x_shape
    P, Q = conv_out_hw(H, W, R, S, stride, pad)
    return Nb * P * Q, Kf, Cc * R * S


def im2col(x, R, S, stride=1, pad=0, out=None, stream=None):
    """A [Nb*P*Q, C*R*S] from NCHW x (fp32 or bf16 CUDA tensor) on the device (tt_im2col)."""
    import torch
    Nb, Cc, H, W = x.shape
    P, Q = conv_out_hw(H, W, R, S, stride, pad)
    if not (x.is_cuda and x.is_contiguous()):
        raise ValueError("im2col needs a contiguous NCHW CUDA tensor")
    if out is None:
        out = torch.empty(Nb * P * Q, Cc * R * S, device=x.device, dtype=x.dtype)
    elif not (out.is_contiguous() and out.dtype == x.dtype and out.numel() == Nb * P * Q * Cc * R * S):
        raise ValueError("im2col out must be contiguous, of x's dtype and [Nb*P*Q, C*R*S] elements")
    dt = {torch.float32: 0, torch.bfloat16: 1}[x.dtype]
    _check(lib.tt_im2col(dt, x.data_ptr(), Nb, Cc, H, W, R, S, stride, pad, out.data_ptr(), _stream(stream)),
           "im2col")
    return out


def conv2d(x, Wm, family: int, s: State, R: int, S: int, stride=1, pad=0, workspace=None, stream=None):
    """Conv layer through im2col + the tiled GEMM: returns y [Nb*P*Q, Kf] fp32 (tt_conv2d);
    Wm is the kernel matrix [C*R*S, Kf]."""
    import torch
    want = _operand_dtype(family)
    if x.dtype != want or Wm.dtype != want or not x.is_contiguous() or not Wm.is_contiguous():
        raise TypeError(f"conv2d with family {family} needs contiguous {want} x and Wm")
    if not (x.is_cuda and Wm.is_cuda and x.device == Wm.device):
        raise ValueError("x and Wm must be CUDA tensors on one device")
    Nb, Cc, H, W = x.shape
    M, Kf, K = conv_gemm_dims(x.shape, Wm.shape[1], R, S, stride, pad)
    if Wm.dim() != 2 or Wm.shape[0] != K:
        raise ValueError(f"kernel matrix must be [C*R*S, Kf] = [{K}, Kf], got {tuple(Wm.shape)}")
    if workspace is None:
        workspace = torch.empty(M * K, device=x.device, dtype=x.dtype)
    y = torch.empty(M, Kf, device=x.device, dtype=torch.float32)
    _check(lib.tt_conv2d(family, x.data_ptr(), Nb, Cc, H, W, Wm.data_ptr(), Kf, R, S, stride, pad, y.data_ptr(),
                         workspace.data_ptr(), workspace.numel() * workspace.element_size(), C.byref(to_config(s)),
                         _stream(stream)), "conv2d")
    return y
