"""Benchmark of the hot path: G-BFS-tuned tiled GEMM on B200 (arXiv 1909.10616).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--workload NAME]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU, NCCL)

Metric (BASELINE.json): best-found GEMM TFLOP/s (and % of peak), tuning wall time and % of the
configuration space explored.  Workload (default ``bf16_4096``, BASELINE configs[3]): C = A.B
at 4096^3 with bf16 operands and fp32 accumulation/output on the tcgen05 family (K3).

One run does, in order:
 1. the tuning pass (every SURVEY §8(a) row): space count / J_hw, G-BFS (Alg. 1 with width
    W = 16, rho = 5; reading Z9) with candidate rounds measured by libtiletune's device
    evaluator (tt_measure_set) -- sharded over the ranks (LPT assignment, one all_reduce of the
    costs per round) when N > 1 -- and the fraction explored;
 2. W untimed warm-up steps and K timed steps of the best-found GEMM, one launch per step on
    each rank's row shard (rank r owns A rows [4096 r, 4096 (r+1)), B replicated, no collective
    on the math path: weak scaling).  The L2 is flushed (256 MiB memset) before every step,
    outside the CUDA-event pair that times the launch; barrier + synchronize on both sides;
    the per-step time is the max over ranks.
 3. ``e2e``: the same GEMM through tt_gemm_host (pinned host A, B in; C out) per step;
 4. ``fp32``: the paper's own arithmetic (fp32 FFMA, K1) on ``--fp32-workload`` (f32_2048):
    G-BFS at 0.1 % of the raw space from the untiled s0, timed steps, fraction of the FFMA peak;
 5. ``cpu_baseline``: the oracle's double GEMM (oracle/gemm_ref.c) on a bounded row sample.

``--impl reference`` times the oracle alone (the reference arm of this tier), rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (M per rank, N, K, family, default budget)
    # UMMA families: 128 evaluations = ~45 % of the 286 feasible states, 0.005 % of the raw space
    # (64 missed the best tile in 1 of 3 seeds once n1 = 2 doubled the feasible set)
    "bf16_4096": (4096, 4096, 4096, 3, 128),
    # BASELINE configs[4]: 8192^3 row-partitioned; M per rank = 8192 / N GPUs (strong scaling)
    "bf16_8192": (8192, 8192, 8192, 3, 128),
    # one rank's shard of bf16_8192 at N = 8 (per-shard config tuned on (1024, 8192, 8192))
    "bf16_8192_shard8": (1024, 8192, 8192, 3, 128),
    "tf32_2048": (2048, 2048, 2048, 2, 128),
    "tf32_4096": (4096, 4096, 4096, 2, 128),
    # fp32 SIMT: 0.1 % of the raw space (the paper's budget, P:375 / P:397), s0 untiled
    "f32_4096": (4096, 4096, 4096, 1, 2691),
    "f32_2048": (2048, 2048, 2048, 1, 1590),
    "f32_512": (512, 512, 512, 1, 484),
    # the paper's main experiment shape: 0.1 % of 899 756 states
    "f32_1024": (1024, 1024, 1024, 1, 900),
    "bf16_1024": (1024, 1024, 1024, 3, 128),
    "bf16_2048": (2048, 2048, 2048, 3, 128),
}
FAMILY_DTYPE = {1: "f32", 2: "tf32", 3: "bf16"}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def fp32_fma_peak_tflops(sm_mhz: float) -> float:
    # 148 SMs x 128 FP32 lanes x 2 flop/FMA x clock (guide unit counts)
    return 148 * 128 * 2 * sm_mhz * 1e6 / 1e12


class ClockSampler:
    """SM clock and clock-event (throttle) reasons polled through NVML every ~2 ms during the timed
    region (the recipe's nvidia-smi clocks line, at a rate that resolves a millisecond-scale region);
    falls back to nvidia-smi -lms 100 when NVML is unavailable."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown", "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown", "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
               "hw_power_brake": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._thr = None
        self.proc = None
        self.lines = []

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            masks = {k: getattr(nv, v) for k, v in self.REASONS.items() if hasattr(nv, v)}

            def poll():
                while not self._stop.is_set():
                    try:
                        self.samples.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for k, m in masks.items():
                            if r & m:
                                self.reasons.add(k)
                    except Exception:  # noqa: BLE001
                        pass
                    time.sleep(0.002)
            self._thr = threading.Thread(target=poll, daemon=True)
            self._thr.start()
        except Exception:  # noqa: BLE001 - NVML missing: nvidia-smi fallback
            try:
                fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                          "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
                self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={fields}",
                                              "--format=csv,noheader,nounits", "-lms", "100"],
                                             stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                threading.Thread(target=lambda: [self.lines.append(ln.strip()) for ln in self.proc.stdout],
                                 daemon=True).start()
            except FileNotFoundError:
                self.proc = None

    def stop(self):
        if self._thr is not None:
            time.sleep(0.01)
            self._stop.set()
            self._thr.join(timeout=1)
            return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                    "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml 2 ms"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"], "samples": 0}
        time.sleep(0.2)
        self.proc.terminate()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi 100 ms"}


def cpu_oracle_sample(M, N, K, family, seconds: float = 12.0, max_rows: int = 4096):
    """Time the oracle's double GEMM (oracle/gemm_ref.c, as it stands) on row blocks of the
    workload until ``seconds`` of CPU work; returns (TFLOP/s, cores, sample description)."""
    import numpy as np

    import synth
    from oracle import gemm as og
    A = synth.uniform_f32(synth.SEED_A, M, K)
    B = synth.uniform_f32(synth.SEED_B, K, N)
    if family == 3:
        A = synth.bf16_bits_to_f32(synth.to_bf16_bits(A))
        B = synth.bf16_bits_to_f32(synth.to_bf16_bits(B))
    A64, B64 = A.astype(np.float64), B.astype(np.float64)
    og.gemm_f64_rows(A64, B64, [0])  # build + warm
    rows_done, t_total, blk = 0, 0.0, 16
    while t_total < seconds and rows_done < max_rows:
        rows = np.arange(rows_done, min(rows_done + blk, M))
        t0 = time.perf_counter()
        og.gemm_f64_rows(A64, B64, rows)
        t_total += time.perf_counter() - t0
        rows_done += len(rows)
        blk = min(blk * 2, 256)
    flops = 2.0 * rows_done * N * K
    cores = len(os.sched_getaffinity(0))
    return flops / t_total / 1e12, cores, f"{rows_done} rows x {N} x {K} of the {M}x{N}x{K} product, " \
                                          f"double triple loop, {t_total:.1f} s"


def run_reference(args):
    """Reference arm of this tier: the oracle as it stands on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np

    import synth
    from oracle import gemm as og
    M, N, K, fam, _ = WORKLOADS[args.workload]
    A = synth.uniform_f32(synth.SEED_A, M, K)
    B = synth.uniform_f32(synth.SEED_B, K, N)
    if fam == 3:
        A = synth.bf16_bits_to_f32(synth.to_bf16_bits(A))
        B = synth.bf16_bits_to_f32(synth.to_bf16_bits(B))
    A64, B64 = A.astype(np.float64), B.astype(np.float64)
    rows_per_step = args.ref_rows
    times = []
    for it in range(args.warmup + args.steps):
        r0 = (it * rows_per_step) % M
        rows = np.arange(r0, r0 + rows_per_step)
        t0 = time.perf_counter()
        og.gemm_f64_rows(A64, B64, rows)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    flops = 2.0 * rows_per_step * N * K
    value = flops / (ms * 1e-3) / 1e12
    cores = len(os.sched_getaffinity(0))
    sample = f"{rows_per_step} rows x {N} x {K} per step of the {M}x{N}x{K} product (double triple loop)"
    print(json.dumps({
        "impl": "reference", "metric": "best-found GEMM TFLOP/s", "value": value, "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": args.workload, "M": M, "N": N, "K": K},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# G-BFS width W per workload when --width is not given (reading Z9; the same for every GPU count).
# W = 16 gives a sharded round enough candidates and finds the same configs as W = 1 at the
# tensor-core spaces and fp32 2048^3 / 4096^3; at the 0.1 % budgets of 512^3 (484 evaluations) and
# 1024^3 (900) a round of 16 pops spends the budget breadth-first and stalls far from the optimum:
# f32_1024 19-23 TF/s at W = 16 vs 32.7-33.0 at W = 1 / 4, f32_512 4-5.5 vs 14.1-14.4 at W = 1
# (3 seeds each, profiles/r13_width_small_fp32.txt).
DEFAULT_WIDTH = {"f32_512": 1, "f32_1024": 4}


def width_of(args, workload):
    return args.width if args.width is not None else DEFAULT_WIDTH.get(workload, 16)


def tune(ctx, sp, Mr, N, K, fam, layout, budget, args, world, coll, local, workload):
    """G-BFS over the config space with candidate rounds sharded over the ranks;
    candidates are scored under the timed region's protocol (L2 flushed before every timed
    launch) so the search optimises what the bench reports.  Returns (best, tuning record)."""
    from paper_1909_10616_b200 import dist as tdist
    from paper_1909_10616_b200 import tiletune as tt
    import torch.distributed as dist

    raw, feasible = tt.count_configs(sp, feasible=True)
    width = width_of(args, workload)
    sopts = tt.search_opts(family=fam, seed=args.seed, width=width, layout=layout,
                           measure={"l2_flush": 1 if args.tune_l2_flush else 0})
    ms_fn, observe, cut_fn, mp_fn = tdist.device_measure_set(ctx, sp, sopts, device=local)
    store = tdist.default_store() if (world > 1 and args.assign in ("dynamic", "auto")) else None
    ev = tdist.TrackingEvaluator(observe=observe, measure_set=ms_fn, device=coll if world > 1 else None,
                                 store=store, assign="lpt" if (args.assign in ("dynamic", "auto") and store is None) else args.assign,
                                 space=sp, cut_s=cut_fn, measure_phase=mp_fn if args.two_phase else None)
    ctx.prepare(sp)                      # one-time setup (operands, flush buffer, kernels loaded) off the clock
    ev.warm_up(tt.enumerate_configs(sp, 0, 16))           # host planning code, off the clock too
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    res = tt.gbfs_search(Mr, N, K, budget, sopts, batch=ev)
    tune_wall = tdist.max_over_ranks(time.perf_counter() - t0, coll)
    rec = {"algorithm": "G-BFS (Alg. 1, width %d, rho 5)" % width, "budget": budget, "evals": res.evals,
           "space_raw": raw, "space_feasible": feasible, "frac_raw": res.frac_raw,
           "frac_feasible": res.frac_feasible, "tuning_wall_s": tune_wall, "best_config": res.best,
           "best_cost_us": res.best_cost * 1e6, "s0_cost_us": res.trace[0]["cost"] * 1e6,
           "local_evals": ev.local_evals, "rounds": ev.rounds,
           "speculative_measured": ev.spec_measured, "speculative_used": ev.spec_used,
           "scoring": ("L2 flushed before every timed launch" if args.tune_l2_flush else "warm L2, CUDA-graph replay")
           + "; slow cut min(max(20 cost_min, 1 ms), 50 t_roof), racing at 1.1 cost_min after 2 repeats (reading Z12)",
           "assignment": ev.assign + (" + two-phase rounds" if args.two_phase else ""),
           "round_modes": ev.round_modes}
    if getattr(args, "dump_tuning", None) and (not dist.is_initialized() or dist.get_rank() == 0):
        with open(args.dump_tuning + f".{sp.family}_{Mr}.jsonl", "w") as f:
            for k, (ts, ws, ph) in enumerate(zip(ev.round_times, ev.round_weights, ev.round_phase1)):
                f.write(json.dumps({"round": k, "secs": ts, "weights": ws, "mode": ev.round_modes[k],
                                    "phase1": [list(x) for x in ph]}) + "\n")
            for r in res.trace:
                f.write(json.dumps({"state": r["state"], "cost": r["cost"], "t": r["t_wall_s"]}) + "\n")
    if world == 1:
        # Projection of the sharded search from this run's per-candidate
        # measurement times: the evaluator's own planning code (weights, assignment, speculation,
        # two-phase rounds) replayed for G ranks on the recorded costs (dist.simulate_sharded);
        # the slowest rank gates each phase, + 50 us per exchange, + the measured cost of one
        # dynamic claim; the host search work (everything but measuring) is replicated on every
        # rank.  Not a multi-GPU measurement (the driver's N = 2/4/8 runs measure tuning_wall_s).
        claim = claim_seconds(ctx, sp, ev.round_states[-1][:1])
        rec["projected_sharded_search"] = project_sharded(
            ev, tune_wall, sp, lambda b: tt.scoring_opts(sp, sopts, b, local).cut_s, claim)
    return res.best, rec


def project_sharded(ev, tune_wall, sp, cut_of, claim):
    """Projection of the one-GPU search recorded by ``ev`` (a ShardedEvaluator) onto 2, 4 and 8
    ranks for each assignment variant: host work other than planning (tune_wall - measuring -
    planning) is replicated, the planning and the measurement come from dist.simulate_sharded."""
    from paper_1909_10616_b200 import dist as tdist
    meas = sum(sum(t) for t in ev.round_times)
    host = max(0.0, tune_wall - meas - ev.plan_s)       # replicated host work other than planning
    rcosts = [[ev.known[s] for s in st] for st in ev.round_states]
    proj = {}
    variants = (("two_phase", dict(assign="auto", two_phase=True)), ("lpt", dict(assign="lpt")),
                ("dynamic", dict(assign="dynamic")), ("static", dict(assign="static", speculate=False)))
    for G in (2, 4, 8):
        e = {}
        for name, kw in variants:
            r = tdist.simulate_sharded(ev.round_states, rcosts, ev.round_times, G, space=sp, cut_of=cut_of,
                                       round_phase1=ev.round_phase1, per_round_s=50e-6, per_claim_s=claim, **kw)
            w = host + r["plan_host_s"] + r["wall_s"]
            e[name + "_wall_s"] = w
            e[name + "_speedup"] = tune_wall / w if w > 0 else None
            if name == "two_phase":
                e["two_phase_rounds"] = r["modes"].count("two-phase")
        proj[str(G)] = e
    return {"rounds": ev.rounds, "round_sizes": [len(t) for t in ev.round_times], "measure_s": meas,
            "host_s": host, "plan_s_1gpu": ev.plan_s, "claim_s": claim, "by_gpus": proj,
            "model": "the evaluator's planning code replayed for G ranks on this run's costs and per-candidate "
                     "seconds (dist.simulate_sharded): per phase the slowest rank + 50 us exchange; two_phase "
                     "(the N > 1 default) = probes, exchange, then the rest of each measurement balanced with the "
                     "probes known; dynamic claims cost claim_s (measured here: a TCPStore add + one measure "
                     "call's marshalling); round 0 speculates g(s0) on the idle ranks; host search work other "
                     "than planning replicated (host_s), planning re-timed per G",
            "kind": "projection from 1-GPU per-candidate times"}


def claim_seconds(ctx, sp, states, n=200):
    """Cost of one dynamic claim on this host: a TCPStore add round trip (loopback, as on one
    node) plus one measure call's argument marshalling with nothing to measure."""
    import datetime

    import torch.distributed as dist
    st = dist.TCPStore("127.0.0.1", 0, 1, True, timeout=datetime.timedelta(seconds=10), wait_for_workers=False)
    st.add("warm", 1)
    t0 = time.perf_counter()
    for _ in range(n):
        st.add("claim", 1)
        ctx.measure_set(sp, states, [False] * len(states))
    return (time.perf_counter() - t0) / n


def time_gemm(tt, A, B, C, fam, best, layout, steps, warmup, flush, world, sampler=None):
    """W untimed + `steps` timed launches, L2 flushed before each (outside the event pair);
    barrier + synchronize on both sides; returns per-step ms on the launching stream.  The GEMM
    runs through a tt_plan (checked and bound once), so a step is one library call."""
    import torch
    import torch.distributed as dist
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    plan = tt.GemmPlan(A, B, C, fam, best, layout=layout)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    for _ in range(warmup):
        flush.fill_(1)
        plan.launch(sptr)
    torch.cuda.synchronize()
    if sampler is not None:
        sampler.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(steps):
        flush.fill_(i & 0xFF)                           # L2 flush between steps (outside the events)
        starts[i].record(stream)
        plan.launch(sptr)
        ends[i].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    plan.close()
    return [s.elapsed_time(e) for s, e in zip(starts, ends)]


def spot_check(A_dev, C, Mr, N, K, r0, fam, tn):
    """Untimed check of the timed output on sampled entries against the oracle's definition."""
    import numpy as np

    import synth
    ii = np.array([0, Mr // 3, Mr - 1])
    jj = np.array([N - 1, N // 2, 0])
    if tn:
        Wsh = synth.uniform_f32(1, K, Mr, row0=r0 * K // Mr)      # the rank's W block
        Arows = np.stack([Wsh[:, int(i)] for i in ii])
    else:
        Arows = np.stack([synth.uniform_f32(1, 1, K, row0=r0 + int(i))[0] for i in ii])
    Bh = synth.uniform_f32(2, K, N)
    if fam == 3:
        Arows = synth.bf16_bits_to_f32(synth.to_bf16_bits(Arows))
        Bh = synth.bf16_bits_to_f32(synth.to_bf16_bits(Bh))
    ref = np.array([float(np.dot(Arows[t].astype(np.float64), Bh[:, jj[t]].astype(np.float64))) for t in range(3)])
    got = C.cpu().numpy()[ii, jj]
    return float(np.max(np.abs(got - ref)) / max(1e-30, np.max(np.abs(ref))))


def peak_of(fam, peaks, peak_src, sm_max_mhz):
    if fam == 3:
        return peaks["bf16_tflops"], f"bf16 dense, burst, {peak_src} (MEASURED_PEAKS.json)", "tensor"
    if fam == 2:
        return peaks["bf16_tflops"] * 0.5, f"tf32 = bf16 burst x 0.5 (nominal 1.1/2.25 ratio), {peak_src}", "tensor"
    smx = sm_max_mhz or 1965.0
    return (fp32_fma_peak_tflops(smx), f"fp32 FFMA: 148 SM x 128 lanes x 2 x {smx:.0f} MHz (DESIGN.md §6)", "alu")


def traffic_entry(workload, best):
    """The committed ncu record of this config (DRAM bytes per launch, and for the bench config the
    SM clock and tensor-pipe activity ncu saw inside the kernel), or {}."""
    tp = os.path.join(ROOT, "profiles", f"traffic_{workload}.json")
    if not os.path.exists(tp):
        return {}
    with open(tp) as f:
        tr = json.load(f)
    want = [list(v) for v in best]
    for e in tr.get("configs", [tr]):
        if e.get("config") == want:
            return e
    return {}


def traffic_of(workload, best):
    """DRAM bytes per launch of this config from the committed ncu captures, or None."""
    return traffic_entry(workload, best).get("dram_bytes_per_launch")


def fp32_record(ctx, args, world, coll, local, dev, peaks, peak_src, sm_max, name):
    """A secondary record on an fp32-storage workload.  f32_*: the paper's own arithmetic (fp32
    CUDA-core FFMA, reading Z13) on its square workload, G-BFS at 0.1 % of the raw space from the
    untiled s0, timed steps of the best config against the FFMA peak.  tf32_*: the
    TF32 tcgen05 family (BASELINE config 3's TF32 half), G-BFS over its space, against the tf32
    tensor peak."""
    import torch

    from paper_1909_10616_b200 import tiletune as tt
    Mr, N, K, fam, budget = WORKLOADS[name]
    sp = tt.make_space(Mr, N, K, family=fam)
    best, rec = tune(ctx, sp, Mr, N, K, fam, tt.LAYOUT_NN, budget, args, world, coll, local, name)
    A = torch.empty(Mr, K, device=dev)
    B = torch.empty(K, N, device=dev)
    C = torch.empty(Mr, N, device=dev)
    tt.fill_uniform(A, seed=1)
    tt.fill_uniform(B, seed=2)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    sampler = ClockSampler(local)             # this record's own clocks: it follows a long tuning pass
    per = time_gemm(tt, A, B, C, fam, best, tt.LAYOUT_NN, max(5, min(args.steps, 20)), 3, flush, world,
                    sampler=sampler)
    clocks = sampler.stop()
    ms = statistics.mean(per)
    flops = 2.0 * Mr * N * K
    achieved = flops / (ms * 1e-3) / 1e12
    peak, note, bound = peak_of(fam, peaks, peak_src, sm_max)
    return {"workload": name, "family": "f32_simt" if fam == 1 else "tf32_umma", "value": achieved, "unit": "TFLOP/s", "ms_per_step": ms,
            "best_config": {"m": list(best[0]), "k": list(best[1]), "n": list(best[2])},
            "roofline": {"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "peak_source": note},
            "tuning": rec, "spot_check_err": spot_check(A, C, Mr, N, K, 0, fam, False),
            "clocks": clocks, "l2": "flushed (256 MiB memset) before every timed launch"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="bf16_4096", choices=sorted(WORKLOADS))
    ap.add_argument("--budget", type=int, default=None, help="G-BFS evaluation budget (distinct configs)")
    ap.add_argument("--width", type=int, default=None,
                    help="G-BFS states popped per round W (reading Z9): the same for every GPU count; "
                         "default per workload (DEFAULT_WIDTH, else 16)")
    ap.add_argument("--assign", choices=["auto", "lpt", "static", "dynamic"], default="auto",
                    help="how a round's candidates are spread over the ranks (paper_1909_10616_b200/dist.py)")
    ap.add_argument("--layout", choices=["nn", "tn"], default="nn",
                    help="tn: A stored as W[K][M] (the paper's perceptron Y = W^T X, P:372)")
    ap.add_argument("--one-phase", dest="two_phase", action="store_false",
                    help="sharded rounds measure each candidate whole on one rank (default: two-phase rounds, "
                         "probes first, then the rest balanced with the probes known)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--ref-rows", type=int, default=16)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--fp32-workload", default="f32_2048,f32_4096",
                    help="comma-separated workloads of the fp32 (paper arithmetic) records: the first is 'fp32', "
                         "the rest 'fp32_more' (f32_2048 = BASELINE config 3; f32_4096 = the bf16 headline's shape)")
    ap.add_argument("--tf32-workload", default="tf32_2048",
                    help="workload of the TF32 record ('tf32'; BASELINE config 3's TF32 half); empty: none")
    ap.add_argument("--no-fp32", action="store_true", help="skip the fp32 and tf32 records")
    ap.add_argument("--config", default=None, help="skip tuning and use this config (JSON triple)")
    ap.add_argument("--dump-tuning", default=None, help="write per-round / per-candidate tuning data to PATH.*.jsonl")
    ap.add_argument("--tune-warm", dest="tune_l2_flush", action="store_false",
                    help="score candidates warm (CUDA-graph replay) instead of with the timed region's L2 flush")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")

    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    from paper_1909_10616_b200 import dist as tdist
    from paper_1909_10616_b200 import tiletune as tt

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TT_BENCH_SHARE_GPU=1: every rank on cuda:0 with gloo collectives -- exercises the N > 1 code
    # path (sharded tuning, row partition, max-over-ranks) on a one-GPU box; its timings are not
    # a scaling measurement (the ranks share one device).
    share = os.environ.get("TT_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    coll = torch.device("cpu") if share else dev     # device of the small collective tensors

    Mr, N, K, fam, default_budget = WORKLOADS[args.workload]
    strong = args.workload == "bf16_8192"
    if strong:                       # fixed total M, rows split over the ranks
        M = Mr
        Mr = M // world
    else:                            # fixed per-rank work (weak scaling)
        M = Mr * world
    budget = args.budget if args.budget is not None else default_budget
    ctx = tt.Context(local, input_seed=1)
    layout = tt.LAYOUT_TN if args.layout == "tn" else tt.LAYOUT_NN
    sp = tt.make_space(Mr, N, K, family=fam, layout=layout)

    # ---------------- 1. tuning pass (G-BFS, candidates sharded over ranks) ----------------
    if args.config:
        best = tuple(tuple(v) for v in json.loads(args.config))
        tune_rec = None
    else:
        best, tune_rec = tune(ctx, sp, Mr, N, K, fam, layout, budget, args, world, coll, local, args.workload)
    info = tt.binding(sp, best)

    # ---------------- 2. timed steps of the best-found GEMM on this rank's row shard ----------
    bf16 = fam == 3
    r0, r1 = tdist.row_shard(M, world, rank)
    tn = layout == tt.LAYOUT_TN
    # NN: A rows are global rows r0.. of the full A.  TN: each rank's W shard [K][Mr] is its own
    # recipe block (index offset rank * K * Mr): the row blocks of Y = W^T X are independent.
    A = torch.empty((K, Mr) if tn else (Mr, K), device=dev, dtype=torch.bfloat16 if bf16 else torch.float32)
    B = torch.empty(K, N, device=dev, dtype=A.dtype)
    C = torch.empty(Mr, N, device=dev, dtype=torch.float32)
    tt.fill_uniform(A, seed=1, idx0=r0 * K)        # NN: global row indices; TN: rank block offset
    tt.fill_uniform(B, seed=2)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    sampler = ClockSampler(local)
    per = time_gemm(tt, A, B, C, fam, best, layout, args.steps, args.warmup, flush, world, sampler=sampler)
    clocks = sampler.stop()
    ms_local = sum(per) / len(per)
    ms = tdist.max_over_ranks(ms_local, coll)
    flops_rank = 2.0 * Mr * N * K
    value = world * flops_rank / (ms * 1e-3) / 1e12                 # whole-job TFLOP/s
    spot_err = spot_check(A, C, Mr, N, K, r0, fam, tn)

    # ---------------- 3. e2e through tt_gemm_host (pinned host buffers) -----------------------
    Ah_t = A.cpu().pin_memory()
    Bh_t = B.cpu().pin_memory()
    Ch_t = torch.empty(Mr, N, dtype=torch.float32).pin_memory()
    ctx.gemm_host(Ah_t, Bh_t, Ch_t, fam, best, layout=layout)       # warm (allocates staging)
    e2e_steps = min(args.steps, 5)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        ctx.gemm_host(Ah_t, Bh_t, Ch_t, fam, best, layout=layout)
    e2e_s = tdist.max_over_ranks((time.perf_counter() - t0) / e2e_steps, coll)
    e2e_val = world * flops_rank / e2e_s / 1e12
    h2d = Ah_t.numel() * Ah_t.element_size() + Bh_t.numel() * Bh_t.element_size()
    d2h = Ch_t.numel() * 4

    # ---------------- 4. roofline, the paper's fp32 arithmetic, cpu baseline -------------------
    peaks, peak_src = load_peaks()
    peak, peak_note, bound = peak_of(fam, peaks, peak_src, clocks.get("sm_max_mhz"))
    achieved = flops_rank / (ms_local * 1e-3) / 1e12
    # memory side of the same launch: compulsory bytes (A, B in at the input width, C out fp32)
    in_bytes = 2 if fam == 3 else 4
    comp_bytes = (Mr * K + K * N) * in_bytes + Mr * N * 4
    hbm_side = {"compulsory_bytes": comp_bytes, "achieved_gbs": comp_bytes / (ms_local * 1e-3) / 1e9,
                "peak_gbs": peaks["hbm_gbs"], "frac": comp_bytes / (ms_local * 1e-3) / 1e9 / peaks["hbm_gbs"],
                "t_floor_us": {"memory": comp_bytes / (peaks["hbm_gbs"] * 1e9) * 1e6,
                               "compute": flops_rank / (peak * 1e12) * 1e6}}
    traffic = traffic_of(args.workload, best)
    fp32 = None
    fp32_more = []
    if not args.no_fp32 and fam != 1:
        names = [w for w in args.fp32_workload.split(",") if w]
        for w in names:
            if w not in WORKLOADS or not w.startswith("f32"):
                raise SystemExit(f"--fp32-workload: unknown fp32 workload {w}")
        recs = [fp32_record(ctx, args, world, coll, local, dev, peaks, peak_src, clocks.get("sm_max_mhz"), w)
                for w in names]
        fp32, fp32_more = recs[0], recs[1:]
    tf32 = None
    if not args.no_fp32 and fam != 2 and args.tf32_workload:
        if args.tf32_workload not in WORKLOADS or not args.tf32_workload.startswith("tf32"):
            raise SystemExit(f"--tf32-workload: unknown tf32 workload {args.tf32_workload}")
        tf32 = fp32_record(ctx, args, world, coll, local, dev, peaks, peak_src, clocks.get("sm_max_mhz"),
                           args.tf32_workload)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, sample = cpu_oracle_sample(Mr, N, K, fam, seconds=args.cpu_seconds)
        cpu = {"value": v, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": sample}

    if rank == 0:
        line = {
            "metric": "best-found GEMM TFLOP/s", "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": FAMILY_DTYPE[fam],
            "data": "synthetic",
            "config": {"workload": args.workload, "M_per_rank": Mr, "M_total": M, "N": N, "K": K,
                       "layout": args.layout,
                       "family": {1: "f32_simt", 2: "tf32_umma", 3: "bf16_umma"}[fam],
                       "parallelism": f"row-partitioned x{world}, candidate sharding x{world}" + (" (shared GPU, gloo: code-path check)" if share else ""),
                       "l2": "flushed (256 MiB memset) before every timed launch",
                       "best_config": {"m": list(best[0]), "k": list(best[1]), "n": list(best[2])},
                       "launch": {"grid": info.grid_x, "cluster": info.cluster_x, "tile": [info.tile_m, info.tile_n,
                                  info.tile_k], "stages": info.stages, "smem": info.smem_bytes,
                                  "split_tiles": info.split_tiles}},
            "tuning": tune_rec,
            "pct_of_peak": 100.0 * achieved / peak,
            "roofline": {"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_note,
                         "algorithmic": f"2*M*N*K = {flops_rank:.4g} flop per launch", "hbm_side": hbm_side},
            "fp32": fp32,
            "fp32_more": fp32_more,
            "tf32": tf32,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "path": "tt_gemm_host (pinned host A,B -> device -> C host)"},
            "gpu_launches": args.steps,
            "clocks": dict(clocks, **({"kernel_sm_ghz_ncu": traffic_entry(args.workload, best)["sm_clock_ghz_ncu"],
                                        "note": "NVML samples every 2 ms land mostly between the ~0.1 ms launches "
                                                "(flush gaps); kernel_sm_ghz_ncu is the clock ncu measured inside "
                                                "one launch of this config (profiles/traffic_*.json)"}
                                       if traffic_entry(args.workload, best).get("sm_clock_ghz_ncu") else {})),
            "spot_check_err": spot_err,
            "per_step_ms": {"min": min(per), "median": statistics.median(per), "max": max(per)},
        }
        print(json.dumps(line))
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
