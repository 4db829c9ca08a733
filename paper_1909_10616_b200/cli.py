"""Command-line front end (SPEC S:440-526 subcommands; every step runs in libtiletune).

    python -m paper_1909_10616_b200.cli count     --m 1024 --k 1024 --n 1024 [--dm 4 --dk 2 --dn 4] [--family bf16]
    python -m paper_1909_10616_b200.cli enumerate --m 64 --k 64 --n 64 [--limit 20] [--feasible]
    python -m paper_1909_10616_b200.cli bench     --m 4096 --k 4096 --n 4096 --family bf16 --config '{"m":[..],"k":[..],"n":[..]}'
    python -m paper_1909_10616_b200.cli tune      --m 512 --k 512 --n 512 --family f32 --strategy gbfs --max-evals 484 --seeds 0,1 --out runs/t
    python -m paper_1909_10616_b200.cli compare   --m 512 --k 512 --n 512 --family f32 --strategies gbfs,na2c,random --max-evals 484 --seeds 0-9 --out runs/c

Problems are given in the paper's (m, k, n) order; C[m x n] = A[m x k] B[k x n].
Configurations use the canonical text form {"m":[...],"k":[...],"n":[...]}, outer -> inner.
``tune`` / ``compare`` write a CSV trace (one row per measured state) and a JSON summary
with the box-plot statistics of the paper's Fig. 8(b) (min, Q1, median, mean, Q3, max over seeds,
P:397).  Cost sources: ``--backend device`` (the B200 evaluator) or ``synthetic`` (S:172 landscape,
for desk runs without a GPU).
"""
from __future__ import annotations

import argparse
import csv
import json
import math
import os
import statistics
import sys
import time
from typing import List

from . import tiletune as tt

FAMILIES = {"none": tt.FAM_NONE, "f32": tt.FAM_F32_SIMT, "tf32": tt.FAM_TF32_UMMA, "bf16": tt.FAM_BF16_UMMA}


def encode(s) -> str:
    return '{"m":[%s],"k":[%s],"n":[%s]}' % tuple(",".join(str(v) for v in s[a]) for a in range(3))


def decode(text: str, depths=(4, 2, 4)):
    d = json.loads(text)
    if not isinstance(d, dict) or set(d) != {"m", "k", "n"}:
        raise ValueError("config must have keys m, k, n")
    s = []
    for key, dep in zip(("m", "k", "n"), depths):
        v = d[key]
        if not isinstance(v, list) or not all(isinstance(x, int) and not isinstance(x, bool) for x in v):
            raise ValueError(f"non-integer entry in {key}")
        if len(v) != dep:
            raise ValueError(f"{key} has {len(v)} factors, depth is {dep}")
        s.append(tuple(v))
    return tuple(s)


def parse_seeds(text: str) -> List[int]:
    out = []
    for part in text.split(","):
        if "-" in part:
            a, b = part.split("-")
            out.extend(range(int(a), int(b) + 1))
        elif part:
            out.append(int(part))
    return out


def box(values):
    xs = sorted(values)
    n = len(xs)

    def q(p):
        if n == 1:
            return xs[0]
        pos = p * (n - 1)
        lo = int(math.floor(pos))
        hi = min(lo + 1, n - 1)
        return xs[lo] + (xs[hi] - xs[lo]) * (pos - lo)

    return {"min": xs[0], "q1": q(0.25), "median": q(0.5), "mean": sum(xs) / n, "q3": q(0.75), "max": xs[-1],
            "n": n}


def synthetic_cost(args):
    """S:175 quadratic-in-log2 landscape with per-slot targets at half the log2 of each dim."""
    dims = (args.m, args.k, args.n)
    depths = (args.dm, args.dk, args.dn)
    targets = [[math.log2(d) / dep for _ in range(dep)] for d, dep in zip(dims, depths)]

    def f(s):
        c = 1.0
        for a in range(3):
            for i, v in enumerate(s[a]):
                c += (math.log2(v) - targets[a][i]) ** 2
        return c
    return f


LAYOUTS = {"nn": tt.LAYOUT_NN, "tn": tt.LAYOUT_TN}


def _space(args):
    return tt.make_space(args.m, args.n, args.k, args.dm, args.dk, args.dn, FAMILIES[args.family], LAYOUTS[args.layout])


def cmd_count(args):
    raw, feas = tt.count_configs(_space(args), feasible=True)
    print(raw if args.family == "none" else f"{raw} raw, {feas} feasible ({args.family})")


def cmd_enumerate(args):
    sp = _space(args)
    if args.feasible:
        cfgs, ranks = tt.enumerate_feasible(sp)
        for r, s in list(zip(ranks, cfgs))[:args.limit]:
            print(r, encode(s))
    else:
        for r, s in enumerate(tt.enumerate_configs(sp, 0, args.limit)):
            print(r, encode(s))


def cmd_bench(args):
    sp = _space(args)
    s = decode(args.config, (args.dm, args.dk, args.dn))
    ctx = tt.Context(args.device)
    smp = ctx.measure(sp, s, tt.measure_opts(repeats=args.repeats, warmup=args.warmup))
    flops = 2.0 * args.m * args.n * args.k
    print(json.dumps({"config": encode(s), "cost_s": smp.cost_s, "mean_s": smp.mean_s, "min_s": smp.min_s,
                      "repeats": smp.repeats, "number": smp.number, "tflops": flops / smp.cost_s / 1e12}))


def _run(strategy, args, seed, ctx):
    opts = tt.search_opts(family=FAMILIES[args.family], dm=args.dm, dk=args.dk, dn=args.dn, seed=seed,
                          rho=args.rho, width=args.width, steps_T=args.steps, epsilon=args.epsilon,
                          batch=args.batch_size, gamma=args.gamma, steps_T_floor=args.steps_floor,
                          steps_T_decay_every=args.decay_every, layout=LAYOUTS[args.layout],
                          budget_seconds=args.max_seconds or 0.0,
                          measure={"repeats": args.repeats, "warmup": args.warmup})
    if args.start_config:
        opts.has_s0 = 1
        opts.s0 = tt.to_config(decode(args.start_config, (args.dm, args.dk, args.dn)))
    fn = {"gbfs": tt.gbfs_search, "na2c": tt.na2c_search, "random": tt.random_search}[strategy]
    recorded = _load_resume(args, strategy, seed)
    if recorded is None and getattr(args, "shared_cache", False) and args.backend == "device":
        # One measurement per distinct state for the whole compare run: every search that reaches
        # a state gets the cost measured the first time (the same hardware test, so strategies are
        # compared on common measurements).  `equiv_wall` = what this search's own measurements
        # took when they were first made, i.e. its stand-alone tuning wall-time.
        sp = _space(args)
        mo = tt.measure_opts(repeats=args.repeats, warmup=args.warmup)
        cache = args._cost_cache
        equiv = [0.0]
        best = [float("inf")]

        def cached(states):
            out = []
            for s in states:
                if s not in cache:
                    t0 = time.perf_counter()
                    # --scoring: the searches' own scoring rules at this search's incumbent (slow
                    # cut, racing, partial-grid probe; reading Z12), as the DEVICE source applies them
                    m = tt.scoring_opts(sp, opts, best[0], args.device) if args.scoring else mo
                    c = ctx.measure(sp, s, m).cost_s
                    cache[s] = (c, time.perf_counter() - t0)
                out.append(cache[s][0])
                equiv[0] += cache[s][1]
                best[0] = min(best[0], cache[s][0])
            return out
        res = fn(args.m, args.n, args.k, args.max_evals, opts, batch=cached)
        res.equiv_wall_s = equiv[0]
        return res
    if recorded is None:
        kw = {"ctx": ctx} if args.backend == "device" else {"cost": synthetic_cost(args)}
        return fn(args.m, args.n, args.k, args.max_evals, opts, **kw)
    # Resume (SURVEY §5 checkpoint): a search is a deterministic function of (seed, cost sequence),
    # so replaying the recorded costs rebuilds Q / S_v / H_v / the RNG state exactly and the search
    # continues live once it reaches states the trace does not hold.
    sp = _space(args)
    live = synthetic_cost(args) if args.backend == "synthetic" else None

    def batch(states):
        out = []
        for s in states:
            if s in recorded:
                out.append(recorded[s])
            elif live is not None:
                out.append(live(s))
            else:
                out.append(ctx.measure(sp, s, tt.measure_opts(repeats=args.repeats, warmup=args.warmup)).cost_s)
        return out
    return fn(args.m, args.n, args.k, args.max_evals, opts, batch=batch)


def _load_resume(args, strategy, seed):
    if not getattr(args, "resume", None):
        return None
    rec = {}
    with open(args.resume, newline="") as f:
        for r in csv.DictReader(f):
            if r["strategy"] == strategy and int(r["trial_seed"]) == seed:
                rec[decode(r["config"], (args.dm, args.dk, args.dn))] = float(r["cost_s"])
    return rec


def _tune(args, strategies):
    seeds = parse_seeds(args.seeds)
    ctx = tt.Context(args.device) if args.backend == "device" else None
    os.makedirs(os.path.dirname(os.path.abspath(args.out)) or ".", exist_ok=True)
    rows, summary = [], {"problem": {"m": args.m, "k": args.k, "n": args.n, "d": [args.dm, args.dk, args.dn],
                                     "family": args.family, "backend": args.backend},
                         "seeds": seeds, "max_evals": args.max_evals, "strategies": {}}
    flops = 2.0 * args.m * args.n * args.k
    args._cost_cache = {}
    for strat in strategies:
        bests, walls, equivs = [], [], []
        for seed in seeds:
            res = _run(strat, args, seed, ctx)
            bests.append(res.best_cost)
            walls.append(res.wall_s)
            if hasattr(res, "equiv_wall_s"):
                equivs.append(res.equiv_wall_s)
            for r in res.trace:
                rows.append([strat, seed, r["eval_index"], f"{r['t_wall_s']:.6f}", encode(r["state"]), repr(r["cost"]),
                             repr(r["best"]), f"{(r['eval_index'] + 1) / res.space_raw:.9f}"])
            print(f"{strat} seed {seed}: best {res.best_cost:.6g} after {res.evals} evals "
                  f"({100 * res.frac_raw:.4f}% of {res.space_raw}, {res.wall_s:.1f} s) {encode(res.best)}", flush=True)
        st = {"best_cost": box(bests), "wall_s": box(walls)}
        if equivs:
            st["equiv_wall_s"] = box(equivs)
            summary["distinct_states_measured"] = len(args._cost_cache)
        if args.backend == "device":
            st["best_tflops"] = box([flops / c / 1e12 for c in bests])
        summary["strategies"][strat] = st
        _write_outputs(args.out, rows, summary)     # after every strategy: a cut-off run keeps its finished part
    print(json.dumps(summary["strategies"], indent=1))


def _write_outputs(out, rows, summary):
    with open(out + ".csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["strategy", "trial_seed", "eval_index", "wall_clock_s", "config", "cost_s", "best_so_far_s",
                    "fraction_explored"])
        w.writerows(rows)
    with open(out + ".json", "w") as f:
        json.dump(summary, f, indent=1)


def cmd_tune(args):
    _tune(args, [args.strategy])


def cmd_compare(args):
    strategies = [s for s in args.strategies.split(",") if s]
    if len(strategies) < 2:
        raise SystemExit("compare needs at least two strategies (S:502)")
    _tune(args, strategies)


def main(argv=None):
    ap = argparse.ArgumentParser(prog="tiletune")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(p):
        p.add_argument("--m", type=int, required=True)
        p.add_argument("--k", type=int, required=True)
        p.add_argument("--n", type=int, required=True)
        p.add_argument("--dm", type=int, default=4)
        p.add_argument("--dk", type=int, default=2)
        p.add_argument("--dn", type=int, default=4)
        p.add_argument("--family", choices=sorted(FAMILIES), default="none")
        p.add_argument("--device", type=int, default=0)
        p.add_argument("--layout", choices=["nn", "tn"], default="nn",
                       help="tn: A given as W[k][m], the paper's Y = W^T X (P:372)")

    p = sub.add_parser("count")
    common(p)
    p.set_defaults(fn=cmd_count)
    p = sub.add_parser("enumerate")
    common(p)
    p.add_argument("--limit", type=int, default=20)
    p.add_argument("--feasible", action="store_true")
    p.set_defaults(fn=cmd_enumerate)
    p = sub.add_parser("bench")
    common(p)
    p.add_argument("--config", required=True)
    p.add_argument("--repeats", type=int, default=10)
    p.add_argument("--warmup", type=int, default=2)
    p.set_defaults(fn=cmd_bench)
    for name, fn in (("tune", cmd_tune), ("compare", cmd_compare)):
        p = sub.add_parser(name)
        common(p)
        if name == "tune":
            p.add_argument("--strategy", choices=["gbfs", "na2c", "random"], default="gbfs")
        else:
            p.add_argument("--strategies", default="gbfs,na2c,random")
        p.add_argument("--backend", choices=["device", "synthetic"], default="device")
        p.add_argument("--seeds", default="0")
        p.add_argument("--max-evals", type=int, default=100)
        p.add_argument("--max-seconds", type=float, default=0.0)
        p.add_argument("--rho", type=int, default=5)
        p.add_argument("--width", type=int, default=1)
        p.add_argument("--steps", type=int, default=3)
        p.add_argument("--steps-floor", type=int, default=1, help="T decay floor (P:336)")
        p.add_argument("--decay-every", type=int, default=0, help="decrease T by 1 every this many episodes")
        p.add_argument("--epsilon", type=float, default=0.8)
        p.add_argument("--batch-size", type=int, default=16)
        p.add_argument("--gamma", type=float, default=0.9)
        p.add_argument("--repeats", type=int, default=10)
        p.add_argument("--warmup", type=int, default=2)
        p.add_argument("--start-config", default=None)
        p.add_argument("--out", default="runs/tune")
        p.add_argument("--resume", default=None, help="CSV trace of an earlier run: replay it, then continue")
        p.add_argument("--scoring", action="store_true",
                       help="shared-cache measurements use the searches' scoring rules (cut, racing; reading Z12)")
        p.add_argument("--shared-cache", action="store_true",
                       help="device: measure each distinct state once for the whole run (common measurements)")
        p.set_defaults(fn=fn)
    args = ap.parse_args(argv)
    args.fn(args)


if __name__ == "__main__":
    main()
