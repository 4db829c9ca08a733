"""Exhaustive device sweep of a feasible set vs G-BFS at 0.1 % of the raw space (SURVEY O10 pin:
G-BFS best within a stated tolerance of the exhaustive best).

    python tools/exhaustive.py --m 512 --k 512 --n 512 --family f32 --budget 484 --seeds 0-9 --out gpurun_out/exh_f32_512
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_10616_b200 import cli, tiletune as tt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, required=True)
ap.add_argument("--k", type=int, required=True)
ap.add_argument("--n", type=int, required=True)
ap.add_argument("--family", default="f32")
ap.add_argument("--budget", type=int, default=484)
ap.add_argument("--seeds", default="0-9")
ap.add_argument("--repeats", type=int, default=3)
ap.add_argument("--out", required=True)
a = ap.parse_args()
fam = cli.FAMILIES[a.family]
sp = tt.make_space(a.m, a.n, a.k, family=fam)
ctx = tt.Context(0)
cfgs, ranks = tt.enumerate_feasible(sp)
t0 = time.time()
mo = tt.measure_opts(repeats=a.repeats, cut_s=0.02)
costs = []
for s in cfgs:
    costs.append(ctx.measure(sp, s, mo).cost_s)
sweep_s = time.time() - t0
order = sorted(range(len(cfgs)), key=lambda i: costs[i])
best = costs[order[0]]
res = {"problem": [a.m, a.k, a.n], "family": a.family, "feasible": len(cfgs), "sweep_s": sweep_s,
       "exhaustive_best_s": best, "exhaustive_best": cli.encode(cfgs[order[0]]),
       "top10": [(cli.encode(cfgs[i]), costs[i]) for i in order[:10]], "gbfs": [],
       "all": [(cli.encode(c), x) for c, x in zip(cfgs, costs)]}
flops = 2.0 * a.m * a.n * a.k
for seed in cli.parse_seeds(a.seeds):
    r = tt.gbfs_search(a.m, a.n, a.k, a.budget, tt.search_opts(family=fam, seed=seed, measure={"repeats": a.repeats}),
                       ctx=ctx)
    res["gbfs"].append({"seed": seed, "best_s": r.best_cost, "ratio_to_exhaustive": r.best_cost / best,
                        "frac_raw": r.frac_raw, "wall_s": r.wall_s, "best": cli.encode(r.best)})
    print(seed, r.best_cost / best, flush=True)
res["exhaustive_best_tflops"] = flops / best / 1e12
with open(a.out + ".json", "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps({k: v for k, v in res.items() if k not in ("top10", "gbfs", "all")}))
