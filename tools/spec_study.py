"""Offline study of speculative measurement for the sharded G-BFS.

Runs the library's G-BFS (Alg. 1, width W, rho 5) on the CPU with the measured costs of every
feasible bf16 4096^3 config (profiles/r11_exhaustive) as its cost table, records the rounds, and
projects the wall time of the same traversal sharded over G ranks under a per-candidate time model
of the bench's scoring rules (reading Z12: flushed launches, racing after 2 repeats at 1.1 cost_min).
Prints the projected speedups (planning host time included) for each assignment variant of
dist.ShardedEvaluator, and the bound of an LPT packing with the true times.  Not a measurement;
the GPU bench's projection uses recorded per-candidate times instead.

usage: python tools/spec_study.py [table.json] [budget 128] [width 16] [claim seconds 21e-6]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1909_10616_b200 import dist as tdist  # noqa: E402
from paper_1909_10616_b200 import tiletune as tt  # noqa: E402


def load_table(path):
    d = json.load(open(path))
    tab = {}
    for txt, c in d["all"]:
        j = json.loads(txt)
        tab[(tuple(j["m"]), tuple(j["k"]), tuple(j["n"]))] = c
    return tab, d["problem"]


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles/r11_exhaustive/r11_exh_bf16_4096.json")
    budget = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    width = int(sys.argv[3]) if len(sys.argv) > 3 else 16
    claim = float(sys.argv[4]) if len(sys.argv) > 4 else 21e-6   # measured on the GPU host (bench claim_s)
    tab, (M, N, K) = load_table(path)
    sp = tt.make_space(M, N, K, family=tt.FAM_BF16_UMMA)
    over = 75e-6                                                # flush + host per launch

    def secs(s, best):
        c = tab[s]
        n = 11 if best == float("inf") or c <= 1.1 * best else 3   # racing (Z12)
        return n * (c + over)

    res = {}
    for seed in range(10):
        rounds = []
        best = [float("inf")]

        def batch(states):
            rounds.append([(s, secs(s, best[0])) for s in states])
            cs = [tab[s] for s in states]
            best[0] = min([best[0]] + cs)
            return cs

        r = tt.gbfs_search(M, N, K, budget, tt.search_opts(family=tt.FAM_BF16_UMMA, seed=seed, width=width), batch=batch)
        st = [[s for s, _ in rd] for rd in rounds]
        ti = [[t for _, t in rd] for rd in rounds]
        costs = [[tab[s] for s in rd] for rd in st]
        one = sum(map(sum, ti))
        for G in (2, 4, 8):
            for name, kw in (("lpt, no speculation", dict(assign="lpt", speculate=False)),
                             ("lpt", dict(assign="lpt")), ("dynamic", dict(assign="dynamic")),
                             ("auto", dict(assign="auto")), ("two-phase (auto)", dict(assign="auto", two_phase=True))):
                w = tdist.simulate_sharded(st, costs, ti, G, space=sp, per_claim_s=claim, **kw)
                res.setdefault((G, name), []).append(one / (w["wall_s"] + w["plan_host_s"]))
            # bound: round 0 speculated, every later round LPT-packed with the true times
            tot = ti[0][0]
            for t in ti[2:]:
                load = [0.0] * G
                for x in sorted(t, reverse=True):
                    load[load.index(min(load))] += x
                tot += max(load)
            res.setdefault((G, "LPT with true times (bound)"), []).append(one / tot)
        print("seed", seed, "rounds", [len(x) for x in st], "one-GPU measure %.1f ms" % (one * 1e3),
              "best %.2f us" % (r.best_cost * 1e6))
    for k, v in sorted(res.items()):
        v = sorted(v)
        print("G=%d %-30s median %.2f  min %.2f  max %.2f" % (k[0], k[1], v[len(v) // 2], v[0], v[-1]))


if __name__ == "__main__":
    main()
