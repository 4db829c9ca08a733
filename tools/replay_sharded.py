"""Replay a recorded one-GPU tuning run (bench.py --dump-tuning PATH -> PATH.<fam>_<M>.jsonl)
through dist.simulate_sharded for every assignment variant, and print the per-round times next to
the bound of an LPT packing of the recorded (phase) times.  Projection tooling, not a test.

    python tools/replay_sharded.py profiles/r12_tune_bf16_4096.jsonl [G ...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1909_10616_b200 import dist as tdist  # noqa: E402
from paper_1909_10616_b200 import tiletune as tt  # noqa: E402


def load(path):
    rows = [json.loads(line) for line in open(path)]
    rounds = [r for r in rows if "round" in r]
    trace = [r for r in rows if "state" in r]
    states, costs, i = [], [], 0
    for r in rounds:
        n = len(r["secs"])
        states.append([tuple(tuple(f) for f in t["state"]) for t in trace[i:i + n]])
        costs.append([t["cost"] for t in trace[i:i + n]])
        i += n
    return states, costs, [r["secs"] for r in rounds], [tuple(r.get("phase1", ([], [], []))) for r in rounds]


def main():
    path = sys.argv[1]
    Gs = [int(g) for g in sys.argv[2:]] or [2, 4, 8]
    states, costs, times, ph = load(path)
    fam = int(os.path.basename(path).split("_")[-2].split(".")[-1]) if "." in path else 3
    M = int(path.rsplit("_", 1)[1].split(".")[0])
    sp = tt.make_space(M, M, M, family=fam)
    sopts = tt.search_opts(family=fam, measure={"l2_flush": 1})
    cut_of = lambda b: tt.scoring_opts(sp, sopts, b, -1).cut_s  # noqa: E731
    one = sum(map(sum, times))
    print("rounds", [len(s) for s in states], "one-GPU measuring %.2f ms" % (one * 1e3))
    for G in Gs:
        for name, kw in (("two-phase", dict(assign="auto", two_phase=True)), ("lpt", dict(assign="lpt")),
                         ("dynamic", dict(assign="dynamic")), ("static", dict(assign="static", speculate=False))):
            r = tdist.simulate_sharded(states, costs, times, G, space=sp, cut_of=cut_of, round_phase1=ph,
                                       per_claim_s=21e-6, **kw)
            print("G=%d %-10s measuring %.2f ms + planning %.2f ms -> %.2fx of the measuring" %
                  (G, name, r["wall_s"] * 1e3, r["plan_host_s"] * 1e3, one / (r["wall_s"] + r["plan_host_s"])))

        def lpt(ts):
            load = [0.0] * G
            for x in sorted(ts, reverse=True):
                load[load.index(min(load))] += x
            return max(load)
        bound = times[0][0]                   # round 0 = s0; rounds 1+ packed with the true phase times
        for k in range(1, len(times)):
            s1 = ph[k][0] if len(ph[k]) and len(ph[k][0]) else [0.0] * len(times[k])
            bound += lpt(s1) + lpt([t - a for t, a in zip(times[k], s1)])
        print("G=%d bound (true-time LPT per phase, round 1 included): %.2f ms -> %.2fx" % (G, bound * 1e3, one / bound))


if __name__ == "__main__":
    main()
