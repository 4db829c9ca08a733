"""Summarise tools/width_study.sh: per G-BFS width W, the best-found cost over 10 seeds and the
evaluations a seed needed to reach its final best (CSV traces in gpurun_out/r11_width_W*.csv)."""
import csv
import glob
import os
import re
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = []
for path in sorted(glob.glob(os.path.join(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out"),
                                          "r11_width_W*.csv")), key=lambda p: int(re.findall(r"W(\d+)", p)[0])):
    W = int(re.findall(r"W(\d+)", path)[0])
    by = {}
    for r in csv.DictReader(open(path)):
        by.setdefault((r["strategy"], int(r["trial_seed"])), []).append(r)
    for strat in ("gbfs", "random"):
        bests, to_best = [], []
        for (s, seed), rs in by.items():
            if s != strat:
                continue
            rs.sort(key=lambda r: int(r["eval_index"]))
            final = float(rs[-1]["best_so_far_s"])
            bests.append(final)
            to_best.append(next(int(r["eval_index"]) for r in rs if float(r["best_so_far_s"]) == final))
        if bests:
            rows.append((W, strat, statistics.median(bests) * 1e6, min(bests) * 1e6, max(bests) * 1e6,
                         statistics.median(to_best)))
print("| W | strategy | best-found median [min, max] (us) | evaluations to final best (median) |")
print("|---|---|---|---|")
for W, strat, med, lo, hi, tb in rows:
    if strat == "random" and W != 1:
        continue
    print(f"| {W if strat == 'gbfs' else '-'} | {strat} | {med:.2f} [{lo:.2f}, {hi:.2f}] | {tb:.0f} |")
