#!/bin/bash
# Final round-2 refresh (tag r13) of the paper-methodology comparisons with the final kernels (K1
# TMA-fed B, one barrier per slab) and evaluator: G-BFS (W = 1, Alg. 1) vs N-A2C vs random search,
# 10 seeds, common measurements scored by the searches' own rules.  1024^3 is the paper's main
# experiment shape, 2048^3 BASELINE config 3.
set -u
OUT=gpurun_out
timeout 1800 python -m paper_1909_10616_b200.cli compare --m 1024 --k 1024 --n 1024 --family f32 \
    --max-evals 900 --seeds 0-9 --repeats 5 --shared-cache --scoring --out $OUT/r13_cmp_f32_1024 > $OUT/r13_cmp_f32_1024.log 2>&1
timeout 2400 python -m paper_1909_10616_b200.cli compare --m 2048 --k 2048 --n 2048 --family f32 \
    --max-evals 1590 --seeds 0-9 --repeats 5 --shared-cache --scoring --out $OUT/r13_cmp_f32_2048 > $OUT/r13_cmp_f32_2048.log 2>&1
tail -n 14 $OUT/r13_cmp_*.log
