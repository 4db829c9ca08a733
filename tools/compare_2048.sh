#!/bin/bash
# SURVEY C3 / paper P:397 "N-A2C outperform[s] G-BFS for larger matrix sizes (2048)": (2048)^3 fp32,
# 0.1 % of 1 589 952 states = 1590 evaluations, 10 seeds, G-BFS vs N-A2C vs random.  Each distinct
# state is measured once for the whole run (--shared-cache); per-search stand-alone tuning time is
# reported as equiv_wall_s.
OUT=gpurun_out
timeout ${CMP_TIMEOUT:-6000} python -m paper_1909_10616_b200.cli compare --m 2048 --k 2048 --n 2048 --family f32 \
    --max-evals 1590 --seeds 0-9 --repeats 5 --shared-cache --out $OUT/cmp_f32_2048 > $OUT/cmp_f32_2048.log 2>&1
tail -40 $OUT/cmp_f32_2048.log
