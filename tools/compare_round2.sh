#!/bin/bash
# Round-2 refresh of the paper-methodology comparisons (Fig. 7-8, P:375 / P:397; BASELINE configs
# 2-3): G-BFS vs N-A2C vs random search, 10 seeds, common measurements (--shared-cache) scored by
# the searches' own rules (--scoring: slow cut, racing; reading Z12).  Outputs gpurun_out/r11_cmp_*.
set -u
OUT=gpurun_out
timeout 2400 python -m paper_1909_10616_b200.cli compare --m 2048 --k 2048 --n 2048 --family f32 \
    --max-evals 1590 --seeds 0-9 --repeats 5 --shared-cache --scoring --out $OUT/r11_cmp_f32_2048 > $OUT/r11_cmp_f32_2048.log 2>&1
timeout 1200 python -m paper_1909_10616_b200.cli compare --m 512 --k 512 --n 512 --family f32 \
    --max-evals 484 --seeds 0-9 --repeats 5 --shared-cache --scoring --out $OUT/r11_cmp_f32_512 > $OUT/r11_cmp_f32_512.log 2>&1
timeout 1200 python -m paper_1909_10616_b200.cli compare --m 2048 --k 2048 --n 2048 --family tf32 \
    --max-evals 64 --seeds 0-9 --repeats 5 --shared-cache --scoring --out $OUT/r11_cmp_tf32_2048 > $OUT/r11_cmp_tf32_2048.log 2>&1
tail -12 $OUT/r11_cmp_*.log
