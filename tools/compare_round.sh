#!/bin/bash
# Device-measured G-BFS vs N-A2C vs random search (paper Fig. 8 methodology) per workload.
set -u
OUT=gpurun_out
C="python -m paper_1909_10616_b200.cli compare --seeds 0-9 --repeats 5"
timeout 1200 $C --m 512 --k 512 --n 512 --family f32 --max-evals 484 --out $OUT/cmp_f32_512 > $OUT/cmp_f32_512.log 2>&1
timeout 900 $C --m 2048 --k 2048 --n 2048 --family tf32 --max-evals 32 --out $OUT/cmp_tf32_2048 > $OUT/cmp_tf32_2048.log 2>&1
timeout 900 $C --m 4096 --k 4096 --n 4096 --family bf16 --max-evals 24 --out $OUT/cmp_bf16_4096 > $OUT/cmp_bf16_4096.log 2>&1
ls -la $OUT/cmp_*
