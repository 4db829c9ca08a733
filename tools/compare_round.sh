#!/bin/bash
# Device-measured G-BFS vs N-A2C vs random search (paper Fig. 8 methodology) on the
# tensor-core families, 10 seeds, each distinct state measured once per run (--shared-cache).
set -u
OUT=gpurun_out
C="python -m paper_1909_10616_b200.cli compare --seeds 0-9 --repeats 5 --shared-cache"
timeout 1500 $C --m 2048 --k 2048 --n 2048 --family tf32 --max-evals 64 --out $OUT/cmp_tf32_2048 > $OUT/cmp_tf32_2048.log 2>&1
timeout 1500 $C --m 4096 --k 4096 --n 4096 --family bf16 --max-evals 64 --out $OUT/cmp_bf16_4096 > $OUT/cmp_bf16_4096.log 2>&1
timeout 1500 $C --m 4096 --k 4096 --n 4096 --family bf16 --max-evals 64 --width 8 --strategies gbfs,random --out $OUT/cmp_bf16_4096_w8 > $OUT/cmp_bf16_4096_w8.log 2>&1
ls -la $OUT/cmp_*
