#!/bin/bash
# The paper's main experiment shape (Fig. 7 / Fig. 8) on the B200: (1024,1024,1024)
# fp32 (the paper's arithmetic), 0.1 % of the 899 756-state space = 900 evaluations, 10 seeds,
# G-BFS vs N-A2C vs random search.
OUT=gpurun_out
timeout 3000 python -m paper_1909_10616_b200.cli compare --m 1024 --k 1024 --n 1024 --family f32 --max-evals 900 \
    --seeds 0-9 --repeats 5 --shared-cache --out $OUT/cmp_f32_1024 > $OUT/cmp_f32_1024.log 2>&1
tail -40 $OUT/cmp_f32_1024.log
