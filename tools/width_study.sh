#!/bin/bash
# G-BFS width W ("explore from the rho most promising red nodes") studied as an
# algorithm -- best-found cost and evaluations to it vs W at the paper's budget (fp32 2048^3, 0.1 %),
# 10 seeds each, device costs scored by the searches' rules.  Outputs gpurun_out/r11_width_W*.
set -u
OUT=gpurun_out
for W in 1 4 16 32; do
  timeout 1500 python -m paper_1909_10616_b200.cli compare --m 2048 --k 2048 --n 2048 --family f32 \
      --strategies gbfs,random --width $W --max-evals 1590 --seeds 0-9 --repeats 5 --shared-cache --scoring \
      --out $OUT/r11_width_W$W > $OUT/r11_width_W$W.log 2>&1
done
tail -5 $OUT/r11_width_W*.log
