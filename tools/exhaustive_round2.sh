#!/bin/bash
# Round-2 refresh of the G-BFS vs exhaustive sweeps (reading O10) with the round-2 kernels.
set -u
OUT=gpurun_out
timeout 1200 python tools/exhaustive.py --m 4096 --k 4096 --n 4096 --family bf16 --budget 128 --seeds 0-9 --out $OUT/r11_exh_bf16_4096 > $OUT/r11_exh_bf16_4096.log 2>&1
timeout 1200 python tools/exhaustive.py --m 2048 --k 2048 --n 2048 --family tf32 --budget 128 --seeds 0-9 --out $OUT/r11_exh_tf32_2048 > $OUT/r11_exh_tf32_2048.log 2>&1
tail -3 $OUT/r11_exh_*.log
