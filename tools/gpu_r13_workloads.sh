#!/bin/bash
# Final-code bench lines for every workload (tag r13): outputs gpurun_out/r13_wl_<workload>.json
set -u
OUT=gpurun_out
for W in bf16_4096 bf16_8192 bf16_8192_shard8 tf32_4096 tf32_2048 bf16_2048 bf16_1024 f32_1024 f32_512; do
  timeout 600 python bench.py --workload $W --no-fp32 --no-cpu-baseline > $OUT/r13_wl_$W.json 2> $OUT/r13_wl_$W.err
done
timeout 600 python bench.py --workload bf16_4096 --layout tn --no-fp32 --no-cpu-baseline > $OUT/r13_wl_bf16_4096_tn.json 2> $OUT/r13_wl_bf16_4096_tn.err
ls $OUT | grep r13_wl_ | grep -c json
