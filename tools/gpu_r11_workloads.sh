# Round-2 bench lines for every reported workload (profiles/r11_workloads/).  Usage: bash tools/gpu_r11_workloads.sh
set -u
OUT=gpurun_out/r11_workloads; mkdir -p $OUT
for W in bf16_4096 bf16_2048 bf16_1024 bf16_8192 bf16_8192_shard8 tf32_4096 tf32_2048 f32_2048 f32_1024; do
  timeout 900 python bench.py --workload $W --no-fp32 --no-cpu-baseline > $OUT/bench_$W.json 2> $OUT/bench_$W.err
done
timeout 1200 python bench.py --workload f32_4096 --no-fp32 --no-cpu-baseline --steps 10 > $OUT/bench_f32_4096.json 2> $OUT/bench_f32_4096.err
timeout 600 python bench.py --layout tn --no-fp32 --no-cpu-baseline > $OUT/bench_bf16_4096_tn.json 2> $OUT/bench_bf16_4096_tn.err
