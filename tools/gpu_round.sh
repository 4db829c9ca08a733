#!/bin/bash
# One GPU session: tests, smoke, bench (+ clocks), launch list and one ncu --set full capture of
# the bench's dominant kernel.  Outputs under gpurun_out/ (scratch); summaries are copied into
# profiles/ by tools/summarize_profiles.py on the CPU side.
set -u
TAG=${1:-r2}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu_$TAG.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -rA > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py --smoke > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
CFG=$(python -c "import json;d=json.load(open('$OUT/bench_$TAG.json'));c=d['config']['best_config'];print(json.dumps([c['m'],c['k'],c['n']]))")
echo "best config $CFG" >> $OUT/bench_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/launches_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_umma -s 3 -c 1 -o $OUT/prof_$TAG \
    python bench.py --config "$CFG" --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref_$TAG.json 2>&1
ls -la $OUT
# N > 1 code path on one GPU (gloo, shared device): must print one JSON line and exit 0
TT_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 > $OUT/bench_n2share_$TAG.json 2> $OUT/bench_n2share_$TAG.err
echo "n2 shared rc=$?" >> $OUT/bench_n2share_$TAG.err
