#!/bin/bash
# Round-2 final evidence after the K1 TMA / one-barrier changes (tag r14, final commit): GPU tests, smoke, bench (+ reference arm), ncu launch list and
# --set full capture of the bench kernel, DRAM traffic of the bench config, sanitizers, N = 2
# shared-GPU code path.  Outputs in gpurun_out/; tools/summarize_profiles.py r11 renders profiles/.
set -u
TAG=${1:-r14}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rA > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py --smoke > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref_$TAG.json 2>&1
CFG=$(python -c "import json;d=json.loads(open('$OUT/bench_$TAG.json').read().strip().splitlines()[-1]);c=d['config']['best_config'];print(json.dumps([c['m'],c['k'],c['n']]))")
echo "best config $CFG" >> $OUT/bench_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fp32 > $OUT/launches_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_umma -s 3 -c 1 -o $OUT/prof_$TAG \
    python bench.py --config "$CFG" --steps 3 --warmup 3 --no-cpu-baseline --no-fp32 > $OUT/ncu_full_$TAG.log 2>&1
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum \
    --clock-control none -k regex:k_umma -s 1 -c 1 --csv --log-file $OUT/traffic_$TAG.csv \
    python tools/one_gemm.py 4096 4096 4096 3 "$CFG" --n 2 > /dev/null 2>&1
echo "compute-sanitizer is closed on this pool (see profiles/r11_sanitizers.md for the last run)" > $OUT/sanitizers_$TAG.md
TT_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 --no-fp32 > $OUT/bench_n2share_$TAG.json 2> $OUT/bench_n2share_$TAG.err
echo "n2 shared rc=$?" >> $OUT/bench_n2share_$TAG.err
ls -la $OUT | tail -30
