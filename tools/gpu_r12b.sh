#!/bin/bash
# Round-2 (r12b): new GPU tests (two-phase measurement), default bench with the two-phase sharded
# projection, a tuning dump, and the N = 2 shared-GPU code path of the two-phase evaluator.
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu.py -q -x -k "measure_phase or two_phase or replay or racing" > $OUT/pytest_r12b.log 2>&1; echo "rc=$?" >> $OUT/pytest_r12b.log
timeout 900 python bench.py --dump-tuning $OUT/tune_r12b > $OUT/bench_r12b.json 2> $OUT/bench_r12b.err
TT_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 --no-fp32 --no-cpu-baseline > $OUT/bench_n2share_r12b.json 2> $OUT/bench_n2share_r12b.err
echo "n2 rc=$?" >> $OUT/bench_n2share_r12b.err
tail -3 $OUT/pytest_r12b.log; tail -c 400 $OUT/bench_r12b.json; tail -3 $OUT/bench_n2share_r12b.err
