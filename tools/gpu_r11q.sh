set -u
OUT=gpurun_out; mkdir -p $OUT
T=${1:-r11q}
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$T.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$T.log
bash tools/ab_simt.sh $T build/variants/git-HEAD
timeout 900 python bench.py > $OUT/bench_$T.json 2> $OUT/bench_$T.err
