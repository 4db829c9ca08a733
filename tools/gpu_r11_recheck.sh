set -u
OUT=gpurun_out; mkdir -p $OUT
rm -rf build/variants/trace      # the schedule test must build its trace variant itself, as on a fresh box
timeout 1800 python -m pytest tests -m gpu -q -rA > $OUT/pytest_gpu_r11b.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_r11b.log
timeout 300 python __graft_entry__.py --smoke > $OUT/smoke_r11b.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_r11b.log
timeout 900 python bench.py > $OUT/bench_r11b.json 2> $OUT/bench_r11b.err
