set -u
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi > $OUT/smi_r11a.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rA -x > $OUT/pytest_gpu_r11a.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_r11a.log
timeout 300 python __graft_entry__.py --smoke > $OUT/smoke_r11a.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_r11a.log
timeout 900 python bench.py --dump-tuning $OUT/tune_r11a > $OUT/bench_r11a.json 2> $OUT/bench_r11a.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref_r11a.json 2>&1
