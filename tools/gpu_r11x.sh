set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu.py -q -x -k "default_policy or gemm_host" > $OUT/pytest_r11x.log 2>&1; echo "rc=$?" >> $OUT/pytest_r11x.log
TT_HOST_TRACE=1 python tools/e2e_probe.py --reps 3 > $OUT/e2e_trace_r11x.txt 2> $OUT/e2e_trace_r11x.err
