set -u
OUT=gpurun_out; mkdir -p $OUT

TT_HOST_TRACE=1 python tools/e2e_probe.py --reps 3 > $OUT/e2e_trace_r11x.txt 2> $OUT/e2e_trace_r11x.err; echo "rc=$?" >> $OUT/e2e_trace_r11x.err
