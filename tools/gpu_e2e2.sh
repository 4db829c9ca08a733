set -u
OUT=gpurun_out; : > $OUT/e2e2.txt
for it in 1 2 3; do
  python tools/e2e_probe.py --reps 20 2>/dev/null | head -1 | sed 's/^/one  /' >> $OUT/e2e2.txt
  TT_HOST_D2H_STREAMS=2 python tools/e2e_probe.py --reps 20 2>/dev/null | head -1 | sed 's/^/two  /' >> $OUT/e2e2.txt
done
TT_HOST_D2H_STREAMS=2 TT_HOST_TRACE=1 python tools/e2e_probe.py --reps 2 > /dev/null 2> $OUT/e2e2_trace.txt
