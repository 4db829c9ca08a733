set -u
OUT=gpurun_out; mkdir -p $OUT
T=${1:-r11k}
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$T.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$T.log
C4='{"m":[16,2,1,128],"k":[32,128],"n":[16,1,1,256]}'
timeout 300 python tools/umma_trace.py --config "$C4" --flush --out $OUT/tr.bin > $OUT/trace4096_$T.txt 2>&1
rm -f $OUT/tr.bin
timeout 900 python bench.py > $OUT/bench_$T.json 2> $OUT/bench_$T.err
