set -u
OUT=gpurun_out; mkdir -p $OUT
python -m paper_1909_10616_b200.build > /dev/null
python tools/launch_floor.py > $OUT/floor_r11b.txt 2>&1
for S in 0 1 2; do
  TT_TAIL_SPLIT=$S timeout 600 python tools/small_probe.py 1024 1024 1024 3 --all --top 15 --reps 15 > $OUT/small1024_s${S}_r11b.txt 2>&1
done
TT_TAIL_SPLIT=0 timeout 300 python tools/small_probe.py 2048 2048 2048 3 --all --top 10 --reps 15 > $OUT/small2048_s0_r11b.txt 2>&1
CFG='{"m":[8,1,1,128],"k":[8,128],"n":[16,1,1,64]}'
timeout 300 python tools/umma_trace.py --m 1024 --n 1024 --k 1024 --config "$CFG" --flush --out $OUT/tr1.bin > $OUT/trace1024_r11b.txt 2>&1
timeout 300 python tools/umma_trace.py --m 1024 --n 1024 --k 1024 --config "$CFG" --out $OUT/tr2.bin > $OUT/trace1024_warm_r11b.txt 2>&1
rm -f $OUT/tr1.bin $OUT/tr2.bin
