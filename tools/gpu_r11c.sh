set -u
OUT=gpurun_out; mkdir -p $OUT
CFG='{"m":[8,1,1,128],"k":[8,128],"n":[16,1,1,64]}'
for V in base pf; do
  if [ $V = pf ]; then export TT_LIB_PATH=build/variants/pf/libtiletune.so; fi
  timeout 300 python tools/umma_trace.py --m 1024 --n 1024 --k 1024 --config "$CFG" --flush --out $OUT/tr.bin > $OUT/trace1024_${V}_r11c.txt 2>&1
  timeout 300 python tools/small_probe.py 1024 1024 1024 3 --reps 21 --cfg '[[8,1,1,128],[8,128],[16,1,1,64]]' > $OUT/probe1024_${V}_r11c.txt 2>&1
done
unset TT_LIB_PATH
C4='{"m":[16,2,1,128],"k":[32,128],"n":[16,1,1,256]}'
timeout 300 python tools/umma_trace.py --config "$C4" --flush --out $OUT/tr.bin > $OUT/trace4096_r11c.txt 2>&1
for S in 0 1 3 4; do
  TT_TAIL_SPLIT=$S timeout 300 python tools/small_probe.py 4096 4096 4096 3 --reps 15 \
    --cfg '[[16,2,1,128],[32,128],[16,1,1,256]]' --cfg '[[8,2,2,128],[64,64],[16,1,1,256]]' \
    --cfg '[[16,2,1,128],[64,64],[16,1,1,256]]' --cfg '[[16,2,1,128],[64,64],[32,1,1,128]]' \
    --cfg '[[16,2,1,128],[32,128],[8,2,1,256]]' > $OUT/split4096_s${S}_r11c.txt 2>&1
done
rm -f $OUT/tr.bin
