set -u
OUT=gpurun_out; mkdir -p $OUT
T=${1:-r11e}
timeout 900 python -m pytest tests/test_gpu.py -q -x -k "umma or bf16 or tf32 or split or smoke or plan or measure" > $OUT/pytest_umma_$T.log 2>&1; echo "rc=$?" >> $OUT/pytest_umma_$T.log
CFG='{"m":[8,1,1,128],"k":[8,128],"n":[16,1,1,64]}'
timeout 300 python tools/umma_trace.py --m 1024 --n 1024 --k 1024 --config "$CFG" --flush --out $OUT/tr.bin > $OUT/trace1024_$T.txt 2>&1
C4='{"m":[16,2,1,128],"k":[32,128],"n":[16,1,1,256]}'
timeout 300 python tools/umma_trace.py --config "$C4" --flush --out $OUT/tr.bin > $OUT/trace4096_$T.txt 2>&1
timeout 300 python tools/small_probe.py 1024 1024 1024 3 --reps 21 --cfg '[[8,1,1,128],[8,128],[16,1,1,64]]' --cfg '[[8,1,1,128],[4,256],[16,1,1,64]]' > $OUT/probe1024_$T.txt 2>&1
timeout 300 python tools/small_probe.py 4096 4096 4096 3 --reps 21 --cfg '[[16,2,1,128],[32,128],[16,1,1,256]]' --cfg '[[8,2,2,128],[64,64],[16,1,1,256]]' > $OUT/probe4096_$T.txt 2>&1
timeout 300 python tools/small_probe.py 2048 2048 2048 3 --reps 21 --cfg '[[16,1,1,128],[32,64],[8,1,1,256]]' --cfg '[[8,2,1,128],[16,128],[8,1,1,256]]' > $OUT/probe2048_$T.txt 2>&1
rm -f $OUT/tr.bin
