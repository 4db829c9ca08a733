set -u
F=gpurun_out/ab_r13_onebar16.txt; : > $F
probe() {
  timeout 300 python tools/small_probe.py 1024 1024 1024 1 --reps 11 --cfg '[[16,4,2,8],[8,128],[8,16,2,4]]' --cfg '[[16,1,8,8],[16,64],[8,4,4,8]]' --cfg '[[32,2,2,8],[32,32],[32,4,2,4]]'
  timeout 300 python tools/small_probe.py 512 512 512 1 --reps 11 --cfg '[[64,1,2,4],[8,64],[4,16,2,4]]' --cfg '[[8,2,4,8],[16,32],[16,2,8,2]]'
  timeout 300 python tools/small_probe.py 2048 2048 2048 1 --reps 7 --cfg '[[16,4,2,16],[32,64],[8,16,2,8]]'
}
for it in 1 2; do
  echo "== A (work) $it" >> $F; probe >> $F 2>&1
  echo "== B (onebar16) $it" >> $F; TT_LIB_PATH=build/variants/onebar16/libtiletune.so probe >> $F 2>&1
done
python tools/ab_summary.py $F
