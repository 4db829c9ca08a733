set -u
OUT=gpurun_out; mkdir -p $OUT
T=${1:-r11m}
for it in 1 2; do
python tools/e2e_probe.py > $OUT/e2e_A${it}_$T.txt 2>&1
TT_LIB_PATH=build/variants/git-HEAD/libtiletune.so python tools/e2e_probe.py > $OUT/e2e_B${it}_$T.txt 2>&1
done
