set -u
OUT=gpurun_out; mkdir -p $OUT
TT_LIB_PATH=build/variants/apair/libtiletune.so timeout 900 python -m pytest tests/test_gpu.py -q -x -k "simt or fmaf or f32 or k16384" > $OUT/pytest_apair.log 2>&1; echo "rc=$?" >> $OUT/pytest_apair.log
bash tools/ab_simt.sh apair build/variants/apair
