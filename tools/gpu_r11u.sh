set -u
OUT=gpurun_out; mkdir -p $OUT
T=${1:-r11u}
timeout 900 python -m pytest tests/test_gpu.py -q -x -k "simt or fmaf or k1 or f32 or stream_k or k16384 or gemm_host or plan or measure" > $OUT/pytest_simt_$T.log 2>&1; echo "rc=$?" >> $OUT/pytest_simt_$T.log
: > $OUT/sk_$T.txt
for it in 1 2; do
  for SK in 1 0; do
    TT_SIMT_SK=$SK timeout 300 python tools/small_probe.py 4096 4096 4096 1 --reps 5 --cfg '[[64,2,2,16],[128,32],[16,16,2,8]]' --cfg '[[32,2,8,8],[128,32],[32,2,4,16]]' | sed "s/^/SK=$SK /" >> $OUT/sk_$T.txt
    TT_SIMT_SK=$SK timeout 300 python tools/small_probe.py 2048 2048 2048 1 --reps 7 --cfg '[[16,1,16,8],[32,64],[8,8,2,16]]' --cfg '[[16,2,8,8],[64,32],[16,2,4,16]]' | sed "s/^/SK=$SK /" >> $OUT/sk_$T.txt
  done
done
