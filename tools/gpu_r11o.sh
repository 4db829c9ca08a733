set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_simt -s 1 -c 1 -o $OUT/prof_r11_f32_2048 \
  python tools/one_gemm.py 2048 2048 2048 1 '[[16,1,16,8],[32,64],[8,8,2,16]]' --n 2 > $OUT/ncu_r11_f32_2048.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_simt -s 1 -c 1 -o $OUT/prof_r11_f32_4096 \
  python tools/one_gemm.py 4096 4096 4096 1 '[[64,2,2,16],[128,32],[16,16,2,8]]' --n 2 > $OUT/ncu_r11_f32_4096.log 2>&1
