#!/bin/bash
# Interleaved A/B of K1 (fp32 SIMT) configs: working tree (A) vs build/variants/* (B, ...).
#   bash tools/ab_simt.sh TAG VARIANT_DIR [...]  -> gpurun_out/ab_TAG.txt
set -u
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
F=$OUT/ab_$TAG.txt; : > $F
probe() {
  timeout 300 python tools/small_probe.py 2048 2048 2048 1 --reps 7 --cfg '[[16,1,16,8],[32,64],[8,8,2,16]]' --cfg '[[16,4,2,16],[32,64],[8,8,4,8]]'
  timeout 300 python tools/small_probe.py 4096 4096 4096 1 --reps 5 --cfg '[[64,2,2,16],[128,32],[16,16,2,8]]'
  timeout 300 python tools/small_probe.py 1024 1024 1024 1 --reps 11 --cfg '[[8,2,8,8],[32,32],[8,4,4,8]]' --cfg '[[16,1,8,8],[16,64],[8,4,4,8]]'
  timeout 300 python tools/small_probe.py 512 512 512 1 --reps 11 --cfg '[[8,2,4,8],[16,32],[16,2,8,2]]'
}
for it in 1 2; do
  echo "== A (work) $it" >> $F; probe >> $F 2>&1
  L=B
  for VAR in "$@"; do
    echo "== $L ($VAR) $it" >> $F; TT_LIB_PATH=$VAR/libtiletune.so probe >> $F 2>&1
    L=$(echo $L | tr 'A-Y' 'B-Z')
  done
done
