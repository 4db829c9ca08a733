#!/bin/bash
# A/B cold/warm timing of the working-tree library (A) against build/variants/* (B, C, ...),
# interleaved in one GPU session so box-to-box clock differences cancel.
#   bash tools/ab_probe.sh TAG VARIANT_DIR [VARIANT_DIR ...]   -> gpurun_out/ab_TAG.txt
set -u
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
F=$OUT/ab_$TAG.txt; : > $F
probe() {
  timeout 300 python tools/small_probe.py 1024 1024 1024 3 --reps 21 --cfg '[[8,1,1,128],[8,128],[16,1,1,64]]' --cfg '[[8,1,1,128],[4,256],[16,1,1,64]]'
  timeout 300 python tools/small_probe.py 2048 2048 2048 3 --reps 21 --cfg '[[16,1,1,128],[32,64],[8,1,1,256]]' --cfg '[[8,2,1,128],[16,128],[8,1,1,256]]'
  timeout 300 python tools/small_probe.py 4096 4096 4096 3 --reps 21 --cfg '[[16,2,1,128],[32,128],[16,1,1,256]]' --cfg '[[8,2,2,128],[64,64],[16,1,1,256]]'
}
for it in 1 2; do
  echo "== A (work) $it" >> $F; probe >> $F 2>&1
  L=B
  for VAR in "$@"; do
    echo "== $L ($VAR) $it" >> $F; TT_LIB_PATH=$VAR/libtiletune.so probe >> $F 2>&1
    L=$(echo $L | tr 'A-Y' 'B-Z')
  done
done
