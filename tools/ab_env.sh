#!/bin/bash
# Interleaved same-build A/B of an environment switch on K1 configs (e.g. TT_SIMT_TMA=0 vs default):
#   bash tools/ab_env.sh TAG 'VAR=VALUE'  -> gpurun_out/ab_TAG.txt  (A = default, B = with VAR=VALUE)
set -u
TAG=$1; ENVSET=$2
OUT=gpurun_out; mkdir -p $OUT
F=$OUT/ab_$TAG.txt; : > $F
probe() {
  timeout 300 python tools/small_probe.py 2048 2048 2048 1 --reps 7 --cfg '[[16,1,16,8],[32,64],[8,8,2,16]]' --cfg '[[16,4,2,16],[32,64],[8,8,4,8]]' --cfg '[[16,4,2,16],[32,64],[8,16,2,8]]'
  timeout 300 python tools/small_probe.py 4096 4096 4096 1 --reps 5 --cfg '[[64,2,2,16],[128,32],[16,16,2,8]]' --cfg '[[64,2,2,16],[128,32],[16,8,4,8]]'
  timeout 300 python tools/small_probe.py 1024 1024 1024 1 --reps 11 --cfg '[[8,2,8,8],[32,32],[8,4,4,8]]' --cfg '[[16,1,8,8],[16,64],[8,4,4,8]]'
  timeout 300 python tools/small_probe.py 512 512 512 1 --reps 11 --cfg '[[8,2,4,8],[16,32],[16,2,8,2]]'
}
for it in 1 2; do
  echo "== A (default) $it" >> $F; probe >> $F 2>&1
  echo "== B ($ENVSET) $it" >> $F; env $ENVSET bash -c "$(declare -f probe); probe" >> $F 2>&1
done
