#!/bin/bash
# Extra round evidence: compute-sanitizer over every kernel family (plain, forced tail split,
# graph-replayed measurement) and the cuBLAS same-protocol context.
set -u
TAG=${1:-r4}
OUT=gpurun_out
mkdir -p $OUT
for TOOL in memcheck synccheck racecheck; do
  echo "## $TOOL" >> $OUT/sanitizers_$TAG.md
  timeout 900 compute-sanitizer --tool $TOOL python tools/sanitize_smoke.py 2>&1 | grep -v "^=========     " | tail -25 >> $OUT/sanitizers_$TAG.md
done
timeout 300 python tools/cublas_ref.py $OUT/cublas_ref_$TAG.json > /dev/null 2>&1
