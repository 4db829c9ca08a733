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
timeout 1200 python bench.py --workload f32_2048 --no-cpu-baseline > $OUT/bench_f32_2048_$TAG.json 2> $OUT/bench_f32_2048_$TAG.err
python - <<'PY' > $OUT/bindings_$TAG.txt 2>&1
from paper_1909_10616_b200 import tiletune as tt
for (M, N, K), cfg in [((4096, 4096, 4096), ((16, 2, 1, 128), (32, 128), (16, 1, 1, 256))),
                       ((4096, 4096, 4096), ((16, 2, 1, 128), (32, 128), (8, 2, 1, 256))),
                       ((8192, 8192, 8192), ((16, 2, 2, 128), (128, 64), (32, 1, 1, 256))),
                       ((8192, 8192, 8192), ((32, 2, 1, 128), (64, 128), (16, 2, 1, 256)))]:
    b = tt.binding(tt.make_space(M, N, K, family=3), cfg)
    print((M, N, K), cfg, "grid", b.grid_x, "cluster", b.cluster_x, "tile", b.tile_m, b.tile_n, b.tile_k,
          "stages", b.stages, "acc", b.acc_buffers, "split", b.split_tiles, b.split_workers)
PY
