#!/bin/bash
# A/B of the tcgen05 tail split: GPU parity of the UMMA family, then exhaustive
# feasible sweeps and the default bench with the split on and off (TT_TAIL_SPLIT=0).
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x -k "umma or bf16 or tf32 or tail or tn_layout or conv" \
    > $OUT/split_pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/split_pytest.log
tail -3 $OUT/split_pytest.log
for S in 1 0; do
  TT_TAIL_SPLIT=$S timeout 900 python tools/exhaustive.py --m 4096 --k 4096 --n 4096 --family bf16 --budget 64 \
      --seeds 0-2 --out $OUT/split${S}_bf16_4096 > $OUT/split${S}_bf16_4096.log 2>&1
  TT_TAIL_SPLIT=$S timeout 900 python tools/exhaustive.py --m 2048 --k 2048 --n 2048 --family tf32 --budget 64 \
      --seeds 0-2 --out $OUT/split${S}_tf32_2048 > $OUT/split${S}_tf32_2048.log 2>&1
  TT_TAIL_SPLIT=$S timeout 600 python bench.py --no-cpu-baseline > $OUT/split${S}_bench.json 2> $OUT/split${S}_bench.err
  tail -1 $OUT/split${S}_bf16_4096.log; tail -1 $OUT/split${S}_tf32_2048.log; cut -c1-300 $OUT/split${S}_bench.json
done
