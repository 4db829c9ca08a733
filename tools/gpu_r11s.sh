set -u
OUT=gpurun_out; mkdir -p $OUT
T=${1:-r11s}
timeout 900 python -m pytest tests/test_gpu.py -q -x -k "umma or bf16 or tf32 or split" > $OUT/pytest_umma_$T.log 2>&1; echo "rc=$?" >> $OUT/pytest_umma_$T.log
python tools/floor_probe2.py > $OUT/floor2_$T.txt 2>&1
: > $OUT/splitdef_$T.txt
for it in 1 2; do
  for V in A B; do
    if [ $V = B ]; then export TT_LIB_PATH=build/variants/git-HEAD/libtiletune.so; else unset TT_LIB_PATH; fi
    for W in "bf16_4096 [[16,2,1,128],[32,128],[16,1,1,256]]" "bf16_4096 [[8,2,2,128],[64,64],[16,1,1,256]]" "tf32_4096 [[8,2,2,128],[128,32],[16,1,1,256]]"; do
      set -- $W
      timeout 300 python bench.py --workload $1 --config "$2" --no-fp32 --no-cpu-baseline --steps 50 > $OUT/b.json 2>/dev/null
      python -c "import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); print('$V it $it $1 $2', round(d['value'],1), round(d['ms_per_step']*1e3,2), d['config']['launch'].get('split_tiles'))" >> $OUT/splitdef_$T.txt
    done
  done
done
unset TT_LIB_PATH
