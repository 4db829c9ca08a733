set -u
OUT=gpurun_out; mkdir -p $OUT
T=${1:-r11r}
CFG='[[16,2,1,128],[32,128],[16,1,1,256]]'
: > $OUT/split_modes_$T.txt
for it in 1 2 3; do
  for S in 1 4 0; do
    TT_TAIL_SPLIT=$S timeout 300 python bench.py --config "$CFG" --no-fp32 --no-cpu-baseline --steps 50 > $OUT/b.json 2>/dev/null
    python -c "import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); print('mode $S it $it', round(d['value'],1), round(d['ms_per_step']*1e3,2), d['config']['launch'].get('split_tiles'))" >> $OUT/split_modes_$T.txt
  done
done
CFG2='[[8,2,1,128],[16,128],[8,1,1,256]]'
for it in 1 2; do
  for S in 1 4 3; do
    TT_TAIL_SPLIT=$S timeout 300 python bench.py --workload bf16_2048 --config "$CFG2" --no-fp32 --no-cpu-baseline --steps 50 > $OUT/b.json 2>/dev/null
    python -c "import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); print('2048 mode $S it $it', round(d['value'],1), round(d['ms_per_step']*1e3,2), d['config']['launch'].get('split_tiles'))" >> $OUT/split_modes_$T.txt
  done
done
