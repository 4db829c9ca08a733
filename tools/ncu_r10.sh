#!/bin/bash
# ncu captures of round 2 (r10): one --set full capture per kernel family at its reported config,
# plus DRAM bytes of the bf16 4096^3 configs the search tends to find (the bench's traffic table).
# Usage (under gpurun): bash tools/ncu_r10.sh ; reports land in gpurun_out/.
set -u
OUT=gpurun_out
mkdir -p $OUT
full() {   # name M N K fam cfg
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$6" -s 1 -c 1 -o $OUT/prof_r10_$1 \
    python tools/one_gemm.py $2 $3 $4 $5 "$7" --n 2 > $OUT/ncu_r10_$1.log 2>&1
}
full bf16_1024 1024 1024 1024 3 k_umma '[[8,1,1,128],[8,128],[16,1,1,64]]'
full f32_4096 4096 4096 4096 1 k1_simt '[[64,2,2,16],[128,32],[16,16,2,8]]'
full f32_2048 2048 2048 2048 1 k1_simt '[[16,4,2,16],[32,64],[8,8,4,8]]'
full tf32_4096 4096 4096 4096 2 k_umma '[[8,2,2,128],[128,32],[16,1,1,256]]'
full bf16_4096 4096 4096 4096 3 k_umma '[[16,2,1,128],[32,128],[16,1,1,256]]'
# DRAM bytes of the bf16 4096^3 configs the search finds (traffic table for bench.py)
for C in '[[16,2,1,128],[32,128],[16,1,1,256]]' '[[8,2,2,128],[64,64],[16,1,1,256]]' \
         '[[16,2,1,128],[64,64],[16,1,1,256]]' '[[8,2,2,128],[32,128],[16,1,1,256]]' \
         '[[16,1,2,128],[64,64],[16,1,1,256]]' '[[16,2,1,128],[32,128],[8,2,1,256]]'; do
  tag=$(echo "$C" | tr -d '[],' | tr ' ' '_')
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum \
    --clock-control none -k regex:k_umma -s 1 -c 1 --csv --log-file $OUT/traffic_r10_$tag.csv \
    python tools/one_gemm.py 4096 4096 4096 3 "$C" --n 2 > /dev/null 2>&1
done
ls -la $OUT | grep r10
