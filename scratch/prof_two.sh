set -x
C1='[[32,1,1,128],[128,32],[8,1,2,256]]'
C2='[[16,2,1,128],[64,64],[8,1,2,256]]'
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_umma -s 3 -c 1 -o gpurun_out/prof_c1 python bench.py --config "$C1" --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_umma -s 3 -c 1 -o gpurun_out/prof_c2 python bench.py --config "$C2" --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/
