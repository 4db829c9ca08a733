set -u
OUT=gpurun_out; mkdir -p $OUT
T=${1:-r11l}
timeout 600 python -m pytest tests/test_gpu.py -q -x -k "gemm_host" > $OUT/pytest_host_$T.log 2>&1; echo "rc=$?" >> $OUT/pytest_host_$T.log
CFG='[[16,2,1,128],[32,128],[16,1,1,256]]'
for it in 1 2; do
  timeout 600 python bench.py --config "$CFG" --no-fp32 --no-cpu-baseline --steps 20 > $OUT/bench_e2e_A${it}_$T.json 2>/dev/null
  TT_LIB_PATH=build/variants/git-HEAD/libtiletune.so timeout 600 python bench.py --config "$CFG" --no-fp32 --no-cpu-baseline --steps 20 > $OUT/bench_e2e_B${it}_$T.json 2>/dev/null
done
python tools/pcie_probe.py > $OUT/pcie_$T.txt 2>&1
