set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_umma -s 1 -c 1 -o $OUT/prof_r11_bf16_1024 \
  python tools/one_gemm.py 1024 1024 1024 3 '[[8,1,1,128],[8,128],[16,1,1,64]]' --n 2 > $OUT/ncu_r11_1024.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_umma -s 1 -c 1 -o $OUT/prof_r11_bf16_4096 \
  python tools/one_gemm.py 4096 4096 4096 3 '[[16,2,1,128],[32,128],[16,1,1,256]]' --n 2 > $OUT/ncu_r11_4096.log 2>&1
python - > $OUT/sleep_probe_r11d.txt 2>&1 <<'PY'
import torch, json
dev=torch.device('cuda:0'); x=torch.empty(1,device=dev); fl=torch.empty(256<<20,dtype=torch.uint8,device=dev)
e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
def run(pre):
    ts=[]
    for r in range(40):
        pre(r); e0.record(); x.fill_(1.0); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1)*1e3)
    ts.sort(); return ts[20], ts[0]
print(json.dumps({"sleep_then_fill": run(lambda r: torch.cuda._sleep(200000))}))
print(json.dumps({"memset_then_fill": run(lambda r: fl.fill_(r&255))}))
print(json.dumps({"memset_sleep_then_fill": run(lambda r: (fl.fill_(r&255), torch.cuda._sleep(200000)))}))
rd=torch.empty(64<<20,dtype=torch.float32,device=dev)
print(json.dumps({"readflush_then_fill": run(lambda r: rd.sum())}))
PY
