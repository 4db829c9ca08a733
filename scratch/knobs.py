import sys, os, subprocess
cfgs = ["((16,2,1,128),(64,64),(16,1,1,256))", "((16,2,1,128),(64,64),(8,1,2,256))", "((32,1,1,128),(64,64),(16,1,1,256))", "((32,1,1,128),(64,64),(8,1,2,256))", "((16,1,2,128),(64,64),(16,1,1,256))"]
print("configs:", cfgs)
for dbg in [int(x) for x in sys.argv[1:]] or [0, 1, 2, 3, 8, 10]:
    code = f"""
import sys; sys.path.insert(0,'.')
from paper_1909_10616_b200 import tiletune as tt
ctx = tt.Context(0); sp = tt.make_space(4096,4096,4096,family=3)
out = []
for c in [{','.join(cfgs)}]:
    s = ctx.measure(sp, c, tt.measure_opts(repeats=5)).cost_s
    out.append(f"{{2*4096**3/s/1e12:7.1f}}")
print("dbg {dbg}:", " ".join(out))
"""
    env = dict(os.environ, TT_UMMA_DBG=str(dbg))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
    print(r.stdout.strip(), r.stderr.strip()[-300:])
