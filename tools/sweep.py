import sys, json, time
sys.path.insert(0, '.')
from paper_1909_10616_b200 import tiletune as tt
fam = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
ctx = tt.Context(0)
sp = tt.make_space(n, n, n, family=fam)
cfgs, _ = tt.enumerate_feasible(sp)
res = []
t0 = time.time()
for s in cfgs:
    smp = ctx.measure(sp, s, tt.measure_opts(repeats=5))
    b = tt.binding(sp, s)
    res.append((smp.cost_s, s, b.stages, b.acc_buffers, b.tile_m, b.tile_n, b.tile_k))
res.sort()
flops = 2.0 * n ** 3
for c, s, st, ab, tm, tn, tk in res[:25]:
    print(f"{c*1e6:9.1f} us {flops/c/1e12:7.1f} TF/s  {s}  tile {tm}x{tn}x{tk} stages {st} accbuf {ab}")
print('...'); 
for c, s, st, ab, tm, tn, tk in res[-5:]:
    print(f"{c*1e6:9.1f} us {flops/c/1e12:7.1f} TF/s  {s}  tile {tm}x{tn}x{tk} stages {st} accbuf {ab}")
print('sweep s', time.time() - t0, 'configs', len(res))
