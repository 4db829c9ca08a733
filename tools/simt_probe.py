import sys
sys.path.insert(0, '.')
from paper_1909_10616_b200 import tiletune as tt
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
ctx = tt.Context(0)
sp = tt.make_space(n, n, n, family=1)
cands = []
for bm, (m1, m2, m3) in {"128a": (2, 8, 8), "128b": (4, 4, 8), "64": (2, 4, 8), "128c": (2, 16, 4), "256": (4, 8, 8)}.items():
    for bn, (n1, n2, n3) in {"128a": (4, 4, 8), "128b": (2, 8, 8), "64": (2, 4, 8), "128c": (4, 2, 16)}.items():
        for bk in (4, 8, 16, 32):
            s = ((n // (m1 * m2 * m3), m1, m2, m3), (n // bk, bk), (n // (n1 * n2 * n3), n1, n2, n3))
            jp, jh = tt.is_legitimate(sp, s)
            if jp and jh:
                cands.append(s)
res = []
for s in cands:
    c = ctx.measure(sp, s, tt.measure_opts(repeats=3)).cost_s
    res.append((c, s))
res.sort()
for c, s in res[:12]:
    b = tt.binding(sp, s)
    print(f"{2*n**3/c/1e12:6.1f} TF/s  {s} threads {b.block_x} tile {b.tile_m}x{b.tile_n}x{b.tile_k}")
