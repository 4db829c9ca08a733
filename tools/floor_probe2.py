"""Per-launch time of the bf16 1024^3 best config under three protocols (profiling aid):
cold single launch between events (bench), warm graph replay of 32 launches (tt_measure graph
mode), warm host-loop launches."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1909_10616_b200 import tiletune as tt  # noqa: E402

cfgs = [((8, 1, 1, 128), (8, 128), (16, 1, 1, 64)), ((16, 2, 1, 128), (32, 128), (16, 1, 1, 256))]
ctx = tt.Context(0)
for cfg, n in zip(cfgs, (1024, 4096)):
    sp = tt.make_space(n, n, n, family=tt.FAM_BF16_UMMA)
    ctx.prepare(sp)
    out = {"n": n, "cfg": cfg}
    for name, kw in (("cold_flush", dict(l2_flush=1)), ("warm_graph", dict(l2_flush=0, graph=1)),
                     ("warm_hostloop", dict(l2_flush=0, graph=0))):
        r = ctx.measure(sp, cfg, tt.measure_opts(**kw))
        out[name + "_us"] = r.cost_s * 1e6
    print(json.dumps(out))
ctx.close()
