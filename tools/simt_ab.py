"""A/B of K1 builds: cost (L2 flushed, 10 repeats) of given fp32 configs; run once per build
(TT_LIB_PATH selects the library).  python tools/simt_ab.py M '[[m..],[k..],[n..]]' ..."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_1909_10616_b200 import tiletune as tt
    M = int(sys.argv[1])
    ctx = tt.Context(0)
    sp = tt.make_space(M, M, M, family=1)
    for c in sys.argv[2:]:
        cfg = tuple(tuple(v) for v in json.loads(c))
        smp = ctx.measure(sp, cfg, tt.measure_opts(l2_flush=1))
        print(json.dumps({"lib": os.environ.get("TT_LIB_PATH", "default"), "M": M, "cfg": cfg,
                          "us": smp.cost_s * 1e6, "tflops": 2 * M ** 3 / smp.cost_s / 1e12}))
    ctx.close()


if __name__ == "__main__":
    main()
