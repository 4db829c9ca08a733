"""K1 with A given transposed (TN, W = A^T row-major: no transposing copy) vs NN, same configs,
bench protocol (L2 flushed, 10 repeats).  Question: would a transpose pre-pass + the TN kernel
beat the NN kernel's transposing slab copies?  python tools/simt_tn_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CFGS = {
    2048: [((16, 4, 2, 16), (32, 64), (8, 16, 2, 8)), ((16, 1, 16, 8), (32, 64), (8, 8, 2, 16)),
           ((16, 4, 2, 16), (32, 64), (8, 8, 4, 8))],
    4096: [((64, 2, 2, 16), (128, 32), (16, 16, 2, 8)), ((32, 2, 8, 8), (128, 32), (32, 2, 4, 16))],
}


def main():
    from paper_1909_10616_b200 import tiletune as tt
    ctx = tt.Context(0)
    for M, cfgs in CFGS.items():
        for cfg in cfgs:
            row = {"M": M, "cfg": cfg}
            for name, lay in (("nn", tt.LAYOUT_NN), ("tn", tt.LAYOUT_TN)):
                sp = tt.make_space(M, M, M, family=1, layout=lay)
                if not all(tt.is_legitimate(sp, cfg)):
                    row[name] = None
                    continue
                best = min(ctx.measure(sp, cfg, tt.measure_opts(l2_flush=1)).cost_s for _ in range(3))
                row[name] = round(best * 1e6, 2)
            if row.get("nn") and row.get("tn"):
                row["tn_over_nn"] = round(row["tn"] / row["nn"], 4)
            print(json.dumps(row), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
